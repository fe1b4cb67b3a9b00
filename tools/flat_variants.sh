#!/bin/bash
# Variants of the flat SpMM (spmm_flat.cu only; the other objects are compiled once into /tmp/slq_objs):
#   tools/flat_variants.sh name1="-DSLQ_FLAT_NB=4 -DSLQ_FLAT_WARPS=6" ...
# -> variants/<name>/libslq_b200.so (run with SLQ_LIB_PATH)
set -e
cd "$(dirname "$0")/.."
C=paper_2003_01282_b200/csrc
FL="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I include"
mkdir -p /tmp/slq_objs
for f in capi graph lanczos spmm_f32 spmm_f64 step_f32_wide step_f32_narrow step_f64_wide step_f64_narrow rules batched rmat; do
  if [ ! -f /tmp/slq_objs/$f.o ] || [ $C/$f.cu -nt /tmp/slq_objs/$f.o ] || [ $C/engine.cuh -nt /tmp/slq_objs/$f.o ]; then
    nvcc $FL -c $C/$f.cu -o /tmp/slq_objs/$f.o &
  fi
done
wait
for spec in "$@"; do
  name="${spec%%=*}"; defs="${spec#*=}"
  mkdir -p variants/$name
  nvcc $FL $defs -c $C/spmm_flat.cu -o /tmp/slq_objs/spmm_flat_$name.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name/libslq_b200.so /tmp/slq_objs/{capi,graph,lanczos,spmm_f32,spmm_f64,step_f32_wide,step_f32_narrow,step_f64_wide,step_f64_narrow,rules,batched,rmat}.o /tmp/slq_objs/spmm_flat_$name.o
done
