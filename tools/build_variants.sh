#!/bin/bash
# Build libslq_b200.so variants of lanczos.cu tuning macros into variants/<name>/ (experiments only):
#   tools/build_variants.sh name1="-DSLQ_SPMM_UNR32=8 -DSLQ_SPMM_MINB1=3" name2="..."
set -e
cd "$(dirname "$0")/.."
FLAGS="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I include"
T=$(mktemp -d)
for f in capi graph rules batched rmat; do nvcc $FLAGS -c paper_2003_01282_b200/csrc/$f.cu -o $T/$f.o & done
pids=""
for spec in "$@"; do
  name="${spec%%=*}"; defs="${spec#*=}"
  mkdir -p variants/$name
  nvcc $FLAGS $defs -c paper_2003_01282_b200/csrc/lanczos.cu -o $T/lanczos_$name.o &
done
wait
for spec in "$@"; do
  name="${spec%%=*}"
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name/libslq_b200.so $T/capi.o $T/graph.o $T/rules.o $T/batched.o $T/rmat.o $T/lanczos_$name.o
done
rm -rf $T
