#!/bin/bash
# SpMM A/B over the libraries in variants/*/ (tools/build_variants.sh) on a folded device R-MAT.
#   tools/variant_sweep.sh [scale] [nv]
scale=${1:-26}; nv=${2:-32}
for lib in variants/*/libslq_b200.so; do
  SLQ_LIB_PATH=$lib python tools/spmm_sweep.py --skip-c2 --scale $scale --nv $nv --reps 3
done
