#!/bin/bash
# A/B of the SpMM L2 policies on a folded, hub-marked R-MAT (SLQ_L2_HINT="hub,cold": 0 normal,
# 1 evict_first, 2 evict_last; -1 off).  Usage: tools/l2hint_sweep.sh [scale] [nv]
scale=${1:-26}; nv=${2:-32}
for mode in -1 2,1 0,1 2,0 1,1; do
  SLQ_L2_HINT=$mode python tools/spmm_sweep.py --skip-c2 --scale $scale --nv $nv --reps 3
done
