#!/bin/bash
# SpMM variant sweep on the GPU box (experiments only; variants/ built by tools/build_variants.sh)
cd "$(dirname "$0")/.."
for v in "" $(ls variants 2>/dev/null); do
  lib=""; [ -n "$v" ] && lib="SLQ_LIB_PATH=variants/$v/libslq_b200.so"
  env $lib timeout 600 python tools/spmm_sweep.py --scale 26 --nv 32 --reps 2 "$@" >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
done
