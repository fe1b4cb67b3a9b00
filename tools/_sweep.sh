timeout 600 python tools/spmm_sweep.py >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
for m in 1 4; do SLQ_STEP_M=$m timeout 600 python tools/spmm_sweep.py --skip-c2 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err; done
