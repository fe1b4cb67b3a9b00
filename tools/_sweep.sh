timeout 600 python tools/spmm_sweep.py >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
