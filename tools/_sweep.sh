timeout 600 python tools/spmm_sweep.py --scale 20 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
SLQ_SPMM_ASYNC=0 timeout 600 python tools/spmm_sweep.py --scale 20 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
