timeout 600 python tools/spmm_sweep.py --scale 20 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
SLQ_LIB_PATH=variants/m4/libslq_b200.so timeout 600 python tools/spmm_sweep.py --scale 20 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
