timeout 600 python tools/spmm_sweep.py --scale 20 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
for v in p8 p16 p16m2; do SLQ_LIB_PATH=variants/$v/libslq_b200.so timeout 600 python tools/spmm_sweep.py --scale 20 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err; done
