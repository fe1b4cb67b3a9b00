set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; tail -n 3 gpurun_out/r2_pytest_gpu.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err; echo rc=$? >> gpurun_out/r2_bench_c5.err
tail -n 4 gpurun_out/r2_bench_c5.err
python tools/rank_share.py --scale 27 --worlds 1,2,4,8 > gpurun_out/r2_rank_share_c5.json 2> gpurun_out/r2_rank_share_c5.err
cat gpurun_out/r2_rank_share_c5.json
