set -x
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err; echo rc=$? >> gpurun_out/r2_bench_c5.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_ref_c5.json 2> gpurun_out/r2_ref_c5.err; echo rc=$? >> gpurun_out/r2_ref_c5.err
python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.err; echo rc=$? >> gpurun_out/r2_bench_c2.err
