set -x
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_ref_c5.json 2> gpurun_out/r2_ref_c5.err; echo rc=$? >> gpurun_out/r2_ref_c5.err
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err; echo rc=$? >> gpurun_out/r2_bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-reps 1 > gpurun_out/r2_ncu_launch.log 2>&1; echo ncu_rc=$? >> gpurun_out/r2_ncu_launch.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cgs_step|spmm_kernel" --launch-skip 40 -c 2 -o gpurun_out/r2_ncu_c5_step_spmm python tools/run_c5.py --reps 1 > gpurun_out/r2_ncu_full.log 2>&1; echo ncu_rc=$? >> gpurun_out/r2_ncu_full.log
