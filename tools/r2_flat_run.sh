set -x
true
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2f_launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-reps 1 > gpurun_out/r2f_ncu_launch.log 2>&1; echo ncu_rc=$? >> gpurun_out/r2f_ncu_launch.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cgs_step|spmm_flat" --launch-skip 40 -c 2 -f -o gpurun_out/r2f_ncu_c5_step_spmm python tools/run_c5.py --reps 1 > gpurun_out/r2f_ncu_full.log 2>&1; echo ncu_rc=$? >> gpurun_out/r2f_ncu_full.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"spmm_flat" --launch-skip 0 -c 1 -f -o gpurun_out/r2f_ncu_c5_step0 python tools/run_c5.py --reps 1 > gpurun_out/r2f_ncu_full0.log 2>&1; echo ncu_rc=$? >> gpurun_out/r2f_ncu_full0.log
