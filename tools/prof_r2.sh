set -x
DP_GRAPHS=0 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2e_launches.csv python bench.py --steps 20 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e > gpurun_out/r2e_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mg_smooth -s 2000 -c 1 -o gpurun_out/r2e_smooth python bench.py --steps 4 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e > gpurun_out/r2e_ncu_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pcg_spmv_p -s 500 -c 1 -o gpurun_out/r2e_spmvp python bench.py --steps 4 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e > gpurun_out/r2e_ncu_full2.log 2>&1
