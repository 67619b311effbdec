# final round-2 profile of the dominant kernel (TMA-bulk fine sweep) + launch list + bench line
set -x
timeout 500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/t13.json 2> gpurun_out/t13.err
DP_GRAPHS=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mg_smooth -s 220 -c 2 \
  -o gpurun_out/t13_smooth python bench.py --steps 3 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu \
  > gpurun_out/t13_ncu_full.log 2>&1
DP_GRAPHS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/t13_launches.csv python bench.py --steps 20 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu \
  > gpurun_out/t13_ncu.log 2>&1
