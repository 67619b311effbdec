# Bench line (default C5 settings) + warm-cache launch list of the bench command.
set -x
timeout 500 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
DP_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 5000 --csv \
  --log-file gpurun_out/f_launches.csv python bench.py --steps 1 --warmup 3 --warmup-seconds 0 --skip-cpu --skip-e2e \
  > gpurun_out/f_ncu.log 2>&1
