set -x
for t in 0 1 0 1; do DP_MG_TAIL=$t timeout 300 python bench.py --config c1 --warmup 3 --skip-insitu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1TAIL', $t, d['value'], d['e2e']['value'])"; done
DP_GRAPHS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/t2_launches.csv python bench.py --steps 20 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu \
  > gpurun_out/t2_ncu.log 2>&1
