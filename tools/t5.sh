# C3 line after the host-path BLAS fix; the cluster tail kernel: ncu --set full and the A/B against the per-level V-cycle
set -x
timeout 600 python bench.py --config c3 --warmup 3 --skip-insitu > gpurun_out/t5_c3.json 2> gpurun_out/t5_c3.err
for t in 0 1 0 1; do DP_MG_TAIL=$t timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-insitu --skip-cpu 2>/dev/null > gpurun_out/t5_tail$t.json; python -c "import json; d=json.load(open('gpurun_out/t5_tail$t.json')); print('TAIL', $t, d['value'], d['e2e']['value'])"; done
DP_GRAPHS=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mg_tail -s 40 -c 1 -o gpurun_out/t5_tail python bench.py --steps 1 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu > gpurun_out/t5_tail_ncu.log 2>&1
DP_GRAPHS=0 DP_MG_TAIL=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/t5_launches_notail.csv python bench.py --steps 20 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu \
  > gpurun_out/t5_ncu.log 2>&1
