# round-2 final artefacts: GPU tests, bench (driver command), reference arm,
# per-config lines, warm launch list (graphs off so ncu sees the kernels)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t3_gputests.log 2>&1; tail -3 gpurun_out/t3_gputests.log
timeout 500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/t3.json 2> gpurun_out/t3.err; head -c 300 gpurun_out/t3.json
timeout 500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/t3_ref.json 2> gpurun_out/t3_ref.err
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --warmup 3 --skip-insitu > gpurun_out/t3_$c.json 2> gpurun_out/t3_$c.err; done
DP_GRAPHS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/t3_launches.csv python bench.py --steps 20 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu \
  > gpurun_out/t3_ncu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t3_smoke.log 2>&1; tail -2 gpurun_out/t3_smoke.log
