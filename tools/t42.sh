# round-2 final artefacts (final code): GPU suite, driver bench command x2, reference arm, C1-C4, c2fold, c5f, launch list, smoke
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t42_gputests.log 2>&1; tail -2 gpurun_out/t42_gputests.log
for i in 1 2; do timeout 500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/t42_$i.json 2> gpurun_out/t42_$i.err; done
timeout 500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/t42_ref.json 2> gpurun_out/t42_ref.err
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --warmup 3 --skip-insitu > gpurun_out/t42_$c.json 2> gpurun_out/t42_$c.err; done
timeout 600 python bench.py --config c2fold --warmup 2 --skip-insitu --skip-cpu > gpurun_out/t42_c2fold.json 2> gpurun_out/t42_c2fold.err
timeout 1200 python bench.py --config c5f --steps 20 --warmup 3 --skip-insitu --skip-cpu > gpurun_out/t42_c5f.json 2> gpurun_out/t42_c5f.err
DP_GRAPHS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/t42_launches.csv python bench.py --steps 20 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu \
  > gpurun_out/t42_ncu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t42_smoke.log 2>&1; tail -1 gpurun_out/t42_smoke.log
