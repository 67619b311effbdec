# round-2 final artefacts (current code): GPU tests, driver bench command, reference arm, C1-C4, launch list, smoke
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t20_gputests.log 2>&1; tail -2 gpurun_out/t20_gputests.log
timeout 500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/t20.json 2> gpurun_out/t20.err
timeout 500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/t20_ref.json 2> gpurun_out/t20_ref.err
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --warmup 3 --skip-insitu > gpurun_out/t20_$c.json 2> gpurun_out/t20_$c.err; done
DP_GRAPHS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/t20_launches.csv python bench.py --steps 20 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu \
  > gpurun_out/t20_ncu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t20_smoke.log 2>&1; tail -1 gpurun_out/t20_smoke.log
BENCH_SMOKE_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --skip-insitu --skip-cpu > gpurun_out/t20_n2.json 2> gpurun_out/t20_n2.err; tail -c 300 gpurun_out/t20_n2.json
