set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t1_gputests.log 2>&1; tail -3 gpurun_out/t1_gputests.log
timeout 500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/t1.json 2> gpurun_out/t1.err; cat gpurun_out/t1.json | head -c 600
for c in c1 c3 c4; do timeout 600 python bench.py --config $c --warmup 3 --skip-insitu > gpurun_out/t1_$c.json 2> gpurun_out/t1_$c.err; done
