# final lines after the GMRES sync changes: C1-C4, c5f, C5 driver command; GPU suite
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t31_gputests.log 2>&1; tail -2 gpurun_out/t31_gputests.log
timeout 500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/t31.json 2> gpurun_out/t31.err
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --warmup 3 --skip-insitu > gpurun_out/t31_$c.json 2> gpurun_out/t31_$c.err; done
timeout 1200 python bench.py --config c5f --steps 20 --warmup 3 --skip-insitu --skip-cpu > gpurun_out/t31_c5f.json 2> gpurun_out/t31_c5f.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t31_smoke.log 2>&1; tail -1 gpurun_out/t31_smoke.log
