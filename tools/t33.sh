# final C1-C4 lines (GMRES sync changes reverted), GPU parity/variant tests
set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/t33_tests.log 2>&1; tail -2 gpurun_out/t33_tests.log
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --warmup 3 --skip-insitu > gpurun_out/t33_$c.json 2> gpurun_out/t33_$c.err; done
timeout 500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/t33.json 2> gpurun_out/t33.err
