# GMRES: device back substitution, one sync per cycle: tests, C1/C4 lines
set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/t30_tests.log 2>&1; tail -2 gpurun_out/t30_tests.log
for c in c1 c4; do timeout 600 python bench.py --config $c --warmup 3 --skip-insitu --skip-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['e2e']['value'], d['host_syncs_per_step'], sum(d['krylov_iterations']))"; done
