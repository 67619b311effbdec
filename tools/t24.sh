# FP32 float4 gather copy of the PCG pre-sweep iterate (DP_XA32): iterations, sweep time, step rate
set -x
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', d['value'], r['ms_per_launch']*1e3, r['frac'], sum(d['krylov_iterations']), d['adjoint_krylov_iterations'], sum(d['newton_iterations']))"; }
for i in 1 2; do DP_XA32=0 run xa0; DP_XA32=1 run xa1; done
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q > gpurun_out/t24_tests.log 2>&1; tail -2 gpurun_out/t24_tests.log
