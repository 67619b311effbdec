# warm-started element projections (DP_WARM): A/B on C5, element kernel time in situ, iteration counts
set -x
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_times_insitu']; print('$1', d['value'], round(1e3*k['elem_jac_ms']/k['elem_jac_calls'],1), sum(d['krylov_iterations']), d['adjoint_krylov_iterations'], sum(d['newton_iterations']))"; }
for i in 1 2; do DP_WARM=0 run warm0; DP_WARM=1 run warm1; done
for v in 0 1; do DP_WARM=$v DP_MG_TAIL=1 timeout 300 python tests/_variant_run.py | grep DIGEST; done
