# fine sweep with FP32 products/accumulation (DP_SMOOTH_F32ACC): iteration counts and speed
set -x
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', d['value'], r['ms_per_launch']*1e3, sum(d['krylov_iterations']), d['adjoint_krylov_iterations'], sum(d['newton_iterations']))"; }
for i in 1 2; do DP_SMOOTH_F32ACC=0 run acc64; DP_SMOOTH_F32ACC=1 run acc32; done
for c in c1 c3; do for v in 0 1; do DP_SMOOTH_F32ACC=$v timeout 600 python bench.py --config $c --warmup 3 --skip-insitu --skip-cpu --skip-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', $v, d['value'], sum(d['krylov_iterations']), d['adjoint_krylov_iterations'])"; done; done
