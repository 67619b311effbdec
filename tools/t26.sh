# coarse multigrid levels reused across Newton iterations of a step (DP_MG_REUSE=k: rebuild every k-th)
set -x
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], sum(d['krylov_iterations']), d['adjoint_krylov_iterations'], sum(d['newton_iterations']))"; }
for i in 1 2; do for k in 1 2 4 1000; do DP_MG_REUSE=$k run reuse$k; done; done
for k in 1 1000; do DP_MG_REUSE=$k timeout 600 python bench.py --config c1 --warmup 3 --skip-insitu --skip-cpu --skip-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1reuse$k', d['value'], sum(d['krylov_iterations']), sum(d['newton_iterations']))"; done
