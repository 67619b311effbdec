# Galerkin products of levels >= 2 with 8-lane groups too (DP_GAL8=2)
set -x
for v in 1 2; do DP_GAL8=$v DP_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:galerkin -c 6 --csv python bench.py --steps 1 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | grep galerkin | awk -F'","' -v v=$v '{print "GAL" v, substr($5,1,30), $NF}' | head -6; done
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], sum(d['krylov_iterations']), d['adjoint_krylov_iterations'], sum(d['newton_iterations']))"; }
for i in 1 2; do DP_GAL8=1 run g1; DP_GAL8=2 run g2; done
