# Galerkin product skips SELL padding slots: digest, per-launch times, A/B
set -x
DP_MG_TAIL=1 timeout 300 python tests/_variant_run.py | grep DIGEST
DP_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:galerkin -c 6 --csv python bench.py --steps 1 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | grep -E "galerkin" | awk -F'","' '{print substr($5,1,40), $NF}'
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], sum(d['krylov_iterations']), d['adjoint_krylov_iterations'])"; }
for i in 1 2; do run pad; done
