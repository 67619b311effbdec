# TMA bulk-copy ring for the fine sweep (DP_SMOOTH_BULK=depth) vs the cp.async ring
set -x
for v in 0 2; do DP_MG_TAIL=1 DP_SMOOTH_BULK=$v timeout 300 python tests/_variant_run.py | grep DIGEST; done
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', d['value'], r['frac'], r['ms_per_launch']*1e3, r['standalone']['ms_per_launch']*1e3)"; }
for i in 1 2; do for v in 0 2 3 4; do DP_SMOOTH_BULK=$v run bulk$v; done; done
