# fine sweep: ring of slot pairs (DP_SMOOTH_BULK=4) vs depth-2 ring with staged row operands (2)
set -x
for v in 2 4; do DP_SMOOTH_BULK=$v DP_MG_TAIL=1 timeout 300 python tests/_variant_run.py | grep DIGEST; done
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', d['value'], r['frac'], r['ms_per_launch']*1e3)"; }
for i in 1 2; do DP_SMOOTH_BULK=2 run b2; DP_SMOOTH_BULK=4 run b4; done
