# fine sweep: row operands staged in shared memory (bulk path) - bitwise digest + bench
set -x
DP_MG_TAIL=1 timeout 300 python tests/_variant_run.py | grep DIGEST
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', d['value'], r['frac'], r['ms_per_launch']*1e3, r['standalone']['ms_per_launch']*1e3)"; }
for i in 1 2 3; do run staged; done
