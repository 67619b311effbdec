# TMA bulk-copy ring in the PCG SpMV (DP_SPMV_BULK) and the fine sweep (DP_SMOOTH_BULK): bitwise digests, A/B
set -x
for v in "DP_SPMV_BULK=0 DP_SMOOTH_BULK=0" "DP_SPMV_BULK=1 DP_SMOOTH_BULK=2"; do env DP_MG_TAIL=1 $v timeout 300 python tests/_variant_run.py | grep DIGEST; done
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=d['kernel_times_insitu']; print('$1', d['value'], r['frac'], r['ms_per_launch']*1e3, 1e3*k['pcg_spmv_ms']/k['pcg_spmv_calls'])"; }
for i in 1 2; do DP_SPMV_BULK=0 run spmv0; DP_SPMV_BULK=1 run spmv1; done
