# coarse-level sweep ring by TMA bulk copies (DP_COARSE_BULK): digests, kernel times, A/B; host syncs per step
set -x
for v in 0 1; do DP_COARSE_BULK=$v DP_MG_TAIL=1 timeout 300 python tests/_variant_run.py | grep DIGEST; done
for v in 0 1; do DP_COARSE_BULK=$v DP_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mg_smooth -s 300 -c 12 --csv python bench.py --steps 1 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | grep -E "double" | awk -F'","' -v v=$v '{print "COARSE" v, substr($5,1,38), $NF}' | head -4; done
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['e2e']['value'], d['host_syncs_per_step'])"; }
for i in 1 2; do DP_COARSE_BULK=0 run cb0; DP_COARSE_BULK=1 run cb1; done
