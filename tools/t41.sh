# level-1 sweep with 16 warps per slice (DP_L1_SPLIT16) vs 8 warps + TMA ring
set -x
for v in 0 1; do DP_L1_SPLIT16=$v DP_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mg_smooth -s 40 -c 24 --csv python bench.py --steps 1 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | grep "double" | awk -F'","' -v v=$v '{s+=$NF; n++} END {print "L1", v, s/n, n}'; done
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], sum(d['krylov_iterations']), d['adjoint_krylov_iterations'], sum(d['newton_iterations']))"; }
for i in 1 2; do DP_L1_SPLIT16=0 run s8; DP_L1_SPLIT16=1 run s16; done
