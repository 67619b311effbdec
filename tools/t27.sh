# PCG x/r update + Jacobi sweep with one thread per vector entry (DP_XR_ENTRY)
set -x
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], sum(d['krylov_iterations']), d['adjoint_krylov_iterations'], sum(d['newton_iterations']))"; }
for i in 1 2; do DP_XR_ENTRY=0 run xr0; DP_XR_ENTRY=1 run xr1; done
for v in 0 1; do DP_XR_ENTRY=$v DP_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pcg_xr -s 200 -c 20 --csv python bench.py --steps 1 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | grep k_pcg_xr | awk -F'","' -v v=$v '{s+=$NF; n++} END {print "XRNCU", v, s/n, n}'; done
