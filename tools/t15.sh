# Galerkin product, thread per coarse slot (DP_GAL_THREAD): GPU tests, A/B
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t15_gputests.log 2>&1; tail -2 gpurun_out/t15_gputests.log
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], sum(d['krylov_iterations']), d['adjoint_krylov_iterations'], sum(d['newton_iterations']))"; }
for i in 1 2; do DP_GAL_THREAD=0 run gal0; DP_GAL_THREAD=1 run gal1; done
DP_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:galerkin -c 20 --csv python bench.py --steps 1 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | grep -E "galerkin" | awk -F'","' '{print $5, $NF}' | head -8
