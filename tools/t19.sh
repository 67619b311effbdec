# one sync per PCG pass (Krylov scalars + true residual together): bitwise variants, syncs per step
set -x
timeout 1200 python -m pytest tests/test_gpu_variants.py -x -q > gpurun_out/t19_var.log 2>&1; tail -2 gpurun_out/t19_var.log
DP_MG_TAIL=1 timeout 300 python tests/_variant_run.py | grep DIGEST
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['e2e']['value'], d['host_syncs_per_step'], sum(d['krylov_iterations']), d['adjoint_krylov_iterations'])"; }
run fused; run fused
