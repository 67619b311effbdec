set -x
timeout 900 python -m pytest tests/test_gpu_variants.py -x -q > gpurun_out/t7_var.log 2>&1; tail -2 gpurun_out/t7_var.log
for t in 0 1 0 1; do DP_PDL=$t timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-insitu --skip-cpu 2>gpurun_out/t7_err$t.log > gpurun_out/t7_pdl$t.json; python -c "import json; d=json.load(open('gpurun_out/t7_pdl$t.json')); print('PDL', $t, d['value'], d['e2e']['value'], sum(d['krylov_iterations']), d['adjoint_krylov_iterations'])"; done
