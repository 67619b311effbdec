# line-search penetration mask: variant tests (bitwise), self-contact tests, A/B
set -x
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_self_contact.py -x -q > gpurun_out/t17_tests.log 2>&1; tail -2 gpurun_out/t17_tests.log
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['e2e']['value'], d['gpu_launches'])"; }
for i in 1 2; do DP_PEN_MASK=0 run mask0; DP_PEN_MASK=1 run mask1; done
