# canonical-slot assembly (DP_ASM_TSLOT): bitwise digests (frictional C5-family and frictionless bench scene), A/B
set -x
for v in 0 1; do DP_ASM_TSLOT=$v timeout 300 python tests/_variant_run.py | grep DIGEST; done
for v in 0 1; do DP_ASM_TSLOT=$v timeout 300 python bench.py --steps 3 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('DIG', $v, d['krylov_iterations'], d['adjoint_krylov_iterations'])"; done
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_times_insitu']; print('$1', d['value'], 1e3*k['assemble_ms']/k['assemble_calls'])"; }
for i in 1 2; do DP_ASM_TSLOT=0 run tslot0; DP_ASM_TSLOT=1 run tslot1; done
