for v in "DP_MG_CSWEEP=1" "DP_MG_CSWEEP=2" "DP_MG_CSWEEP=3" "DP_MG_CSWEEP=4"; do
env $v timeout 600 python bench.py --skip-insitu --skip-cpu --skip-e2e --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), sum(d['krylov_iterations']), d['adjoint_krylov_iterations'], sum(d['newton_iterations']))"
done
