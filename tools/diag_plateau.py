"""Diagnostic: Newton histories of the C5 bench rollout (run with DP_DEBUG=3
for the largest residual rows per iteration).  argv: steps [lin_rtol_max]."""
import sys, json, time
sys.path.insert(0, '.')
import bench
from paper_2603_16478_b200 import forward as fw, core

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rmax = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-3
cfgname = sys.argv[3] if len(sys.argv) > 3 else "c5"
rmin = float(sys.argv[4]) if len(sys.argv) > 4 else fw.ForwardConfig().lin_rtol_min
c = bench.CONFIGS[cfgname]
import os
eps = float(os.environ["EPS"]) if "EPS" in os.environ else None
sc = bench.make_scene(cfgname, eps_fb=eps, E=float(os.environ.get("E", bench.E_YOUNG)))
if "TOL" in os.environ:
    c = dict(c, tol=float(os.environ["TOL"]))
sm = core.assemble_system_matrix(sc)
st = sc.rest_state()
cfg = fw.ForwardConfig(tol=c["tol"], lin_rtol_max=rmax, lin_rtol_min=rmin)
T0 = time.time()
for k in range(steps):
    bench.move_fingers(sc, k + int(os.environ.get("K0", "0")))
    t0 = time.time()
    print(f"=== step {k}", file=sys.stderr, flush=True)
    st, rep = fw.forward_step(sc, st, sm, cfg)
    print(json.dumps(dict(k=k, conv=rep.converged, it=rep.iterations, kry=rep.krylov_iterations,
                          ls=rep.line_search_trials, nc=rep.n_contacts, t=round(time.time() - t0, 3), r=rep.residual_history[-1])), flush=True)
print("total", round(time.time() - T0, 3), flush=True)
