"""C5 (or family at n cells) forward K steps + reverse sweep with DP_DEBUG
output: per Newton iteration Krylov counts, per adjoint solve method/iters."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_16478_b200 import adjoint as aj, core, forward as fw  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 55
K = int(sys.argv[2]) if len(sys.argv) > 2 else 6
fam = bench.c5_family(n) if n != 55 else dict(bench.CONFIGS["c5"])
sc = bench.make_scene(fam)
sm = core.assemble_system_matrix(sc)
st = sc.rest_state()
caches = []
t0 = time.time()
for k in range(K):
    bench.move_fingers(sc, k)
    st, rep = fw.forward_step(sc, st, sm, fw.ForwardConfig(tol=fam["tol"], pullback_margin=float(os.environ.get("MARGIN", "1e-6"))))
    print(f"step {k}: its {rep.iterations} kry {rep.krylov_iterations} conv {rep.converged}", file=sys.stderr, flush=True)
    caches.append(rep.cache)
t1 = time.time()
reps = []
g = aj.backprop_rollout(caches, sc.vertices.reshape(-1) + 1e-3,
                        solver_cfg=aj.SolverConfig(tol=1e-10, max_iter=2000, gmres_restart=20), solve_reports=reps)
print("adjoint iters", [r.iterations for r in reps], "fwd", round(t1 - t0, 2), "bwd", round(time.time() - t1, 2),
      file=sys.stderr, flush=True)
