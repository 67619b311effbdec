"""Repeatable timing of a forward(+adjoint) rollout of a bench workload:
R repetitions of the same K-step rollout in one process, median and min
wall time per repetition (the iteration counts are deterministic, so the
spread is host/device noise).  argv: config K R [adjoint 0/1]."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np
import bench
from paper_2603_16478_b200 import adjoint as aj, core, forward as fw

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c5"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 6
R = int(sys.argv[3]) if len(sys.argv) > 3 else 5
adj = len(sys.argv) > 4 and sys.argv[4] == "1"
c = bench.CONFIGS[cfgname]
sc = bench.make_scene(cfgname)
sm = core.assemble_system_matrix(sc)
cfg = fw.ForwardConfig(tol=c["tol"])
times, its, per = [], None, []
for rep in range(R + 1):
    st = sc.rest_state()
    caches = []
    sm.dev.lib.dp_scene_synchronize(sm.dev.handle)
    t0 = time.perf_counter()
    it = []
    steps = []
    for k in range(K):
        bench.move_fingers(sc, k)
        ts = time.perf_counter()
        st, r = fw.forward_step(sc, st, sm, cfg)
        steps.append(round(1e3 * (time.perf_counter() - ts), 1))
        caches.append(r.cache)
        it.append(r.iterations)
    if adj:
        ts = time.perf_counter()
        import os
        rs = int(os.environ.get("ADJ_RESTART", "50"))
        aj.backprop_rollout(caches, sc.rest_state().q + 1e-3, solver_cfg=aj.SolverConfig(tol=1e-10, max_iter=2000, gmres_restart=rs))
        sm.dev.lib.dp_scene_synchronize(sm.dev.handle)
        steps.append(round(1e3 * (time.perf_counter() - ts), 1))
    sm.dev.lib.dp_scene_synchronize(sm.dev.handle)
    dt = time.perf_counter() - t0
    if rep > 0:
        times.append(dt)
        per.append(steps)
    its = it
order = np.argsort(times)
for i in list(order[:3]) + list(order[-3:]):
    print(f"rep {i}: {times[i]:.4f} s, per step ms {per[i]}")
print(json.dumps(dict(config=cfgname, K=K, adjoint=adj, newton=its, median_s=float(np.median(times)),
                      min_s=float(np.min(times)), all=[round(t, 4) for t in times])))
