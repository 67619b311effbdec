"""Diagnostic: MG hierarchy + Newton/Krylov stats of the bench scene family.
Runs the rollout twice in one process and reports the second (warm) pass."""
import ctypes as C, json, os, sys, time
import numpy as np
sys.path.insert(0, '.')
import bench
from paper_2603_16478_b200 import forward as fw, core, adjoint as aj, _lib

n = int(sys.argv[1]); steps = int(sys.argv[2]); fingers = sys.argv[3] == '1'
sc = bench.make_scene(n, fingers=fingers)
sm = core.assemble_system_matrix(sc)
L = sm.dev.lib
nl = C.c_int32(); rows = np.zeros(16, np.int32)
L.dp_scene_get_mg_levels(sm.dev.handle, C.byref(nl), _lib.ptr(rows), 16)
print("levels", nl.value, rows[:nl.value].tolist(), flush=True)
cfg = fw.ForwardConfig(lin_rtol_max=float(os.environ.get('ETA_MAX', '1e-3')), gmres_restart=int(os.environ.get('RESTART', '50')), tol=float(os.environ.get('TOL', '1e-9')))
for rep_i in range(2):
    st = sc.rest_state()
    caches, fwd = [], []
    t0 = time.time()
    for k in range(steps):
        bench.move_fingers(sc, k)
        t1 = time.time()
        st, rep = fw.forward_step(sc, st, sm, cfg)
        caches.append(rep.cache)
        fwd.append(dict(k=k, it=rep.iterations, kry=rep.krylov_iterations, ls=rep.line_search_trials,
                        t=round(time.time() - t1, 3)))
    t1 = time.time()
    reps = []
    g = aj.backprop_rollout(caches, st.q + 1e-3, solve_reports=reps)
    tb = time.time() - t1
    if rep_i == 1:
        for f in fwd:
            print(json.dumps(f))
        print("adjoint", round(tb, 3), [r.iterations for r in reps], "dE", g.dL_dE)
        print("total", round(time.time() - t0, 3), flush=True)
