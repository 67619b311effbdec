"""GPU side of the preconditioner study (tools/precond_study.py): replay each
fixture's last step on the GPU from the same start state, assemble the
adjoint operator, and solve it for the same rhs with the library's
multigrid-preconditioned Krylov solver (default) and with block-Jacobi
(use_mg = 0): iterations, relative residual, device time.  Writes
profiles/r02_precond_gpu.json."""
import ctypes as C
import glob
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_16478_b200 import _lib, adjoint as aj, core, forward as fw  # noqa: E402

out = []
for path in sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "precond_*.npz"))):
    g = dict(np.load(path))
    name = os.path.basename(path)[8:-4]
    scene = core.scene_from_arrays(g)
    if "finger_x" in g:
        scene.colliders[1].center[0], scene.colliders[2].center[0] = g["finger_x"][-1]
    sm = core.assemble_system_matrix(scene)
    st, rep = fw.forward_step(scene, core.SimState(g["q_bar"], g["v_bar"]), sm,
                              fw.ForwardConfig(tol=float(g["tol"])))
    assert rep.converged, name
    dev = sm.dev
    rows = []
    for label, use_mg in (("multigrid", 2), ("block_jacobi", 0)):
        _lib.check(dev.lib.dp_scene_set_solver_options(dev.handle, use_mg, 0.0, 0))
        ws = aj.assemble_adjoint_operator(rep.cache)
        for rep_i in range(2):   # second run timed (first pays graph capture / warm-up)
            _lib.check(dev.lib.dp_grads_reset(dev.handle))   # no warm start from the previous repeat
            t0 = time.perf_counter()
            try:
                rr = _lib.SolveReportC()
                c = aj.SolverConfig(tol=1e-10, max_iter=2000).to_c()
                gq = np.ascontiguousarray(g["rhs"], dtype=np.float64)
                gv = np.zeros_like(gq)
                z = np.empty_like(gq)
                rc = dev.lib.dp_adjoint_solve(dev.handle, rep.cache._dc.handle, _lib.ptr(gq), _lib.ptr(gv),
                                              _lib.PTR_HOST, C.byref(c), _lib.ptr(z), C.byref(rr))
                dt = time.perf_counter() - t0
                ok = rc == 0
            except Exception as ex:  # noqa: BLE001
                ok, dt = False, time.perf_counter() - t0
        rows.append(dict(precond=label, method="cg" if rr.symmetric else "gmres", iterations=int(rr.iterations),
                         converged=bool(rr.converged), relres=float(rr.rel_residual), solve_s=round(dt, 5)))
        print(name, rows[-1], flush=True)
    _lib.check(dev.lib.dp_scene_set_solver_options(dev.handle, 2, 0.0, 0))
    out.append(dict(scene=name, ndof=scene.ndof, contacts=int(rep.n_contacts), gpu=rows))
json.dump(out, open(os.path.join(ROOT, "profiles", "r02_precond_gpu.json"), "w"), indent=1)
