"""SURVEY.md §8(f)1 / VERDICT r1 item 9: the reference's own adjoint
preconditioners (linsolve.py:200-336: Jacobi, sparse-inverse S^T S, Woodbury
with the contact-space Delassus matrix) measured with the REFERENCE code on
the same adjoint systems our GPU solves with the aggregation multigrid.

Runs in the build container only (imports /root/reference read-only).  For
each scene it runs the reference forward for `steps` steps, assembles the
adjoint operator of the last step (adjoint.py:93-120) and solves it for a
seeded random right-hand side with CG (symmetric) or GMRES (friction), once
per preconditioner, recording setup time, solve time, iterations and the
final relative residual.  Writes profiles/r02_precond_reference.json and one
fixture per scene (tests/golden/precond_<name>.npz: scene arrays, the state
the last step starts from, the rhs) that tools/precond_gpu.py replays on the
GPU with the multigrid / block-Jacobi solvers.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import scipy.sparse as sp  # noqa: E402
import scipy.sparse.linalg as spla  # noqa: E402
from diffproj import adjoint as aj, core, forward as fw, linsolve  # noqa: E402
from diffproj.cli import _bench_scene  # noqa: E402

import make_golden as mg  # noqa: E402  (scene_to_arrays, c5_family_scene, cube_scene)


def study(name, scene, steps, hook=None, tol=1e-9):
    sysmat = core.assemble_system_matrix(scene)
    st = scene.rest_state()
    finger = []
    for k in range(steps):
        if hook is not None:
            finger.append(hook(scene, k)["finger_x"])
        prev = st
        st, rep = fw.forward_step(scene, st, sysmat, fw.ForwardConfig(tol=tol))
        if not rep.converged:
            raise RuntimeError(f"{name}: step {k} did not converge")
    ws = aj.assemble_adjoint_operator(rep.cache)
    rng = np.random.default_rng(0)
    rhs = rng.standard_normal(scene.ndof)
    op = ws.apply if ws.symmetric else ws.apply_transpose
    A_base = sp.csc_matrix(ws.A_elastic + sp.diags(ws.kb_diag))
    J = np.zeros((3 * len(ws.contacts), scene.ndof))
    K_blocks = []
    for i, (cp, blk) in enumerate(zip(ws.contacts, ws.contact_blocks)):
        J[3 * i:3 * i + 3, cp.dofs] = cp.frame
        K_blocks.append(blk.Kc_local.T if not ws.symmetric else blk.Kc_local)
    method = "cg" if ws.symmetric else "gmres"
    solver = linsolve.cg if method == "cg" else linsolve.gmres
    cfg = linsolve.SolverConfig(tol=1e-10, max_iter=2000)
    rows = []
    for pname in ("none", "jacobi", "sparse_inverse", "woodbury"):
        t0 = time.perf_counter()
        if pname == "none":
            pre = None
        elif pname == "jacobi":
            pre = linsolve.jacobi_precond(ws.diagonal())
        elif pname == "sparse_inverse":
            pre = linsolve.sparse_inverse_precond(A_base)
        else:
            lu = spla.splu(A_base)
            pre = linsolve.woodbury_precond(lu.solve, J, K_blocks, scene.h)
        t_setup = time.perf_counter() - t0
        t0 = time.perf_counter()
        try:
            _, rep_s = solver(op, rhs, precond=pre, cfg=cfg)
            conv, its, rel = bool(rep_s.converged), int(rep_s.iterations), float(rep_s.residual_history[-1])
        except RuntimeError as ex:
            conv, its, rel = False, None, str(ex)[:80]
        rows.append(dict(precond=pname, method=method, setup_s=round(t_setup, 4),
                         solve_s=round(time.perf_counter() - t0, 4), iterations=its, converged=conv, relres=rel,
                         fallback=bool(getattr(pre, "fallback", False))))
        print(name, rows[-1], flush=True)
    arrs = mg.scene_to_arrays(scene)
    arrs.update(steps=np.int64(steps), tol=np.float64(tol), q_bar=prev.q, v_bar=prev.v, rhs=rhs,
                n_contacts=np.int64(len(ws.contacts)), symmetric=np.int64(ws.symmetric))
    if finger:
        arrs["finger_x"] = np.array(finger)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"precond_{name}.npz"), **arrs)
    return dict(scene=name, ndof=scene.ndof, tets=len(scene.elements), contacts=len(ws.contacts),
                symmetric=bool(ws.symmetric), reference=rows)


def main():
    out = []
    out.append(study("regime_frictionless", _bench_scene("frictionless"), 1))
    out.append(study("regime_frictional", _bench_scene("frictional"), 1))
    out.append(study("c1_cube", mg.cube_scene(9), 2))
    out.append(study("c5fam8", mg.c5_family_scene(8), 3, hook=mg.c5_fingers(), tol=1e-10 * (55 / 8) ** 3))
    json.dump(out, open(os.path.join(ROOT, "profiles", "r02_precond_reference.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
