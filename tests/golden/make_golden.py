"""Generate golden fixtures by running the *reference* diffproj package.

Test infrastructure only.  Run in the build container (the reference lives
read-only at /root/reference and does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes small ``.npz`` fixtures next to this script.  They pin
``oracle/diffproj_oracle.py`` (CPU restatement) and the CUDA path:

* ``elements.npz``  per-element projection outputs for random and
  degenerate deformation gradients (reference ``elasticity.py:137-324``).
* ``contacts.npz``  per-contact multipliers / blocks / residual rows
  (reference ``contact.py:139-248``) incl. sliding, capped and guarded.
* ``scene_<name>.npz``  full rollouts (``forward.py:251``) with per-step
  states, contact sets and the reverse-sweep gradients
  (``adjoint.py:228``) for a final-state loss.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from diffproj import adjoint as aj  # noqa: E402
from diffproj import contact as ct  # noqa: E402
from diffproj import core  # noqa: E402
from diffproj import elasticity as el  # noqa: E402
from diffproj import forward as fw  # noqa: E402
from diffproj import ident  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------------------
# helpers mirroring the reference tests' fixtures (tests/conftest.py:18-32)


def random_rotation(rng):
    A = rng.standard_normal((3, 3))
    Q, R = np.linalg.qr(A)
    Q = Q * np.sign(np.diag(R))
    if np.linalg.det(Q) < 0:
        Q[:, 0] = -Q[:, 0]
    return Q


def random_F(rng, spread=0.4):
    Q1 = random_rotation(rng)
    Q2 = random_rotation(rng)
    sig = 1.0 + spread * (2.0 * rng.random(3) - 1.0)
    return Q1 @ np.diag(sig) @ Q2.T


def scene_to_arrays(scene):
    """Flatten a reference Scene into plain arrays (our fixture format)."""
    mats = scene.materials
    out = dict(
        vertices=scene.vertices.copy(),
        elements=scene.elements.copy(),
        masses=scene.masses.copy(),
        mat_model=np.array([1 if m.model == "neohookean" else 0 for m in mats],
                           dtype=np.int32),
        mat_E=np.array([m.E for m in mats], dtype=float),
        mat_nu=np.array([m.nu for m in mats], dtype=float),
        mat_stiffness=np.array([m.stiffness for m in mats], dtype=float),
        gravity=scene.gravity.copy(),
        h=np.float64(scene.h),
        eps_fb=np.float64(scene.eps_fb),
        contact_activation=np.float64(scene.contact_activation),
        fext=(np.zeros(0) if scene.fext is None else scene.fext.copy()),
        bind_vertex=np.array([b.vertex for b in scene.bindings], dtype=np.int64),
        bind_target=np.array([b.target for b in scene.bindings],
                             dtype=float).reshape(-1, 3),
        bind_compliance=np.array([b.compliance for b in scene.bindings],
                                 dtype=float),
        col_kind=np.array([0 if c.kind == "halfspace" else 1
                           for c in scene.colliders], dtype=np.int32),
        col_vec=np.array([c.normal if c.kind == "halfspace" else c.center
                          for c in scene.colliders], dtype=float).reshape(-1, 3),
        col_scalar=np.array([c.offset if c.kind == "halfspace" else c.radius
                             for c in scene.colliders], dtype=float),
        col_mu=np.array([c.mu for c in scene.colliders], dtype=float),
    )
    return out


# ---------------------------------------------------------------------------
# per-element goldens


def gen_elements(rng):
    Fs = [random_F(rng) for _ in range(48)]
    # repeated / near-repeated singular values (App. B4 branch, elasticity.py:287-295)
    for sig in ([1.2, 1.2, 0.8], [1.0, 1.0, 1.0], [1.1, 1.1 + 5e-7, 0.9],
                [1.3, 0.9, 0.9], [0.7, 0.7, 0.7], [1.5, 1.0, 1.0 - 1e-9]):
        Fs.append(random_rotation(rng) @ np.diag(sig) @ random_rotation(rng).T)
    Fs.append(np.eye(3))
    Fs = np.array(Fs)
    lame = [el.lame_from_young(5e4, 0.3), el.lame_from_young(1e4, 0.3),
            el.lame_from_young(3e4, 0.45)]
    out = {"F": Fs}
    for tag in ("arap", "nh0", "nh1", "nh2"):
        sig, th, P, W, J, M, N, dmu, dlam, en = ([] for _ in range(10))
        for F in Fs:
            svd = el.svd_polar(F)
            if tag == "arap":
                proj = el.project_arap(svd)
            else:
                mu, lam = lame[int(tag[2])]
                proj = el.project_neohookean(svd, mu, lam)
            jac = el.proj_jacobian(svd, proj,
                                   tau_sigma=1e-6 * float(np.max(svd.sigma)))
            sig.append(svd.sigma)
            th.append(proj.theta)
            P.append(proj.P)
            W.append(proj.W)
            J.append(jac.dP_dF)
            M.append(jac.M_mat)
            N.append(jac.N_mat)
            en.append(proj.energy_density)
            if tag != "arap":
                a, b = el.dP_dlame(svd, proj, mu, lam)
            else:
                a, b = np.zeros((3, 3)), np.zeros((3, 3))
            dmu.append(a)
            dlam.append(b)
        for k, v in (("sigma", sig), ("theta", th), ("P", P), ("W", W),
                     ("dPdF", J), ("M", M), ("N", N), ("dP_dmu", dmu),
                     ("dP_dlam", dlam), ("energy", en)):
            out[f"{tag}_{k}"] = np.array(v)
    out["lame"] = np.array(lame)
    # thin (triangle) SVD path, elasticity.py:156-164, :302-305
    Ft = []
    while len(Ft) < 24:
        F = rng.standard_normal((3, 2)) * 0.3 + np.array(
            [[1, 0], [0, 1], [0, 0]])
        if np.linalg.matrix_rank(F) == 2:
            Ft.append(F)
    Ft = np.array(Ft)
    out["tri_F"] = Ft
    sig, P, J = [], [], []
    for F in Ft:
        svd = el.svd_polar(F)
        proj = el.project_arap(svd)
        jac = el.proj_jacobian(svd, proj,
                               tau_sigma=1e-6 * float(np.max(svd.sigma)))
        sig.append(svd.sigma)
        P.append(proj.P)
        J.append(jac.dP_dF)
    out["tri_sigma"] = np.array(sig)
    out["tri_P"] = np.array(P)
    out["tri_dPdF"] = np.array(J)
    np.savez_compressed(os.path.join(HERE, "elements.npz"), **out)
    print("elements.npz", len(Fs), "tets", len(Ft), "tris")


# ---------------------------------------------------------------------------
# per-contact goldens


def gen_contacts(rng):
    rows = []
    frames, dn_list, qv, qbv, mus, eps = [], [], [], [], [], []
    for k in range(160):
        n = rng.standard_normal(3)
        n /= np.linalg.norm(n)
        t1, t2 = ct._tangent_basis(n)
        frame = np.vstack([n, t1, t2])
        mu = [0.0, 0.1, 0.3, 0.8][k % 4]
        eps2 = [1e-6, 2e-6, 1e-4][k % 3]
        q_bar = rng.standard_normal(3) * 0.1
        dn = 10 ** rng.uniform(-6, -3)
        regime = k % 5
        if regime == 0:      # sliding
            slip = 10 ** rng.uniform(-4, -2)
        elif regime == 1:    # sticking / cone cap
            slip = 10 ** rng.uniform(-8, -6)
        elif regime == 2:    # guarded, |df| < tau
            slip = 10 ** rng.uniform(-12, -9.5)
        elif regime == 3:    # zero slip
            slip = 0.0
        else:
            slip = 10 ** rng.uniform(-7, -3)
        ang = rng.uniform(0, 2 * np.pi)
        df = slip * np.array([np.cos(ang), np.sin(ang)])
        x = q_bar + df[0] * t1 + df[1] * t2
        d_n = float(n @ x) - dn
        frames.append(frame)
        dn_list.append(d_n)
        qv.append(x)
        qbv.append(q_bar)
        mus.append(mu)
        eps.append(eps2)
    lam, delta, s, capped, Kc, kmu, res = ([] for _ in range(7))
    for i in range(len(frames)):
        cp = ct.ContactPoint(vertex=0, frame=frames[i], d_n=dn_list[i],
                             mu=mus[i], eps2=eps[i])
        ct.solve_multipliers(cp, qv[i], qbv[i])
        blk = ct.contact_block(cp)
        lam.append(cp.lam)
        delta.append(cp.delta)
        s.append(cp.s_signed)
        capped.append(cp.cone_capped)
        Kc.append(blk.Kc_local)
        kmu.append(blk.k_mu)
        res.append(ct.contact_residual(cp, qv[i], qbv[i]))
    np.savez_compressed(
        os.path.join(HERE, "contacts.npz"),
        frame=np.array(frames), d_n=np.array(dn_list), q=np.array(qv),
        q_bar=np.array(qbv), mu=np.array(mus), eps2=np.array(eps),
        lam=np.array(lam), delta=np.array(delta), s=np.array(s),
        capped=np.array(capped), Kc=np.array(Kc), k_mu=np.array(kmu),
        residual=np.array(res),
        fb_kat=np.array([ct.fb_smooth(0.0, 0.0, 1e-6)]))
    print("contacts.npz", len(frames))


# ---------------------------------------------------------------------------
# scene rollouts + gradients


def single_tet_scene(model="arap", **mat_kw):
    v = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0],
                  [0.0, 0.0, 1.0]]) * 0.3
    t = np.array([[0, 1, 2, 3]])
    kw = dict(stiffness=1e4, E=5e4, nu=0.3)
    kw.update(mat_kw)
    return core.Scene(vertices=v, elements=t,
                      masses=core.lumped_masses(v, t, density=1000.0),
                      materials=[core.MaterialParams(model=model, **kw)],
                      bindings=[core.BindingSpec(0, v[0], compliance=1e-6)],
                      h=0.01)


def cube_scene(n, model="neohookean", E=1e4, mu=0.3, sphere=False,
               size_total=0.1, gap=5e-4, v0=None):
    """C1-family scene: box_tet_mesh cube resting above a frictional plane
    (SURVEY.md §8(d) item 1)."""
    v, t = ident.box_tet_mesh(n, n, n, size=size_total / n,
                              origin=(0.0, 0.0, gap))
    cols = [core.HalfSpace([0, 0, 1], 0.0, mu=mu)]
    if sphere:
        c = size_total / 2
        cols.append(core.Sphere([c, -0.02 + 1e-4 * 0, c], 0.02 + 0.0004,
                                mu=mu))
    mats = [core.MaterialParams(model=model, E=E, nu=0.3, stiffness=E)
            for _ in range(len(t))]
    return core.Scene(vertices=v, elements=t,
                      masses=core.lumped_masses(v, t, density=1000.0),
                      materials=mats, colliders=cols, h=0.01)


def _label(scene, q, cp):
    """Collider index of a contact: the collider whose normal at the
    contact's vertex reproduces the contact frame (detection order is vertex,
    then collider, contact.py:124-136)."""
    x = q[3 * cp.vertex:3 * cp.vertex + 3]
    for j, col in enumerate(scene.colliders):
        _, nrm = col.gap_normal(x)
        if np.array_equal(nrm, cp.frame[0]) and col.mu == cp.mu:
            return j
    return -1


def run_scene(name, scene, T, tol=1e-12, v0=None, target_shift=1e-3,
              dense_newton=True, before_step=None):
    t0 = time.time()
    state0 = scene.rest_state()
    if v0 is not None:
        state0.v[:] = v0
    cfg = fw.ForwardConfig(tol=tol)
    extra = {}
    if before_step is not None:
        # per-step scene changes (kinematic colliders): forward.rollout's
        # loop (forward.py:251-267) with the hook before every step
        sysmat = core.assemble_system_matrix(scene)
        states, caches, st = [state0.copy()], [], state0
        for k in range(T):
            for key, val in before_step(scene, k).items():
                extra.setdefault(key, []).append(val)
            st, rep = fw.forward_step(scene, st, sysmat, cfg)
            # collider labels while the colliders are where this step saw them
            rep.cache._labels = [_label(scene, rep.cache.q_new, cp) for cp in rep.contacts]
            if not rep.converged:
                raise RuntimeError(f"forward step {k} did not converge "
                                   f"(residual {rep.residual_history[-1]:.3e})")
            states.append(st)
            caches.append(rep.cache)
            print(f"  {name} step {k}: {rep.iterations} its, {len(rep.contacts)} contacts, "
                  f"{time.time() - t0:.0f}s", flush=True)
        extra = {k: np.array(v) for k, v in extra.items()}
    else:
        try:
            states, caches = fw.rollout(scene, state0, T, cfg=cfg)
        except RuntimeError:
            cfg = fw.ForwardConfig()
            states, caches = fw.rollout(scene, state0, T, cfg=cfg)
    target = states[-1].q + target_shift
    grads = aj.backprop_rollout(caches, target)
    out = scene_to_arrays(scene)
    out.update(
        T=np.int64(T), tol=np.float64(cfg.tol), v0=state0.v.copy(),
        q=np.array([s.q for s in states]), v=np.array([s.v for s in states]),
        iterations=np.array([c.report.iterations for c in caches]),
        target=target,
        g_dqbar=grads.dL_dqbar, g_dvbar=grads.dL_dvbar,
        g_dfext=np.array(grads.dL_dfext),
        g_dmu=np.float64(grads.dL_dmu_friction),
        g_dEb=grads.dL_dEb, g_ddb=grads.dL_ddb, g_dw=grads.dL_dw,
        g_dstiffness=np.float64(grads.dL_dstiffness),
        g_dE=np.float64(grads.dL_dE), g_dnu=np.float64(grads.dL_dnu),
        **extra,
    )
    # contact sets per step (vertex, collider) in detection order
    cstep, cvert, ccol, cframe, cdn, clam, cdelta, cs, ccap = \
        ([] for _ in range(9))
    for k, c in enumerate(caches):
        # recover collider index: detection order is vertex-major, collider
        # minor (contact.py:124-136); re-run detection at q_new to label them
        q = c.q_new
        labels = getattr(c, "_labels", None)
        for ci, cp in enumerate(c.contacts):
            cstep.append(k)
            cvert.append(cp.vertex)
            ccol.append(labels[ci] if labels is not None else _label(scene, q, cp))
            cframe.append(cp.frame)
            cdn.append(cp.d_n)
            clam.append(cp.lam)
            cdelta.append(cp.delta)
            cs.append(cp.s_signed)
            ccap.append(cp.cone_capped)
    out.update(c_step=np.array(cstep, dtype=np.int64),
               c_vertex=np.array(cvert, dtype=np.int64),
               c_collider=np.array(ccol, dtype=np.int64),
               c_frame=np.array(cframe).reshape(-1, 3, 3),
               c_dn=np.array(cdn), c_lam=np.array(clam).reshape(-1, 3),
               c_delta=np.array(cdelta).reshape(-1, 3),
               c_s=np.array(cs), c_capped=np.array(ccap, dtype=bool))
    # Newton / adjoint operator of the first step, dense (small scenes only)
    if scene.ndof <= 300 and dense_newton:
        ws = aj.assemble_adjoint_operator(caches[0])
        out["newton_matrix_step1"] = ws.to_dense()
    np.savez_compressed(os.path.join(HERE, f"scene_{name}.npz"), **out)
    print(f"scene_{name}.npz T={T} iters={out['iterations'].tolist()} "
          f"contacts={len(cstep)} tol={cfg.tol} ({time.time() - t0:.1f}s)")


def gen_scenes():
    lib = ident.scene_library()
    run_scene("bar_arap", lib["bar_arap"].copy(), 4)
    run_scene("bar_neohookean", lib["bar_neohookean"].copy(), 4)
    run_scene("hanging_sheet", lib["hanging_sheet"].copy(), 4)
    run_scene("block_on_plane", lib["block_on_plane"].copy(), 10)
    run_scene("friction_high", lib["friction_high"].copy(), 10)
    run_scene("friction_ident", lib["friction_ident"].copy(), 10)
    run_scene("block_lift", lib["block_lift"].copy(), 10)
    tet = single_tet_scene("neohookean")
    run_scene("single_tet_nh", tet, 5)
    # sliding cube on a frictional plane + sphere (all collider kinds)
    sc = cube_scene(2, model="arap", E=5e3, mu=0.3, sphere=True)
    v0 = np.tile([0.3, 0.0, 0.0], sc.n_verts)
    run_scene("cube2_slide", sc, 6, v0=v0)
    # C1-lite: 384 NH tets, E=1e4, mu=0.3 (SURVEY.md §7 parity table)
    run_scene("c1lite", cube_scene(4), 3)


def gen_c1():
    # C1 proper: 4,374 NH tets, E=1e4, mu=0.3
    run_scene("c1", cube_scene(9), 2)


def c5_family_scene(n):
    """The C5 workload family (bench.c5_family) at n cells per side, built
    with the reference's own classes: frictionless ground + two kinematic
    sphere fingers, eps_fb scaled with the vertex mass (55/n)^3."""
    f = (55.0 / n) ** 3
    edge = 0.1 / n
    v, t = ident.box_tet_mesh(n, n, n, size=edge, origin=(0.0, 0.0, 5e-4))
    L = n * edge
    r, zc = 0.02, 5e-4 + L / 2
    cols = [core.HalfSpace([0, 0, 1], 0.0, mu=0.0),
            core.Sphere([-r - 5e-4, L / 2, zc], r, mu=0.0),
            core.Sphere([L + r + 5e-4, L / 2, zc], r, mu=0.0)]
    mats = [core.MaterialParams(model="neohookean", E=1e4, nu=0.3) for _ in range(len(t))]
    return core.Scene(vertices=v, elements=t, masses=core.lumped_masses(v, t, density=1000.0),
                      materials=mats, colliders=cols, h=0.01, eps_fb=1e-9 * f)


def c5_fingers(speed=1e-5, hold=20):
    """bench.move_fingers for the C5 family: close `speed` m per step up to
    finger index `hold`, then hold; returns the finger x centres."""
    def hook(scene, k):
        lx = scene.vertices[:, 0].max()
        p = speed * min(k, hold)
        scene.colliders[1].center[0] = -0.02 - 5e-4 + p
        scene.colliders[2].center[0] = lx + 0.02 + 5e-4 - p
        return {"finger_x": np.array([scene.colliders[1].center[0], scene.colliders[2].center[0]])}
    return hook


def gen_c5family(n=12, T=24, tol=1e-11):
    # the bench workload's regime:
    # C5 family at n^3 cells over the bench finger schedule incl. the hold
    run_scene(f"c5fam{n}", c5_family_scene(n), T, tol=tol, dense_newton=False,
              before_step=c5_fingers())


if __name__ == "__main__":
    rng = np.random.default_rng(0)
    which = sys.argv[1:] or ["elements", "contacts", "scenes"]
    if "elements" in which:
        gen_elements(rng)
    if "contacts" in which:
        gen_contacts(np.random.default_rng(1))
    if "scenes" in which:
        gen_scenes()
    if "c1" in which:
        gen_c1()
    if "c5fam" in which:
        gen_c5family()
