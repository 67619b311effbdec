"""Callers of the hot path: procedural meshes, the identification loss, its
finite-difference check, the gradient-descent driver and its convergence
metrics (the parts of diffproj.ident that drive ``rollout`` /
``backprop_rollout``; reference ident.py:81-316, :320-453).

Host-side Python like the reference.  The finite-difference gradient runs
its 2 x n_params perturbed rollouts concurrently, one scene (CUDA stream)
and host thread each; every rollout is independent,
so the result is bitwise the sequential one.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import adjoint as aj
from . import core
from . import forward as fw

# cube split into six tetrahedra along the main diagonal, one per axis order
_AXIS_ORDERS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


def box_tet_mesh(nx, ny, nz, size=1.0, origin=(0.0, 0.0, 0.0)):
    """Grid of nx*ny*nz cubes, 6 positively oriented tets each (same vertex
    and element order as the reference generator, ident.py:320-352)."""
    n1 = np.array([nx + 1, ny + 1, nz + 1])
    idx = np.stack(np.meshgrid(np.arange(n1[0]), np.arange(n1[1]), np.arange(n1[2]),
                               indexing="ij"), axis=-1).reshape(-1, 3)
    verts = np.asarray(origin, dtype=np.float64) + idx * float(size)
    cubes = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"),
                     axis=-1).reshape(-1, 3)

    def vid(p):
        return (p[..., 0] * n1[1] + p[..., 1]) * n1[2] + p[..., 2]

    tets = np.empty((cubes.shape[0], 6, 4), dtype=np.int64)
    for t, order in enumerate(_AXIS_ORDERS):
        cur = cubes.copy()
        tets[:, t, 0] = vid(cur)
        for k, ax in enumerate(order):
            cur = cur.copy()
            cur[:, ax] += 1
            tets[:, t, k + 1] = vid(cur)
    tets = tets.reshape(-1, 4)
    x = verts[tets]
    det = np.linalg.det(np.stack([x[:, 1] - x[:, 0], x[:, 2] - x[:, 0], x[:, 3] - x[:, 0]], axis=2))
    neg = det < 0
    tets[neg, 2], tets[neg, 3] = tets[neg, 3].copy(), tets[neg, 2].copy()
    return verts, tets


def triangle_sheet(nx, nz, size=0.2, origin=(0.0, 0.0, 0.0)):
    """Vertical sheet in the x-z plane (ident.py:355-369)."""
    j, i = np.meshgrid(np.arange(nz + 1), np.arange(nx + 1), indexing="ij")
    verts = np.stack([origin[0] + i.ravel() * size, np.full(i.size, origin[1]),
                      origin[2] - j.ravel() * size], axis=1)
    jj, ii = np.meshgrid(np.arange(nz), np.arange(nx), indexing="ij")
    a = (jj * (nx + 1) + ii).ravel()
    b, c = a + 1, a + nx + 1
    d = c + 1
    tris = np.stack([np.stack([a, b, c], 1), np.stack([b, d, c], 1)], axis=1).reshape(-1, 3)
    return verts, tris


def horizontal_sheet(nx, ny, size, origin=(0.0, 0.0, 0.0)):
    """Triangle sheet in the x-y plane (C2 cloth)."""
    j, i = np.meshgrid(np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    verts = np.stack([origin[0] + i.ravel() * size, origin[1] + j.ravel() * size,
                      np.full(i.size, origin[2])], axis=1)
    jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    a = (jj * (nx + 1) + ii).ravel()
    b, c = a + 1, a + nx + 1
    d = c + 1
    tris = np.stack([np.stack([a, b, c], 1), np.stack([b, d, c], 1)], axis=1).reshape(-1, 3)
    return verts, tris


def _mats(n, **kw):
    return [core.MaterialParams(**kw) for _ in range(n)]


def scene_library():
    """Desk-scale scenes of the reference test-suite (ident.py:376-453)."""
    out = {}
    v, t = box_tet_mesh(2, 1, 1, size=0.5)
    left = np.nonzero(v[:, 0] == 0.0)[0]
    m = core.lumped_masses(v, t, 1000.0)
    out["bar_arap"] = core.Scene(v, t, m, _mats(len(t), model="arap", stiffness=2e4),
                                 bindings=[core.BindingSpec(i, v[i], 1e-6) for i in left], h=0.01)
    out["bar_neohookean"] = core.Scene(v.copy(), t.copy(), m.copy(),
                                       _mats(len(t), model="neohookean", E=5e4, nu=0.3),
                                       bindings=[core.BindingSpec(i, v[i], 1e-6) for i in left], h=0.01)
    vs, ts = triangle_sheet(3, 3, size=0.2, origin=(0.0, 0.0, 1.0))
    out["hanging_sheet"] = core.Scene(vs, ts, core.lumped_masses(vs, ts, 0.3),
                                      _mats(len(ts), model="arap", stiffness=50.0),
                                      bindings=[core.BindingSpec(i, vs[i], 1e-6) for i in range(4)],
                                      h=0.01)
    vb, tb = box_tet_mesh(1, 1, 1, size=0.4, origin=(0.0, 0.0, 0.001))
    out["block_on_plane"] = core.Scene(vb, tb, core.lumped_masses(vb, tb, 1000.0),
                                       _mats(len(tb), model="arap", stiffness=5e4),
                                       colliders=[core.HalfSpace([0, 0, 1], 0.0, mu=0.0)], h=0.01)
    for tag, mu in (("high", 0.101), ("low", 0.099)):
        out[f"friction_{tag}"] = core.Scene(
            np.array([[0.0, 0.0, 1e-6]]), np.zeros((0, 4), np.int64), np.array([1000.0]), [],
            colliders=[core.HalfSpace([0, 0, 1], 0.0, mu=mu)], eps_fb=1e-6,
            fext=np.array([0.1 * 1000.0 * 9.8, 0.0, 0.0]), h=0.01)
    out["friction_ident"] = core.Scene(
        np.array([[0.0, 0.0, 1e-6]]), np.zeros((0, 4), np.int64), np.array([1.0]), [],
        colliders=[core.HalfSpace([0, 0, 1], 0.0, mu=0.55)], eps_fb=2e-6,
        fext=np.array([6.0, 0.0, 0.0]), h=0.01)
    out["block_lift"] = core.Scene(
        np.array([[0.0, 0.0, 1e-5]]), np.zeros((0, 4), np.int64), np.array([1.0]), [],
        colliders=[core.HalfSpace([0, 0, 1], 0.0, mu=0.0)], eps_fb=2e-1,
        contact_activation=10.0, h=0.01)
    return out


# ---------------------------------------------------------------------------
# identification problem (ident.py:81-216)


def _setter_material(attr, model):
    def f(scene, state0, x):
        for m in scene.materials:
            if m.model == model:
                setattr(m, attr, float(x))
    return f


def _set_mu(scene, state0, x):
    for c in scene.colliders:
        c.mu = float(x)


def _set_fext(axis):
    def f(scene, state0, x):
        g = np.zeros(scene.ndof)
        g[axis::3] = float(x) / scene.n_verts
        scene.fext = g
    return f


def _set_v0(axis):
    def f(scene, state0, x):
        state0.v[axis::3] = float(x)
    return f


def _set_eb(scene, state0, x):
    for b in scene.bindings:
        b.compliance = float(x)


def _set_db_z(scene, state0, x):
    for b in scene.bindings:
        b.target[2] += float(x)


def _get_fext(axis):
    return lambda g, s: sum(float(np.sum(f[axis::3])) for f in g.dL_dfext) / s.n_verts


VARIABLES = {
    "stiffness": (_setter_material("stiffness", "arap"), lambda g, s: g.dL_dstiffness),
    "E": (_setter_material("E", "neohookean"), lambda g, s: g.dL_dE),
    "nu": (_setter_material("nu", "neohookean"), lambda g, s: g.dL_dnu),
    "mu": (_set_mu, lambda g, s: g.dL_dmu_friction),
    "fext_x": (_set_fext(0), _get_fext(0)),
    "fext_y": (_set_fext(1), _get_fext(1)),
    "fext_z": (_set_fext(2), _get_fext(2)),
    "v0_x": (_set_v0(0), lambda g, s: float(np.sum(g.dL_dvbar[0::3]))),
    "v0_z": (_set_v0(2), lambda g, s: float(np.sum(g.dL_dvbar[2::3]))),
    "Eb": (_set_eb, lambda g, s: float(np.sum(g.dL_dEb))),
    "db_z": (_set_db_z, lambda g, s: float(np.sum(g.dL_ddb[:, 2]))),
}


@dataclass
class OptProblem:
    scene: core.Scene
    horizon: int
    variable: str
    init_value: float | np.ndarray
    learning_rate: float = 1.0
    iterations: int = 1
    target_state: np.ndarray | None = None
    target_value: float | np.ndarray | None = None
    log_space: bool = False
    fd_every: int = 0
    fd_eta: float = 1e-4
    initial_velocity: np.ndarray | None = None

    def __post_init__(self):
        # ident.py:119-124
        if self.learning_rate <= 0:
            raise ValueError("learning_rate must be positive")
        self.names()

    def names(self):
        names = [v.strip() for v in str(self.variable).split(",") if v.strip()]
        if not names:
            raise ValueError("empty variable list")
        for n in names:
            if n not in VARIABLES:
                raise ValueError(f"unknown variable {n!r}; known: {sorted(VARIABLES)}")
        return names

    @property
    def scalar(self):
        return len(self.names()) == 1


def _prepared(problem, x):
    scene = problem.scene.copy()
    state0 = scene.rest_state()
    if problem.initial_velocity is not None:
        state0.v[:] = problem.initial_velocity
    xv = np.atleast_1d(np.asarray(x, dtype=np.float64))
    names = problem.names()
    if xv.size != len(names):
        raise ValueError(f"expected {len(names)} parameter values, got {xv.size}")
    for name, xi in zip(names, xv):
        VARIABLES[name][0](scene, state0, xi)
    return scene, state0


def resolve_target(problem, cfg=None):
    """Self-generate the target trajectory at target_value (ident.py:178-186)."""
    if problem.target_state is None:
        if problem.target_value is None:
            raise ValueError("either target_state or target_value required")
        scene, state0 = _prepared(problem, problem.target_value)
        states, _ = fw.rollout(scene, state0, problem.horizon, cfg=cfg)
        problem.target_state = states[-1].q.copy()
    return problem.target_state


def rollout_loss(problem, x, with_grad=False, cfg=None):
    target = resolve_target(problem, cfg)
    scene, state0 = _prepared(problem, x)
    states, caches = fw.rollout(scene, state0, problem.horizon, cfg=cfg)
    L, _ = aj.loss_final_state(states[-1].q, target)
    if not with_grad:
        return L
    grads = aj.backprop_rollout(caches, target)
    g = np.array([VARIABLES[n][1](grads, scene) for n in problem.names()])
    return L, (float(g[0]) if problem.scalar else g)


_MATERIAL_VARS = ("stiffness", "E", "nu")


class FDPool:
    """Pooled device scenes for batched finite differences (SURVEY.md
    §8(f)3).  Each slot owns a scene copy and its device scene, built ONCE;
    a candidate is evaluated by resetting the slot's parameters to the base
    values, applying the candidate through the variable setters, pushing
    only what changed to the device (materials via dp_scene_set_materials;
    colliders, bindings and fext via the per-step sync) and running the
    rollout on the slot's stream.  No scene copy or device-scene rebuild per
    rollout; the slots' rollouts run concurrently on their own streams."""

    def __init__(self, problem, n_slots, device=0):
        self.problem = problem
        self.names = problem.names()
        self.slots = []
        for _ in range(n_slots):
            sc = problem.scene.copy()
            self.slots.append((sc, core.assemble_system_matrix(sc, device)))
        base = problem.scene
        self._base = dict(mats=[(m.E, m.nu, m.stiffness) for m in base.materials],
                          mu=[c.mu for c in base.colliders],
                          fext=None if base.fext is None else base.fext.copy(),
                          binds=[(b.compliance, b.target.copy()) for b in base.bindings])

    def _reset(self, sc):
        b = self._base
        if any(n in _MATERIAL_VARS for n in self.names):
            for m, (E, nu, st) in zip(sc.materials, b["mats"]):
                m.E, m.nu, m.stiffness = E, nu, st
        for c, mu in zip(sc.colliders, b["mu"]):
            c.mu = mu
        sc.fext = None if b["fext"] is None else b["fext"].copy()
        for bd, (comp, tgt) in zip(sc.bindings, b["binds"]):
            bd.compliance, bd.target = comp, tgt.copy()

    def loss(self, slot, x, cfg=None):
        """Rollout loss of candidate x on pooled slot `slot`."""
        problem = self.problem
        sc, sm = self.slots[slot]
        self._reset(sc)
        state0 = sc.rest_state()
        if problem.initial_velocity is not None:
            state0.v[:] = problem.initial_velocity
        xv = np.atleast_1d(np.asarray(x, dtype=np.float64))
        for name, xi in zip(self.names, xv):
            VARIABLES[name][0](sc, state0, xi)
        if any(n in _MATERIAL_VARS for n in self.names):
            sm.dev.set_materials(sc)
            sm._A = sm._elements = None
        states, _ = fw.rollout(sc, state0, problem.horizon, sysmat=sm, cfg=cfg)
        return aj.loss_final_state(states[-1].q, problem.target_state)[0]


def fd_gradient(problem, x, eta=None, cfg=None, workers=None, pool=None, batched=True):
    """Central finite difference of the rollout loss per component
    (ident.py:202-216).  The 2 n perturbed rollouts run concurrently
    (``workers`` host threads, each rollout on its own scene stream).
    batched (default): the rollouts reuse pooled device scenes (FDPool;
    pass ``pool`` to keep it across calls) with the perturbations applied in
    place; batched=False rebuilds a scene per rollout (the reference's
    path, rollout_loss)."""
    if eta is not None and eta <= 0:
        raise ValueError("eta must be positive")
    xv = np.atleast_1d(np.asarray(x, dtype=np.float64))
    resolve_target(problem, cfg)          # once, before the threads start
    steps = []
    for i in range(xv.size):
        e = eta if eta is not None else problem.fd_eta * max(abs(xv[i]), 1.0)
        d = np.zeros(xv.size)
        d[i] = e
        steps.append((e, xv + d, xv - d))
    pts = [p for _, xp, xm in steps for p in (xp, xm)]
    nw = workers if workers is not None else min(len(pts), 8)
    if batched:
        nw = max(1, nw)
        pool = pool or FDPool(problem, nw)
        nw = min(nw, len(pool.slots))
        # candidate i runs on slot i % nw; each slot's candidates in order
        def run_slot(k):
            return [(i, pool.loss(k, pts[i], cfg)) for i in range(k, len(pts), nw)]
        if nw == 1:
            res = run_slot(0)
        else:
            with ThreadPoolExecutor(max_workers=nw) as ex:
                res = [r for part in ex.map(run_slot, range(nw)) for r in part]
        losses = [l for _, l in sorted(res)]
    elif nw <= 1:
        losses = [rollout_loss(problem, p, cfg=cfg) for p in pts]
    else:
        with ThreadPoolExecutor(max_workers=nw) as ex:
            losses = list(ex.map(lambda p: rollout_loss(problem, p, cfg=cfg), pts))
    g = np.array([(losses[2 * i] - losses[2 * i + 1]) / (2 * e) for i, (e, _, _) in enumerate(steps)])
    return float(g[0]) if problem.scalar else g


@dataclass
class OptTrace:
    """ident.py:141-147."""
    losses: list = field(default_factory=list)
    params: list = field(default_factory=list)
    grads_ana: list = field(default_factory=list)
    grads_fd: list = field(default_factory=list)   # None where not computed
    diverged: bool = False


@dataclass
class MetricsReport:
    """ident.py:150-159."""
    t50: float
    t90: float
    auc_e: float
    auc_m: float
    auc_l: float
    mre_e: float
    mre_m: float
    mre_l: float
    degenerate: bool = False


def optimize(problem, use_fd=False, cfg=None):
    """Plain gradient descent, optionally in log-space, with a trace
    (ident.py:219-261).  A forward/adjoint failure (ValueError /
    RuntimeError) ends the run and marks the trace diverged."""
    x = np.atleast_1d(np.asarray(problem.init_value, dtype=np.float64)).copy()
    scalar = problem.scalar

    def unwrap(v):
        v = np.atleast_1d(np.asarray(v, dtype=np.float64))
        return float(v[0]) if scalar else v.copy()

    trace = OptTrace()
    for it in range(problem.iterations):
        try:
            if use_fd:
                L = rollout_loss(problem, x, cfg=cfg)
                g = fd_gradient(problem, x, cfg=cfg)
            else:
                L, g = rollout_loss(problem, x, with_grad=True, cfg=cfg)
            g_fd = None
            if problem.fd_every and it % problem.fd_every == 0:
                g_fd = fd_gradient(problem, x, cfg=cfg)
        except (RuntimeError, ValueError):
            trace.diverged = True
            break
        g = np.atleast_1d(np.asarray(g, dtype=np.float64))
        trace.losses.append(L)
        trace.params.append(unwrap(x))
        trace.grads_ana.append(unwrap(g))
        trace.grads_fd.append(None if g_fd is None else unwrap(g_fd))
        if not np.isfinite(L) or not np.all(np.isfinite(g)):
            trace.diverged = True
            break
        if problem.log_space:
            x = np.exp(np.log(x) - problem.learning_rate * g * x)
        else:
            x = x - problem.learning_rate * g
    return trace


def metrics(trace, eps_g=1e-12):
    """Stage-wise convergence metrics of a trace (ident.py:264-316): t_p =
    first iteration fraction reaching p of the total loss reduction; AUC =
    stage mean of the normalised remaining loss; MRE = stage mean of the
    relative analytic-vs-FD gradient error where an FD gradient exists."""
    L = np.asarray(trace.losses, dtype=np.float64)
    if L.size == 0:
        raise ValueError("empty trace")
    T = L.size - 1
    total = L[0] - L[-1]
    if T == 0 or total <= 0:
        return MetricsReport(t50=1.0, t90=1.0, auc_e=0.0, auc_m=0.0, auc_l=0.0,
                             mre_e=0.0, mre_m=0.0, mre_l=0.0, degenerate=True)
    drop = L[0] - L
    i50 = int(np.argmax(drop >= 0.5 * total))
    i90 = int(np.argmax(drop >= 0.9 * total))
    stages = (np.arange(0, max(i50, 1)), np.arange(i50, max(i90, i50 + 1)), np.arange(i90, T + 1))

    def auc(idx):
        return float(np.mean((L[idx] - L[-1]) / total)) if idx.size else 0.0

    def mre(idx):
        vals = [np.linalg.norm(np.atleast_1d(trace.grads_ana[i]) - np.atleast_1d(trace.grads_fd[i]))
                / (np.linalg.norm(np.atleast_1d(trace.grads_fd[i])) + eps_g)
                for i in idx if i < len(trace.grads_fd) and trace.grads_fd[i] is not None]
        return float(np.mean(vals)) if vals else 0.0

    e, m, l_ = stages
    return MetricsReport(t50=i50 / T, t90=i90 / T, auc_e=auc(e), auc_m=auc(m), auc_l=auc(l_),
                         mre_e=mre(e), mre_m=mre(m), mre_l=mre(l_))
