"""Implicit position-velocity step on the GPU (drop-in for diffproj.forward).

``forward_step`` runs the whole condensed Newton solve of the reference
(forward.py:174-248) inside ``dp_forward_step`` of libdiffproj_b200.so:

  predict + pullback -> per Newton iteration: contact detection, element
  projections + projection-Jacobian blocks, contact condensation, residual
  (one fused gather) -> Newton matrix A - dA + K_b + K_c assembled into
  SELL-32 BSR -> multigrid-preconditioned PCG (all contacts frictionless) /
  GMRES (friction) solve -> penetration-aware backtracking line search on
  max|r|.

The reference solves each Newton system exactly with SuperLU
(linsolve.py:386-392); here it is an inexact Krylov solve with a constant
forcing term 1e-3 under the reference's own stop test, so
iterates differ while the converged root agrees to the Newton tolerance.

Reports, caches and contact lists keep the reference field names and are
materialised from device memory lazily (only when a caller reads them).
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import _pinned
from . import core


@dataclass
class ForwardConfig:
    """forward.py:29-34, plus the Krylov controls of the inexact Newton."""

    tol: float = 1e-9
    max_iter: int = 100
    max_line_search: int = 40
    pullback_margin: float = 1e-6
    lin_rtol_max: float = 1e-2     # Krylov rtol while max|r| > 1000 tol
    lin_rtol_min: float = 1e-3     # ... and once it is within 1000 tol
    lin_max_iter: int = 5000
    gmres_restart: int = 50

    def to_c(self):
        c = _lib.ForwardCfg()
        c.tol = self.tol
        c.max_iter = self.max_iter
        c.max_line_search = self.max_line_search
        c.pullback_margin = self.pullback_margin
        c.lin_rtol_max = self.lin_rtol_max
        c.lin_rtol_min = self.lin_rtol_min
        c.lin_max_iter = self.lin_max_iter
        c.gmres_restart = self.gmres_restart
        return c


class DeviceCache:
    """Owner of a ``dp_cache*`` (device copies of q_bar, v_bar, q_hat, q_new,
    the Jacobian-evaluation point and the final contact list)."""

    def __init__(self, dev):
        self.dev = dev
        h = C.c_void_p()
        _lib.check(dev.lib.dp_cache_create(dev.handle, C.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.dev.lib.dp_cache_destroy(h)
            except Exception:
                pass
            self.handle = None

    def n_contacts(self):
        n = C.c_int32()
        _lib.check(self.dev.lib.dp_cache_n_contacts(self.handle, C.byref(n)))
        return n.value

    def states(self):
        n = 3 * self.dev.n_verts
        out = [_pinned.empty(n) for _ in range(4)]   # direct DMA
        _lib.check(self.dev.lib.dp_cache_get_states(self.handle, *[_lib.ptr(a) for a in out]))
        return out

    def contact_arrays(self):
        C_ = self.n_contacts()
        a = dict(vertex=np.empty(C_, np.int32), collider=np.empty(C_, np.int32),
                 frame=np.empty((C_, 3, 3)), d_n=np.empty(C_), mu=np.empty(C_),
                 lam=np.empty((C_, 3)), delta=np.empty((C_, 3)), s_signed=np.empty(C_),
                 capped=np.empty(C_, np.int32))
        if C_:
            _lib.check(self.dev.lib.dp_cache_get_contacts(
                self.handle, _lib.ptr(a["vertex"]), _lib.ptr(a["collider"]), _lib.ptr(a["frame"]),
                _lib.ptr(a["d_n"]), _lib.ptr(a["mu"]), _lib.ptr(a["lam"]), _lib.ptr(a["delta"]),
                _lib.ptr(a["s_signed"]), _lib.ptr(a["capped"])))
        return a

    def projections(self):
        E = self.dev.n_elems
        d = 3 if self.dev.verts_per_elem == 4 else 2
        sig, th = np.empty((E, d)), np.empty((E, d))
        P, en = np.empty((E, 3, d)), np.empty(E)
        _lib.check(self.dev.lib.dp_cache_get_projections(self.dev.handle, self.handle, _lib.ptr(sig),
                                                          _lib.ptr(th), _lib.ptr(P), _lib.ptr(en)))
        return sig, th, P, en


@dataclass
class Projection:
    """elasticity.Projection fields for report.projections."""

    theta: np.ndarray
    P: np.ndarray
    W: np.ndarray | None = None
    energy_density: float = 0.0


class ForwardReport:
    """forward.py:37-44; contacts/projections/contact_residuals are lazy
    (materialised from the step's device cache on first access)."""

    def __init__(self):
        self.residual_history = []
        self.converged = False
        self.iterations = 0
        self.krylov_iterations = 0
        self.line_search_trials = 0
        self.n_contacts = 0
        self.cache = None

    @property
    def contacts(self):
        return self.cache.contacts

    @contacts.setter
    def contacts(self, v):
        self.cache._contacts = v

    @property
    def projections(self):
        return self.cache.elem_caches

    @property
    def contact_residuals(self):
        from . import contact as ct
        return [ct.contact_residual(cp, None, None) for cp in self.contacts]


class _ReportView:
    """``StepCache.report``: the report's fields without a strong reference
    back to the cache.  ForwardReport -> StepCache -> ForwardReport would be a
    reference cycle that only the cyclic GC frees, and the cache owns pooled
    device buffers that must return to the pool when the step is dropped."""

    def __init__(self, rep, cache):
        self.residual_history = rep.residual_history
        self.converged = rep.converged
        self.iterations = rep.iterations
        self.krylov_iterations = rep.krylov_iterations
        self.line_search_trials = rep.line_search_trials
        self.n_contacts = rep.n_contacts
        self._cache = weakref.ref(cache)

    @property
    def cache(self):
        return self._cache()

    @property
    def contacts(self):
        return self._cache().contacts

    @property
    def projections(self):
        return self._cache().elem_caches

    @property
    def contact_residuals(self):
        from . import contact as ct
        return [ct.contact_residual(cp, None, None) for cp in self.contacts]


class StepCache:
    """forward.py:47-60.  State vectors are device-resident; reading a field
    downloads it once.  ``fext`` (scene.external_force() at step time) is
    computed on first access from a snapshot of the scene's fext/gravity."""

    def __init__(self, scene, sysmat, dc, fext, report):
        self.scene = scene
        self.sysmat = sysmat
        self._dc = dc
        self._fext_src = fext
        self._fext = None
        self.report = _ReportView(report, self)
        self._states = None
        self._contacts = None
        self._projections = None

    @property
    def fext(self):
        if self._fext is None and self._fext_src is not None:
            f, g, m = self._fext_src
            grav = m.repeat(3) * np.tile(g, m.size)
            self._fext = grav if f is None else f + grav
        return self._fext

    def _st(self):
        if self._states is None:
            self._states = self._dc.states()
        return self._states

    q_bar = property(lambda self: self._st()[0])
    v_bar = property(lambda self: self._st()[1])
    q_hat = property(lambda self: self._st()[2])
    q_new = property(lambda self: self._st()[3])

    @property
    def contacts(self):
        if self._contacts is None:
            from . import contact as ct
            self._contacts = ct.contacts_from_arrays(self._dc.contact_arrays(), self.scene.eps_fb)
        return self._contacts

    @property
    def elem_caches(self):
        if self._projections is None:
            _, th, P, en = self._dc.projections()
            self._projections = [Projection(theta=th[e], P=P[e], energy_density=float(en[e]))
                                 for e in range(th.shape[0])]
        return self._projections


def binding_multiplier(binding, q):
    """lambda_b = -(J_b q - d_b) / E_b  (forward.py:96-98)."""
    return -(q[binding.dofs()] - binding.target) / binding.compliance


def forward_step(scene, state, sysmat, cfg=None, device_io=None):
    """One implicit step (forward.py:174-248).  Returns (SimState, report);
    ``report.cache`` is the StepCache the adjoint consumes.

    ``device_io`` (optional) = dict(q_bar, v_bar, q_out, v_out) of CUDA
    float64 tensors for a device-resident rollout (no host copies)."""
    cfg = cfg or ForwardConfig()
    dev = sysmat.dev
    L = dev.lib
    dev.sync(scene)
    n = scene.ndof
    rep_c = _lib.ForwardReportC()
    hist = np.empty(max(cfg.max_iter, 1))
    dc = DeviceCache(dev)
    if device_io is None:
        if state.q.shape[0] != n:
            raise ValueError("state does not match scene")
        q0 = _lib.f64(state.q)
        v0 = _lib.f64(state.v)
        # outputs in page-locked memory: the step's device-to-host copies are
        # direct DMA, and the next step's host-to-device copies of them too
        q1 = _pinned.empty(n)
        v1 = _pinned.empty(n)
        kind = _lib.PTR_HOST
    else:
        q0, v0 = device_io["q_bar"], device_io["v_bar"]
        q1, v1 = device_io["q_out"], device_io["v_out"]
        kind = _lib.PTR_DEVICE
    c = cfg.to_c()
    _lib.check(L.dp_forward_step(dev.handle, _lib.ptr(q0), _lib.ptr(v0), kind, C.byref(c),
                                 _lib.ptr(q1), _lib.ptr(v1), dc.handle, C.byref(rep_c),
                                 _lib.ptr(hist), len(hist)))
    report = ForwardReport()
    report.residual_history = hist[:min(rep_c.iterations, len(hist))].tolist()
    report.converged = bool(rep_c.converged)
    report.iterations = int(rep_c.iterations)
    report.krylov_iterations = int(rep_c.krylov_iterations)
    report.line_search_trials = int(rep_c.line_search_trials)
    report.n_contacts = int(rep_c.n_contacts)
    step_index = getattr(state, "step_index", 0) + 1 if state is not None else 0
    # snapshot for StepCache.fext (scene.external_force() at this step)
    fext = (None if scene.fext is None else scene.fext.copy(), scene.gravity.copy(), scene.masses)
    if device_io is not None:
        new_state = None
    elif report.converged:
        new_state = core.SimState._converged(q1, v1, step_index)
    else:
        new_state = core.SimState(q1, v1, step_index)
    report.cache = StepCache(scene, sysmat, dc, fext, report)
    return new_state, report


def rollout(scene, state0, n_steps, sysmat=None, cfg=None, raise_on_failure=True):
    """n_steps implicit steps with per-step caches (forward.py:251-267)."""
    if sysmat is None:
        sysmat = core.assemble_system_matrix(scene)
    states = [state0.copy()]
    caches = []
    state = state0
    for k in range(n_steps):
        state, report = forward_step(scene, state, sysmat, cfg)
        if raise_on_failure and not report.converged:
            raise RuntimeError(f"forward step {k} did not converge "
                               f"(residual {report.residual_history[-1]:.3e})")
        states.append(state)
        caches.append(report.cache)
    return states, caches
