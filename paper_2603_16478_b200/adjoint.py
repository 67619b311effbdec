"""Adjoint backward pass on the GPU (drop-in for diffproj.adjoint).

Per step (reverse time): ``assemble_adjoint_operator`` re-evaluates the
element projections and Jacobian blocks at the cached Newton point and
assembles A_hat^T in SELL-32 BSR (contact blocks transposed);
``solve_adjoint`` solves A_hat^T z = dL/dq + dL/dv / h to the reference's
relative tolerance (default 1e-10) by multigrid-preconditioned PCG (all
mu == 0) or GMRES(50) (adjoint.py:123-139; warm-started from the previous
step's z within a reverse sweep); ``backprop_step`` forms
every z-product (adjoint.py:154-219) with deterministic device reductions.
Parameter gradients accumulate on the device and are read once at the end
of ``backprop_rollout`` (adjoint.py:228-271).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import _pinned
from . import elasticity as el
from .linsolve import SolverConfig, SolveReport


@dataclass
class GradientReport:
    """adjoint.py:70-90 (state gradients refer to the rollout start)."""

    dL_dqbar: np.ndarray | None = None
    dL_dvbar: np.ndarray | None = None
    dL_dfext: list = field(default_factory=list)
    dL_dmu_friction: float = 0.0
    dL_dEb: np.ndarray | None = None
    dL_ddb: np.ndarray | None = None
    dL_dw: np.ndarray | None = None
    dL_dstiffness: float = 0.0
    dL_dE: float = 0.0
    dL_dnu: float = 0.0

    def ensure_shapes(self, n_bind, n_elem):
        if self.dL_dEb is None:
            self.dL_dEb = np.zeros(n_bind)
            self.dL_ddb = np.zeros((n_bind, 3))
        if self.dL_dw is None:
            self.dL_dw = np.zeros(n_elem)


class AdjointWorkspace:
    """A_hat^T assembled on device for one cached step (adjoint.py:25-67)."""

    def __init__(self, step_cache, symmetric):
        self.cache = step_cache
        self.scene = step_cache.scene
        self.symmetric = bool(symmetric)
        self.z = None

    def _dense_T(self):
        return self.cache.sysmat.dev.export_bsr(2).to_dense()

    def to_dense(self):
        """A_hat (untransposed), as the reference's to_dense."""
        return self._dense_T().T

    def apply(self, x):
        return self.to_dense() @ x

    def apply_transpose(self, x):
        return self._dense_T() @ x

    def diagonal(self):
        return np.diag(self._dense_T())


def assemble_adjoint_operator(step_cache):
    """adjoint.py:93-120."""
    dev = step_cache.sysmat.dev
    sym = C.c_int32()
    _lib.check(dev.lib.dp_adjoint_assemble(dev.handle, step_cache._dc.handle, C.byref(sym)))
    return AdjointWorkspace(step_cache, sym.value)


def solve_adjoint(workspace, dL_dq, dL_dv, solver_cfg=None, report=None):
    """A_hat^T z = dL/dq + (1/h) dL/dv  (adjoint.py:123-139)."""
    cfg = solver_cfg or SolverConfig(tol=1e-10, max_iter=2000)
    cache = workspace.cache
    dev = cache.sysmat.dev
    n = workspace.scene.ndof
    gq = _lib.f64(dL_dq)
    gv = _lib.f64(dL_dv)
    z = np.empty(n)
    rep = _lib.SolveReportC()
    c = cfg.to_c()
    _lib.check(dev.lib.dp_adjoint_solve(dev.handle, cache._dc.handle, _lib.ptr(gq), _lib.ptr(gv),
                                        _lib.PTR_HOST, C.byref(c), _lib.ptr(z), C.byref(rep)))
    if report is not None:
        report.converged = bool(rep.converged)
        report.iterations = rep.iterations
        report.residual_history = [rep.rel_residual]
    if not rep.converged:
        # adjoint.py:134-137
        raise RuntimeError("adjoint solve did not converge; residual history tail "
                           f"{[rep.rel_residual]}")
    workspace.z = z
    return z


def backprop_step(step_cache, z, dL_dq, dL_dv, grads=None):
    """adjoint.py:154-219.  Parameter gradients of this step are added to the
    device accumulators and folded into ``grads``."""
    dev = step_cache.sysmat.dev
    scene = step_cache.scene
    n = scene.ndof
    if grads is None:
        grads = GradientReport()
    grads.ensure_shapes(len(scene.bindings), dev.n_elems)
    zz = _lib.f64(z)
    gv = _lib.f64(dL_dv)
    dqbar, dvbar, dfext = np.empty(n), np.empty(n), np.empty(n)
    _lib.check(dev.lib.dp_grads_reset(dev.handle))
    _lib.check(dev.lib.dp_backprop_step(dev.handle, step_cache._dc.handle, _lib.ptr(zz), _lib.ptr(gv),
                                        _lib.PTR_HOST, _lib.ptr(dqbar), _lib.ptr(dvbar),
                                        _lib.ptr(dfext)))
    _fold_device_grads(dev, scene, grads)
    grads.dL_dfext.append(dfext)
    return grads, dqbar, dvbar


def _read_device_grads(dev, scene):
    gs = _lib.GradScalars()
    _lib.check(dev.lib.dp_grads_get(dev.handle, C.byref(gs)))
    nb = len(scene.bindings)
    dw = np.zeros(dev.n_elems)
    dEb = np.zeros(nb)
    ddb = np.zeros((nb, 3))
    _lib.check(dev.lib.dp_grads_get_arrays(dev.handle, _lib.ptr(dw), _lib.ptr(dEb), _lib.ptr(ddb)))
    return gs, dw, dEb, ddb


def _fold_device_grads(dev, scene, grads):
    gs, dw, dEb, ddb = _read_device_grads(dev, scene)
    grads.dL_dmu_friction += gs.dL_dmu_friction
    grads.dL_dstiffness += gs.dL_dstiffness
    grads.dL_dw = grads.dL_dw + dw
    grads.dL_dEb = grads.dL_dEb + dEb
    grads.dL_ddb = grads.dL_ddb + ddb
    _chain_lame(scene, gs.dmu_lame, gs.dlam_lame, grads)


def device_gradient_report(dev, scene, device):
    """GradientReport of the device accumulators with the per-element and
    per-binding arrays left on the GPU (torch float64 tensors on `device`):
    the packed-gradient all-reduce (parallel.pack_gradients) then never goes
    through the host."""
    import torch
    gs = _lib.GradScalars()
    _lib.check(dev.lib.dp_grads_get(dev.handle, C.byref(gs)))
    nb = len(scene.bindings)
    dd = dict(device=device, dtype=torch.float64)
    g = GradientReport(dL_dw=torch.empty(dev.n_elems, **dd), dL_dEb=torch.empty(nb, **dd),
                       dL_ddb=torch.empty((nb, 3), **dd))
    _lib.check(dev.lib.dp_grads_get_arrays(dev.handle, _lib.ptr(g.dL_dw) if dev.n_elems else None,
                                           _lib.ptr(g.dL_dEb) if nb else None,
                                           _lib.ptr(g.dL_ddb) if nb else None))
    g.dL_dmu_friction = gs.dL_dmu_friction
    g.dL_dstiffness = gs.dL_dstiffness
    _chain_lame(scene, gs.dmu_lame, gs.dlam_lame, g)
    return g


def _chain_lame(scene, dmu, dlam, grads):
    """[dE, dnu] = J_lame^T [dmu, dlam] with the first NH element's (E, nu)
    (adjoint.py:211-217)."""
    if not (dmu or dlam):
        return
    first = next((m for m in scene.materials if m.model == "neohookean"), None)
    if first is None:
        return
    dE, dnu = el.lame_jacobian(first.E, first.nu).T @ np.array([dmu, dlam])
    grads.dL_dE += float(dE)
    grads.dL_dnu += float(dnu)


def loss_final_state(q_final, q_target):
    """L = |q - q*|^2 and dL/dq (adjoint.py:222-225)."""
    d = np.asarray(q_final, dtype=np.float64) - np.asarray(q_target, dtype=np.float64)
    # einsum, not BLAS ddot: a threaded ddot leaves OpenBLAS workers spinning
    # on every core for milliseconds, which starves the host threads of
    # concurrent rollouts (measured: C3 public-API path 455 -> 260 steps/s)
    return float(np.einsum("i,i->", d, d)), 2.0 * d


def _torch_cuda():
    """torch with CUDA if importable (device-resident reverse sweep), else None."""
    try:
        import torch
    except ImportError:
        return None
    return torch if torch.cuda.is_available() else None


def backprop_rollout(caches, loss_spec, solver_cfg=None, solve_reports=None):
    """Reverse sweep over the cached steps (adjoint.py:228-271).

    loss_spec: target positions (final-state squared loss) or a callable
    (k, q, v) -> (dL/dq, dL/dv) with 1-based k."""
    if not caches:
        raise ValueError("empty rollout")
    scene = caches[0].scene
    dev = caches[0].sysmat.dev
    n = scene.ndof
    T = len(caches)
    if callable(loss_spec):
        loss_fn = loss_spec
    else:
        target = np.asarray(loss_spec, dtype=np.float64)

        def loss_fn(k, q, v):
            if k == T:
                return loss_final_state(q, target)[1], np.zeros(n)
            return np.zeros(n), np.zeros(n)
    cfg = solver_cfg or SolverConfig(tol=1e-10, max_iter=2000)
    c = cfg.to_c()
    L = dev.lib
    _lib.check(L.dp_grads_reset(dev.handle))
    fext = [None] * T

    def check_solve(rep, k):
        if solve_reports is not None:
            solve_reports.append(SolveReport(residual_history=[rep.rel_residual],
                                             converged=bool(rep.converged),
                                             iterations=rep.iterations))
        if not rep.converged:
            # adjoint.py:134-137
            raise RuntimeError(f"adjoint solve did not converge at step {k}; residual history tail "
                               f"{[rep.rel_residual]}")

    torch = _torch_cuda()
    if torch is not None:
        # the adjoint state chain (dL/dq, dL/dv -> z -> dL/dq_bar, dL/dv_bar)
        # stays on the device; loss gradients go up and dL/dfext comes down
        dd = dict(device="cuda:%d" % dev.device, dtype=torch.float64)
        stream = torch.cuda.ExternalStream(L.dp_scene_stream(dev.handle), device=dd["device"])
        with torch.cuda.stream(stream):
            dq, dv = torch.zeros(n, **dd), torch.zeros(n, **dd)
            z, dqb, dvb, f = (torch.empty(n, **dd) for _ in range(4))
            for k in range(T, 0, -1):
                cache = caches[k - 1]
                if callable(loss_spec) or k == T:
                    q_new = cache.q_new
                    gq, gv = loss_fn(k, q_new, (q_new - cache.q_bar) / scene.h)
                    dq += torch.from_numpy(_lib.f64(gq)).to(dd["device"], non_blocking=False)
                    dv += torch.from_numpy(_lib.f64(gv)).to(dd["device"], non_blocking=False)
                _lib.check(L.dp_adjoint_assemble(dev.handle, cache._dc.handle, None))
                rep = _lib.SolveReportC()
                _lib.check(L.dp_adjoint_solve(dev.handle, cache._dc.handle, _lib.ptr(dq), _lib.ptr(dv),
                                              _lib.PTR_DEVICE, C.byref(c), _lib.ptr(z), C.byref(rep)))
                check_solve(rep, k)
                _lib.check(L.dp_backprop_step(dev.handle, cache._dc.handle, _lib.ptr(z), _lib.ptr(dv),
                                              _lib.PTR_DEVICE, _lib.ptr(dqb), _lib.ptr(dvb), _lib.ptr(f)))
                # dL/dfext of the step, straight into page-locked host memory
                fk = _pinned.empty(n)
                torch.from_numpy(fk).copy_(f, non_blocking=True)
                fext[k - 1] = fk
                dq, dqb = dqb, dq
                dv, dvb = dvb, dv
            stream.synchronize()   # the non-blocking dL/dfext copies have landed
            dq = dq.cpu().numpy()
            dv = dv.cpu().numpy()
    else:
        dq = np.zeros(n)
        dv = np.zeros(n)
        z = np.empty(n)
        dqbar, dvbar = np.empty(n), np.empty(n)
        for k in range(T, 0, -1):
            cache = caches[k - 1]
            if callable(loss_spec) or k == T:
                q_new = cache.q_new
                gq, gv = loss_fn(k, q_new, (q_new - cache.q_bar) / scene.h)
                dq = dq + gq
                dv = dv + gv
            dq = _lib.f64(dq)
            dv = _lib.f64(dv)
            _lib.check(L.dp_adjoint_assemble(dev.handle, cache._dc.handle, None))
            rep = _lib.SolveReportC()
            _lib.check(L.dp_adjoint_solve(dev.handle, cache._dc.handle, _lib.ptr(dq), _lib.ptr(dv),
                                          _lib.PTR_HOST, C.byref(c), _lib.ptr(z), C.byref(rep)))
            check_solve(rep, k)
            f = np.empty(n)
            _lib.check(L.dp_backprop_step(dev.handle, cache._dc.handle, _lib.ptr(z), _lib.ptr(dv),
                                          _lib.PTR_HOST, _lib.ptr(dqbar), _lib.ptr(dvbar), _lib.ptr(f)))
            fext[k - 1] = f
            dq, dv = dqbar.copy(), dvbar.copy()
    grads = GradientReport()
    grads.ensure_shapes(len(scene.bindings), dev.n_elems)
    _fold_device_grads(dev, scene, grads)
    grads.dL_dfext = fext
    grads.dL_dqbar = dq
    grads.dL_dvbar = dv
    return grads
