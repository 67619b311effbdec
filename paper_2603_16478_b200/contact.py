"""Vertex-vs-collider contact (drop-in surface of diffproj.contact).

Detection, condensation and the per-contact Jacobian blocks run on the GPU
(csrc/dp_contact.cu); this module exposes the reference's record type
``ContactPoint`` (contact.py:58-99) and batch entry points mirroring
``detect_contacts`` (:115-136), ``solve_multipliers`` (:139-165),
``contact_block`` (:212-248) and ``contact_residual`` (:168-183).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib

TAU_FALLBACK = 1e-9


def fb_smooth(x, y, eps2):
    """x + y - sqrt(x^2 + y^2 + eps2)  (contact.py:28-32)."""
    if eps2 <= 0:
        raise ValueError("eps2 must be positive")
    return x + y - np.sqrt(x * x + y * y + eps2)


def fb_grad(x, y, eps2):
    if eps2 <= 0:
        raise ValueError("eps2 must be positive")
    root = np.sqrt(x * x + y * y + eps2)
    return 1.0 - x / root, 1.0 - y / root


@dataclass
class ContactBlock:
    Kc_local: np.ndarray
    k_mu: np.ndarray


@dataclass
class ContactPoint:
    """One contact in its frame (rows n, t1, t2); fields as the reference."""

    vertex: int
    frame: np.ndarray
    d_n: float
    mu: float
    eps2: float
    d_f: np.ndarray = field(default_factory=lambda: np.zeros(2))
    lam: np.ndarray = field(default_factory=lambda: np.zeros(3))
    delta: np.ndarray = field(default_factory=lambda: np.zeros(3))
    s_signed: float = 0.0
    cone_capped: bool = False
    collider: int = -1

    @property
    def dofs(self):
        return 3 * int(self.vertex) + np.arange(3)

    def gaps(self, q, q_bar):
        x = q[self.dofs]
        return float(self.frame[0] @ x) - self.d_n, \
            self.frame[1:] @ (x - q_bar[self.dofs]) - self.d_f

    def apply_J(self, x):
        return self.frame @ x[self.dofs]

    def scatter_Jt(self, y, out):
        out[self.dofs] += self.frame.T @ y
        return out


def contacts_from_arrays(a, eps2):
    return [ContactPoint(vertex=int(a["vertex"][k]), frame=a["frame"][k].copy(),
                         d_n=float(a["d_n"][k]), mu=float(a["mu"][k]), eps2=eps2,
                         lam=a["lam"][k].copy(), delta=a["delta"][k].copy(),
                         s_signed=float(a["s_signed"][k]), cone_capped=bool(a["capped"][k]),
                         collider=int(a["collider"][k]))
            for k in range(a["vertex"].shape[0])]


def detect_contacts(scene, q, q_bar=None, sysmat=None):
    """GPU detection with the reference's arithmetic (bit-exact sets)."""
    from . import core
    if sysmat is None:
        sysmat = core.assemble_system_matrix(scene)
    dev = sysmat.dev
    dev.sync(scene)
    qd = _lib.f64(q)
    cap = max(1, scene.n_verts * max(1, len(scene.colliders)))
    n = C.c_int32()
    vtx = np.empty(cap, np.int32)
    col = np.empty(cap, np.int32)
    frame = np.empty((cap, 3, 3))
    dn = np.empty(cap)
    _lib.check(dev.lib.dp_detect_contacts(dev.handle, _lib.ptr(qd), _lib.PTR_HOST, cap, C.byref(n),
                                          _lib.ptr(vtx), _lib.ptr(col), _lib.ptr(frame), _lib.ptr(dn)))
    k = n.value
    mus = np.array([scene.colliders[j].mu for j in col[:k]]) if k else np.zeros(0)
    return [ContactPoint(vertex=int(vtx[i]), frame=frame[i].copy(), d_n=float(dn[i]),
                         mu=float(mus[i]), eps2=scene.eps_fb, collider=int(col[i]))
            for i in range(k)]


def contact_batch(frame, d_n, mu, eps2, x, x_bar):
    """Batched solve_multipliers + contact_block + contact_residual on the
    GPU.  Returns dict of arrays (lam, delta, s_signed, capped, Kc, k_mu,
    residual, status)."""
    L = _lib.lib()
    frame = _lib.f64(frame).reshape(-1, 3, 3)
    n = frame.shape[0]
    out = dict(lam=np.zeros((n, 3)), delta=np.zeros((n, 3)), s_signed=np.zeros(n),
               capped=np.zeros(n, np.int32), Kc=np.zeros((n, 3, 3)), k_mu=np.zeros((n, 3)),
               residual=np.zeros((n, 3)), status=np.zeros(n, np.int32))
    args = [_lib.f64(np.broadcast_to(a, (n,) + np.shape(a)[1:] if np.ndim(a) else (n,)))
            for a in (d_n, mu, eps2)]
    xv = _lib.f64(x).reshape(n, 3)
    xb = _lib.f64(x_bar).reshape(n, 3)
    _lib.check(L.dp_contact_batch(n, _lib.ptr(frame), _lib.ptr(args[0]), _lib.ptr(args[1]),
                                  _lib.ptr(args[2]), _lib.ptr(xv), _lib.ptr(xb),
                                  _lib.ptr(out["lam"]), _lib.ptr(out["delta"]),
                                  _lib.ptr(out["s_signed"]), _lib.ptr(out["capped"]),
                                  _lib.ptr(out["Kc"]), _lib.ptr(out["k_mu"]),
                                  _lib.ptr(out["residual"]), _lib.ptr(out["status"])))
    return out


def solve_multipliers(cp, q, q_bar, tau=TAU_FALLBACK):
    """In-place condensation of one ContactPoint (contact.py:139-165)."""
    i = cp.dofs
    r = contact_batch(cp.frame[None], [cp.d_n], [cp.mu], [cp.eps2], q[i][None], q_bar[i][None])
    if r["status"][0]:
        raise ValueError("contact multiplier solve requires delta_n > 0")
    cp.lam = r["lam"][0]
    cp.delta = r["delta"][0]
    cp.s_signed = float(r["s_signed"][0])
    cp.cone_capped = bool(r["capped"][0])
    return cp


def contact_block(cp, rot=None, tau=TAU_FALLBACK):
    """Kc_local and k_mu of a solved contact (contact.py:212-248)."""
    eye = np.eye(3)
    r = contact_batch(eye[None], [0.0], [cp.mu], [cp.eps2], cp.delta[None], np.zeros((1, 3)))
    return ContactBlock(Kc_local=r["Kc"][0], k_mu=r["k_mu"][0])


def contact_residual(cp, q=None, q_bar=None):
    """Smoothed complementarity rows at the cached state (contact.py:168-183)."""
    dn, df = cp.delta[0], cp.delta[1:]
    if q is not None:
        dn, df = cp.gaps(q, q_bar)
    lam_n, lam_f = cp.lam[0], cp.lam[1:]
    nf = float(np.linalg.norm(df))
    nl = float(np.linalg.norm(lam_f))
    align = nl * df + nf * lam_f
    return np.array([fb_smooth(dn, lam_n, cp.eps2), fb_smooth(nf, cp.mu * lam_n - nl, cp.eps2),
                     float(np.linalg.norm(align))])
