"""Element projections (drop-in surface of diffproj.elasticity).

The per-element work (SVD with the reference conventions, ARAP/Neo-Hookean
projection, projection Jacobian with the within-block-commutation limits,
Lame sensitivities) runs in csrc/dp_kernels.cu, one thread per element.
``project_batch`` exposes it for unit-level parity checks against the
reference (elasticity.py:137-324); the scalar helpers below are host-side
parameter algebra (elasticity.py:327-346).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import rest_measure  # noqa: F401  (reference name)


def lame_from_young(E, nu):
    """mu = E / (2(1+nu)), lambda = E nu / ((1+nu)(1-2nu))."""
    if not -1.0 < nu < 0.5:
        raise ValueError("nu must lie in (-1, 0.5)")
    return E / (2.0 * (1.0 + nu)), E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))


def lame_jacobian(E, nu):
    """d(mu, lambda) / d(E, nu) as a 2x2 array."""
    if not -1.0 < nu < 0.5:
        raise ValueError("nu must lie in (-1, 0.5)")
    a = 1.0 + nu
    b = 1.0 - 2.0 * nu
    den = a * b
    return np.array([[1.0 / (2.0 * a), -E / (2.0 * a * a)],
                     [nu / den, E * (den - nu * (b - 2.0 * a)) / (den * den)]])


def element_weight(material, vol):
    if material.model == "neohookean":
        mu, _ = lame_from_young(material.E, material.nu)
        return 2.0 * mu * vol
    return material.stiffness * vol


def project_batch(F, model, mu=None, lam=None, tau_rel=1e-6):
    """Project a batch of deformation gradients on the GPU.

    F: (n,3,3) or (n,3,2); model: "arap"/"neohookean" or per-item codes.
    Returns dict(sigma, theta, W, P, dPdF, dP_dmu, dP_dlam, status) with
    dPdF in the column-stacked vec basis of the reference (9x9 / 6x6)."""
    L = _lib.lib()
    F = np.asarray(F, dtype=np.float64)
    n, _, d = F.shape
    if isinstance(model, str):
        model = np.full(n, 1 if model == "neohookean" else 0, np.int32)
    model = _lib.i32(model)
    mu = _lib.f64(np.broadcast_to(0.0 if mu is None else mu, (n,)))
    lam = _lib.f64(np.broadcast_to(0.0 if lam is None else lam, (n,)))
    Fc = _lib.f64(F)
    out = dict(sigma=np.zeros((n, d)), theta=np.zeros((n, d)), W=np.zeros((n, d, d)),
               P=np.zeros((n, 3, d)), dPdF=np.zeros((n, 3 * d, 3 * d)),
               dP_dmu=np.zeros((n, 3, d)), dP_dlam=np.zeros((n, 3, d)),
               status=np.zeros(n, np.int32))
    _lib.check(L.dp_project_batch(n, d, _lib.ptr(Fc), _lib.ptr(model), _lib.ptr(mu),
                                  _lib.ptr(lam), tau_rel, _lib.ptr(out["sigma"]),
                                  _lib.ptr(out["theta"]), _lib.ptr(out["W"]), _lib.ptr(out["P"]),
                                  _lib.ptr(out["dPdF"]), _lib.ptr(out["dP_dmu"]),
                                  _lib.ptr(out["dP_dlam"]), _lib.ptr(out["status"])))
    return out
