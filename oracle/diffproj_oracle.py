"""CPU oracle: a vectorised NumPy/SciPy restatement of the reference hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2603_16478_b200`` imports this
module.  It is used by ``tests/`` (as the parity checker for the CUDA path),
by ``__graft_entry__.smoke()`` (checker) and by ``bench.py`` (the timed CPU
baseline leg, ``cpu_baseline.kind == "port"``).

It restates, function by function, the algorithm of the reference package
``diffproj`` (arXiv 2603.16478, mounted read-only at ``/root/reference``),
batched over elements with NumPy instead of the reference's per-element
Python loops.  Each function cites the reference ``file:line`` it follows
(paths relative to ``/root/reference/pkg/src/diffproj``).

Parity pinning: ``tests/test_oracle_golden.py`` checks this module against
the golden vectors in ``tests/golden/*.npz`` that
``tests/golden/make_golden.py`` produced by running the reference itself
(per-element projections, per-contact blocks, whole rollouts and reverse
sweeps).

Scene format: a plain ``dict`` of arrays with the keys written by
``make_golden.scene_to_arrays`` (vertices, elements, masses, mat_model,
mat_E, mat_nu, mat_stiffness, gravity, h, eps_fb, contact_activation, fext,
bind_vertex, bind_target, bind_compliance, col_kind, col_vec, col_scalar,
col_mu).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

TAU_FALLBACK = 1e-9          # contact.py:25


# ---------------------------------------------------------------------------
# scene


class OScene:
    """Arrays of one scene (core.py:146-196 fields, flattened)."""

    def __init__(self, d):
        self.vertices = np.asarray(d["vertices"], float).reshape(-1, 3)
        self.elements = np.asarray(d["elements"], np.int64)
        if self.elements.size == 0:
            self.elements = self.elements.reshape(0, 4)
        self.masses = np.asarray(d["masses"], float)
        self.mat_model = np.asarray(d["mat_model"], np.int32)
        self.mat_E = np.asarray(d["mat_E"], float)
        self.mat_nu = np.asarray(d["mat_nu"], float)
        self.mat_stiffness = np.asarray(d["mat_stiffness"], float)
        self.gravity = np.asarray(d["gravity"], float)
        self.h = float(d["h"])
        self.eps_fb = float(d["eps_fb"])
        self.contact_activation = float(d["contact_activation"])
        fx = np.asarray(d.get("fext", np.zeros(0)), float).ravel()
        self.fext = fx if fx.size else None
        self.bind_vertex = np.asarray(d["bind_vertex"], np.int64)
        self.bind_target = np.asarray(d["bind_target"], float).reshape(-1, 3)
        self.bind_compliance = np.asarray(d["bind_compliance"], float)
        self.col_kind = np.asarray(d["col_kind"], np.int32)
        self.col_vec = np.asarray(d["col_vec"], float).reshape(-1, 3)
        self.col_scalar = np.asarray(d["col_scalar"], float)
        self.col_mu = np.asarray(d["col_mu"], float)

    @property
    def n_verts(self):
        return self.vertices.shape[0]

    @property
    def ndof(self):
        return 3 * self.n_verts

    def mass_vector(self):                      # core.py:186-188
        return np.repeat(self.masses, 3)

    def external_force(self):                   # core.py:190-196
        f = np.zeros(self.ndof) if self.fext is None else self.fext.copy()
        return f + self.mass_vector() * np.tile(self.gravity, self.n_verts)


# ---------------------------------------------------------------------------
# analytic colliders, evaluated with the reference's scalar arithmetic
# (core.py:110-112 HalfSpace, core.py:133-139 Sphere).  Kept per point so
# the rounding of ``n @ x`` is the reference's own (contact sets are
# compared bit-exactly).


def collider_gap_normal(sc, j, x):
    if sc.col_kind[j] == 0:
        n = sc.col_vec[j]
        return float(n @ x - sc.col_scalar[j]), n
    d = x - sc.col_vec[j]
    r = np.linalg.norm(d)
    if r < 1e-14:
        return -sc.col_scalar[j], np.array([0.0, 0.0, 1.0])
    return float(r - sc.col_scalar[j]), d / r


# ---------------------------------------------------------------------------
# element kinematics (elasticity.py:47-108)


def lame_from_young(E, nu):                    # elasticity.py:327-333
    E = np.asarray(E, float)
    nu = np.asarray(nu, float)
    return E / (2.0 * (1.0 + nu)), E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))


def lame_jacobian(E, nu):                      # elasticity.py:336-346
    den = (1.0 + nu) * (1.0 - 2.0 * nu)
    dden = (1.0 - 2.0 * nu) - 2.0 * (1.0 + nu)
    return np.array([[1.0 / (2.0 * (1.0 + nu)), -E / (2.0 * (1.0 + nu) ** 2)],
                     [nu / den, E * (den - nu * dden) / den ** 2]])


@dataclass
class Elements:
    """Batched Element records (elasticity.py:21-44)."""

    verts: np.ndarray    # (E, nv)
    dofs: np.ndarray     # (E, 3nv)
    G: np.ndarray        # (E, 3d, 3nv)
    vol: np.ndarray
    w: np.ndarray
    dim: int
    model: np.ndarray    # 0 arap / 1 neohookean
    mu: np.ndarray       # Lame mu (nh only)
    lam: np.ndarray


def _selector_kron(B):
    """Batched G = kron(B^T, I3) @ S_diff (elasticity.py:57-64, :86-87)."""
    ne, d, _ = B.shape
    nv = d + 1
    # F = sum_k x_k beta_k^T with beta_k = B[k-1, :], beta_0 = -sum_k beta_k
    beta = np.zeros((ne, nv, d))
    beta[:, 1:, :] = B
    beta[:, 0, :] = -B.sum(axis=1)
    G = np.zeros((ne, 3 * d, 3 * nv))
    eye = np.eye(3)
    for c in range(d):          # column c of F (column-stacked vec)
        for a in range(nv):
            G[:, 3 * c:3 * c + 3, 3 * a:3 * a + 3] = \
                beta[:, a, c][:, None, None] * eye
    return G


def build_elements(sc):
    """elasticity.build_elements (elasticity.py:74-108), batched."""
    el = sc.elements
    ne, nv = el.shape
    x = sc.vertices[el]
    if ne == 0:
        return Elements(el, np.zeros((0, 3 * nv), np.int64),
                        np.zeros((0, 9, 12)), np.zeros(0), np.zeros(0), 3,
                        np.zeros(0, np.int32), np.zeros(0), np.zeros(0))
    if nv == 4:
        dm = np.stack([x[:, 1] - x[:, 0], x[:, 2] - x[:, 0],
                       x[:, 3] - x[:, 0]], axis=2)
        vol = np.linalg.det(dm) / 6.0
        if np.any(vol <= 1e-14):
            raise ValueError(f"degenerate or inverted tet "
                             f"{int(np.nonzero(vol <= 1e-14)[0][0])}")
        B = np.linalg.inv(dm)
        dim = 3
    elif nv == 3:
        e1 = x[:, 1] - x[:, 0]
        e2 = x[:, 2] - x[:, 0]
        area = 0.5 * np.linalg.norm(np.cross(e1, e2), axis=1)
        if np.any(area <= 1e-14):
            raise ValueError("degenerate triangle")
        t1 = e1 / np.linalg.norm(e1, axis=1)[:, None]
        t2v = e2 - np.sum(e2 * t1, axis=1)[:, None] * t1
        t2 = t2v / np.linalg.norm(t2v, axis=1)[:, None]
        dm2 = np.zeros((ne, 2, 2))
        dm2[:, 0, 0] = np.sum(e1 * t1, axis=1)
        dm2[:, 0, 1] = np.sum(e2 * t1, axis=1)
        dm2[:, 1, 1] = np.sum(e2 * t2, axis=1)
        B = np.linalg.inv(dm2)
        vol = area
        dim = 2
    else:
        raise ValueError("elements must be tetrahedra or triangles")
    G = _selector_kron(B)
    dofs = (3 * el[:, :, None] + np.arange(3)).reshape(ne, -1)
    model = sc.mat_model.copy()
    mu, lam = lame_from_young(sc.mat_E, sc.mat_nu)
    w = np.where(model == 1, 2.0 * mu * vol, sc.mat_stiffness * vol)
    return Elements(el, dofs, G, vol, w, dim, model, mu, lam)


# ---------------------------------------------------------------------------
# SVD and projections (elasticity.py:137-306)


def svd_polar(F):
    """Batched svd_polar (elasticity.py:137-165).  Returns U, s, V and a
    per-element error code (0 ok, 1 non-finite, 2 inverted/rank-deficient)."""
    F = np.asarray(F, float)
    ne = F.shape[0]
    err = np.zeros(ne, np.int32)
    err[~np.all(np.isfinite(F.reshape(ne, -1)), axis=1)] = 1
    Fs = np.where(err[:, None, None] == 0, F, 0.0)
    if F.shape[1:] == (3, 3):
        det = np.linalg.det(Fs)
        err[(err == 0) & (det <= 0)] = 2
        Fs = np.where(err[:, None, None] == 0, Fs, np.eye(3))
        U, s, Vt = np.linalg.svd(Fs)
        V = np.swapaxes(Vt, 1, 2).copy()
        flip = np.linalg.det(U) < 0
        U[flip, :, 2] *= -1.0
        V[flip, :, 2] *= -1.0
        return U, s, V, err
    U, s, Vt = np.linalg.svd(Fs, full_matrices=False)
    V = np.swapaxes(Vt, 1, 2).copy()
    err[(err == 0) & (s[:, -1] <= 0)] = 2
    flip = np.linalg.det(V) < 0
    U[flip, :, 1] *= -1.0
    V[flip, :, 1] *= -1.0
    return U, s, V, err


def _nh_g(theta, sigma, mu, lam):               # elasticity.py:181-184
    logj = np.sum(np.log(theta), axis=1, keepdims=True)
    return 2.0 * mu[:, None] * (theta - sigma) \
        + mu[:, None] * (theta - 1.0 / theta) + lam[:, None] * logj / theta


def _nh_dg(theta, mu, lam):                     # elasticity.py:187-192
    logj = np.sum(np.log(theta), axis=1)
    d = 3.0 * mu[:, None] + (mu - lam * logj)[:, None] / theta ** 2
    J = lam[:, None, None] * (1.0 / theta)[:, :, None] * (1.0 / theta)[:, None, :]
    idx = np.arange(theta.shape[1])
    J[:, idx, idx] += d
    return J


class NHStall(RuntimeError):
    pass


def project_neohookean(sigma, mu, lam, tol=1e-11, max_iter=50):
    """Damped Newton for theta (elasticity.py:195-242), active-set batched.

    Returns theta, W, energy density."""
    ne, d = sigma.shape
    theta = sigma.copy()
    if ne == 0:
        return theta, np.zeros((0, d, d)), np.zeros(0)
    r = _nh_g(theta, sigma, mu, lam)
    thr = tol * np.maximum(1.0, mu)
    done = np.zeros(ne, bool)
    for _ in range(max_iter):
        rn = np.linalg.norm(r, axis=1)
        done |= rn <= thr
        act = np.nonzero(~done)[0]
        if act.size == 0:
            break
        step = np.linalg.solve(_nh_dg(theta[act], mu[act], lam[act]),
                               -r[act][:, :, None])[:, :, 0]
        t = np.ones(act.size)
        accepted = np.zeros(act.size, bool)
        for _ls in range(40):
            pend = np.nonzero(~accepted)[0]
            if pend.size == 0:
                break
            cand = theta[act[pend]] + t[pend, None] * step[pend]
            pos = np.all(cand > 0, axis=1)
            ok = np.zeros(pend.size, bool)
            if np.any(pos):
                pi = pend[pos]
                ei = act[pi]
                rc = _nh_g(cand[pos], sigma[ei], mu[ei], lam[ei])
                better = np.linalg.norm(rc, axis=1) < rn[ei]
                acc = pi[better]
                theta[act[acc]] = cand[pos][better]
                r[act[acc]] = rc[better]
                ok_idx = np.nonzero(pos)[0][better]
                ok[ok_idx] = True
            accepted[pend[ok]] = True
            t[pend[~ok]] *= 0.5
        if not np.all(accepted):
            raise NHStall("neo-hookean projection stalled")
    else:
        rn = np.linalg.norm(r, axis=1)
        if np.any(rn > thr):
            raise NHStall("neo-hookean projection did not converge")
    logj = np.sum(np.log(theta), axis=1)
    dinv = 1.0 / (3.0 * mu[:, None] + (mu - lam * logj)[:, None] / theta ** 2)
    u = 1.0 / theta
    du = dinv * u
    denom = 1.0 + lam * np.sum(u * du, axis=1)
    W = 2.0 * mu[:, None, None] * (
        dinv[:, :, None] * np.eye(d)
        - du[:, :, None] * du[:, None, :] * (lam / denom)[:, None, None])
    energy = 0.5 * mu * (np.sum(theta * theta, axis=1) - 2.0 * logj - d) \
        + 0.5 * lam * logj ** 2
    return theta, W, energy


def _vecF(X):
    """Column-stacked vec of a batch of matrices."""
    return np.swapaxes(X, 1, 2).reshape(X.shape[0], -1)


def proj_jacobian(U, s, V, theta, W, tau_rel=1e-6):
    """dP/dF in the singular basis with the B4 degenerate limits
    (elasticity.py:262-306), batched."""
    ne, d = s.shape
    tau = tau_rel * np.max(np.abs(s), axis=1)
    M = np.zeros((ne, d, d))
    N = np.zeros((ne, d, d))
    for i in range(d):
        for j in range(d):
            if i == j:
                continue
            si, sj, ti, tj = s[:, i], s[:, j], theta[:, i], theta[:, j]
            far = np.abs(si - sj) > tau
            den = np.where(far, si * si - sj * sj, 1.0)
            wd = 0.5 * (W[:, i, i] + W[:, j, j])
            ts = (ti + tj) / (si + sj)
            M[:, i, j] = np.where(far, (si * ti - sj * tj) / den,
                                  0.5 * (wd - W[:, i, j] + ts))
            N[:, i, j] = np.where(far, (sj * ti - si * tj) / den,
                                  0.5 * (wd - W[:, i, j] - ts))
    # inner = D W D^T + Diag(vec M) + Diag(vec N) T   (elasticity.py:245-300)
    inner = np.zeros((ne, d * d, d * d))
    for i in range(d):
        for j in range(d):
            inner[:, i * d + i, j * d + j] += W[:, i, j]
    vM = _vecF(M)
    vN = _vecF(N)
    idx = np.arange(d * d)
    inner[:, idx, idx] += vM
    # (Diag(vec N) T)[k, l] = vN[k] * T[k, l], T[j*d+i, i*d+j] = 1
    for i in range(d):
        for j in range(d):
            inner[:, j * d + i, i * d + j] += vN[:, j * d + i]
    VU = np.einsum("eab,ecd->eacbd", V, U).reshape(
        ne, V.shape[1] * U.shape[1], V.shape[2] * U.shape[2])
    J = VU @ inner @ np.swapaxes(VU, 1, 2)
    if U.shape[1:] == (3, 2):
        u3 = np.cross(U[:, :, 0], U[:, :, 1])
        oop = V @ ((theta / s)[:, :, None] * np.swapaxes(V, 1, 2))
        J = J + np.einsum("eab,ecd->eacbd", oop,
                          u3[:, :, None] * u3[:, None, :]).reshape(ne, 6, 6)
    return J, M, N


def dP_dlame(U, s, V, theta, mu, lam):          # elasticity.py:309-324
    logj = np.sum(np.log(theta), axis=1)
    Jg = _nh_dg(theta, mu, lam)
    dmu = np.linalg.solve(Jg, -(3.0 * theta - 2.0 * s - 1.0 / theta)[:, :, None])[:, :, 0]
    dlam = np.linalg.solve(Jg, -(logj[:, None] / theta)[:, :, None])[:, :, 0]
    Vt = np.swapaxes(V, 1, 2)
    return U @ (dmu[:, :, None] * Vt), U @ (dlam[:, :, None] * Vt)


@dataclass
class ElemState:
    """Batched ElementCache (elasticity.py:353-362)."""

    F: np.ndarray
    U: np.ndarray
    s: np.ndarray
    V: np.ndarray
    theta: np.ndarray
    W: np.ndarray
    P: np.ndarray
    p: np.ndarray        # vec(P)
    energy: np.ndarray
    J: np.ndarray | None = None


class ProjectionError(ValueError):
    pass


def project_elements(els, q, with_jacobian=True, tau_rel=1e-6):
    """project_element over all elements (elasticity.py:365-383).

    Raises ProjectionError (a ValueError) on non-finite/inverted F, NHStall
    (RuntimeError) on a stalled Neo-Hookean projection."""
    ne = els.G.shape[0]
    d = els.dim
    if ne == 0:
        z = np.zeros((0, 3, d))
        return ElemState(z, np.zeros((0, 3, d)), np.zeros((0, d)),
                         np.zeros((0, d, d)), np.zeros((0, d)),
                         np.zeros((0, d, d)), z, np.zeros((0, 3 * d)),
                         np.zeros(0), np.zeros((0, 3 * d, 3 * d)))
    qe = q[els.dofs]
    vecF = np.einsum("eij,ej->ei", els.G, qe)
    F = np.swapaxes(vecF.reshape(ne, d, 3), 1, 2) if ne else \
        np.zeros((0, 3, d))
    U, s, V, err = svd_polar(F)
    if np.any(err):
        raise ProjectionError("inverted element or non-finite F")
    theta = np.ones((ne, d))
    W = np.zeros((ne, d, d))
    energy = np.zeros(ne)
    nh = np.nonzero(els.model == 1)[0]
    if nh.size:
        th, Wn, en = project_neohookean(s[nh], els.mu[nh], els.lam[nh])
        theta[nh], W[nh], energy[nh] = th, Wn, en
    P = U @ (theta[:, :, None] * np.swapaxes(V, 1, 2))
    J = None
    if with_jacobian:
        J, _, _ = proj_jacobian(U, s, V, theta, W, tau_rel)
    return ElemState(F, U, s, V, theta, W, P, _vecF(P), energy, J)


# ---------------------------------------------------------------------------
# system matrix (core.py:339-389)


def assemble_A(sc, els):
    """A = M + h^2 sum w G^T G as scipy CSR (core.py:367-389)."""
    n = sc.ndof
    h2 = sc.h ** 2
    rows = [np.arange(n)]
    cols = [np.arange(n)]
    vals = [sc.mass_vector()]
    if els.G.shape[0]:
        blk = h2 * els.w[:, None, None] * (np.swapaxes(els.G, 1, 2) @ els.G)
        r = np.repeat(els.dofs[:, :, None], els.dofs.shape[1], axis=2)
        c = np.repeat(els.dofs[:, None, :], els.dofs.shape[1], axis=1)
        rows.append(r.ravel())
        cols.append(c.ravel())
        vals.append(blk.ravel())
    A = sp.csr_matrix((np.concatenate(vals),
                       (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n))
    A.sum_duplicates()
    A.sort_indices()
    return A


def predict(sc, q, v):                          # core.py:392-397
    return q + sc.h * v + sc.h ** 2 * (1.0 / sc.mass_vector()) \
        * sc.external_force()


# ---------------------------------------------------------------------------
# contacts (contact.py)


def fb_smooth(x, y, eps2):                       # contact.py:28-32
    return x + y - np.sqrt(x * x + y * y + eps2)


def tangent_basis(n):                            # contact.py:102-112
    axis = np.zeros(3)
    axis[int(np.argmin(np.abs(n)))] = 1.0
    t1 = axis - (axis @ n) * n
    t1 /= math.sqrt(t1 @ t1)
    t2 = np.array([n[1] * t1[2] - n[2] * t1[1],
                   n[2] * t1[0] - n[0] * t1[2],
                   n[0] * t1[1] - n[1] * t1[0]])
    return t1, t2


@dataclass
class Contacts:
    """Struct-of-arrays ContactPoint list (contact.py:58-99)."""

    vertex: np.ndarray
    collider: np.ndarray
    frame: np.ndarray        # (C,3,3) rows n,t1,t2
    d_n: np.ndarray
    mu: np.ndarray
    eps2: float
    lam: np.ndarray = None
    delta: np.ndarray = None
    s: np.ndarray = None
    capped: np.ndarray = None

    def __len__(self):
        return self.vertex.shape[0]


def detect_contacts(sc, q):
    """detect_contacts (contact.py:115-136): vertex-major, collider-minor."""
    vs, cs, frs, dns, mus = [], [], [], [], []
    nc = sc.col_kind.shape[0]
    if nc:
        act = sc.contact_activation
        X = q.reshape(-1, 3)
        # cheap conservative prefilter, exact test below in reference order
        cand = np.zeros(X.shape[0], bool)
        for j in range(nc):
            if sc.col_kind[j] == 0:
                g = X @ sc.col_vec[j] - sc.col_scalar[j]
            else:
                g = np.linalg.norm(X - sc.col_vec[j], axis=1) - sc.col_scalar[j]
            cand |= g <= act + 1e-9 * (1.0 + abs(act))
        for v in np.nonzero(cand)[0]:
            x = X[v]
            for j in range(nc):
                gap, n = collider_gap_normal(sc, j, x)
                if gap > act:
                    continue
                t1, t2 = tangent_basis(n)
                vs.append(v)
                cs.append(j)
                frs.append(np.vstack([n, t1, t2]))
                dns.append(float(n @ x) - gap)
                mus.append(sc.col_mu[j])
    C = len(vs)
    return Contacts(np.array(vs, np.int64), np.array(cs, np.int64),
                    np.array(frs).reshape(C, 3, 3), np.array(dns),
                    np.array(mus), sc.eps_fb,
                    np.zeros((C, 3)), np.zeros((C, 3)), np.zeros(C),
                    np.zeros(C, bool))


class PenetrationError(ValueError):
    pass


def solve_multipliers(ct, q, q_bar, tau=TAU_FALLBACK):
    """Closed-form condensation (contact.py:139-165), batched; in place."""
    C = len(ct)
    if C == 0:
        return ct
    eps_sq = 0.5 * ct.eps2
    x = q.reshape(-1, 3)[ct.vertex]
    xb = q_bar.reshape(-1, 3)[ct.vertex]
    dn = np.einsum("ci,ci->c", ct.frame[:, 0], x) - ct.d_n
    df = np.einsum("cki,ci->ck", ct.frame[:, 1:], x - xb)
    if np.any(dn <= 0):
        raise PenetrationError("contact multiplier solve requires delta_n > 0")
    lam_n = eps_sq / dn
    nf = np.sqrt(df[:, 0] * df[:, 0] + df[:, 1] * df[:, 1])
    nfg = np.maximum(nf, tau)
    s = ct.mu * lam_n - eps_sq / nfg
    capped = s < -ct.mu * lam_n
    s = np.where(capped, -ct.mu * lam_n, s)
    lam_f = -s[:, None] * (df / nfg[:, None])
    ct.lam = np.column_stack([lam_n, lam_f])
    ct.delta = np.column_stack([dn, df])
    ct.s = s
    ct.capped = capped
    return ct


def contact_residual(ct):                        # contact.py:168-183
    dn = ct.delta[:, 0]
    df = ct.delta[:, 1:]
    lam_n = ct.lam[:, 0]
    lf = ct.lam[:, 1:]
    nf = np.linalg.norm(df, axis=1)
    nl = np.linalg.norm(lf, axis=1)
    align = nl[:, None] * df + nf[:, None] * lf
    return np.column_stack([fb_smooth(dn, lam_n, ct.eps2),
                            fb_smooth(nf, ct.mu * lam_n - nl, ct.eps2),
                            np.linalg.norm(align, axis=1)])


def contact_blocks(ct, tau=TAU_FALLBACK):
    """build_R + contact_block (contact.py:186-248), batched.

    Returns Kc_local (C,3,3) and k_mu (C,3)."""
    C = len(ct)
    lam_n = ct.lam[:, 0]
    dn = ct.delta[:, 0]
    df = ct.delta[:, 1:]
    lf = ct.lam[:, 1:]
    nf = np.linalg.norm(df, axis=1)
    nl = np.linalg.norm(lf, axis=1)
    R = np.tile(np.eye(3), (C, 1, 1))
    use_d = nf > tau
    use_l = (~use_d) & (nl > tau)
    a = np.where(use_d, df[:, 0] / np.where(use_d, nf, 1.0),
                 lf[:, 0] / np.where(use_l, nl, 1.0))
    b = np.where(use_d, df[:, 1] / np.where(use_d, nf, 1.0),
                 lf[:, 1] / np.where(use_l, nl, 1.0))
    R[use_d, 1, 1], R[use_d, 1, 2] = a[use_d], b[use_d]
    R[use_d, 2, 1], R[use_d, 2, 2] = -b[use_d], a[use_d]
    R[use_l, 1, 1], R[use_l, 1, 2] = -a[use_l], -b[use_l]
    R[use_l, 2, 1], R[use_l, 2, 2] = b[use_l], -a[use_l]
    sign = np.where(ct.capped, -1.0, 1.0)
    s = ct.s
    Bm = np.zeros((C, 3, 3))
    Bm[:, 0, 0] = lam_n / dn
    big = nf >= tau
    nfs = np.where(big, nf, 1.0)
    a22 = np.where(ct.capped, 0.0, (ct.mu * lam_n - s) / nfs)
    ratio = nf / tau
    Bm[:, 1, 0] = np.where(big, -sign * ct.mu * lam_n / dn,
                           -sign * ct.mu * lam_n / dn * ratio)
    Bm[:, 1, 1] = np.where(big, a22, s / tau)
    Bm[:, 2, 2] = np.where(big, s / nfs, s / tau)
    kvec = np.zeros((C, 3))
    kvec[:, 1] = np.where(big, lam_n, lam_n * ratio)
    Rt = np.swapaxes(R, 1, 2)
    Kc = Rt @ Bm @ R
    kmu = sign[:, None] * np.einsum("cij,cj->ci", Rt, kvec)
    return Kc, kmu


# ---------------------------------------------------------------------------
# forward step (forward.py)


@dataclass
class ForwardConfig:                             # forward.py:29-34
    tol: float = 1e-9
    max_iter: int = 100
    max_line_search: int = 40
    pullback_margin: float = 1e-6


def pullback(sc, q, margin, q_bar=None):         # forward.py:63-83
    X = q.reshape(-1, 3)
    for j in range(sc.col_kind.shape[0]):
        for v in range(X.shape[0]):
            gap, n = collider_gap_normal(sc, j, X[v])
            if gap <= 0:
                target = margin
                if q_bar is not None:
                    gp, _ = collider_gap_normal(sc, j, q_bar[3 * v:3 * v + 3])
                    if gp > 0:
                        target = min(margin, gp)
                target = max(target, 1e-12)
                X[v] = X[v] + (target - gap) * n
    return q


def _gaps_all(sc, q):
    X = q.reshape(-1, 3)
    out = []
    for j in range(sc.col_kind.shape[0]):
        if sc.col_kind[j] == 0:
            out.append(X @ sc.col_vec[j] - sc.col_scalar[j])
        else:
            r = np.linalg.norm(X - sc.col_vec[j], axis=1)
            out.append(np.where(r < 1e-14, -sc.col_scalar[j],
                                r - sc.col_scalar[j]))
    return out


def any_penetration(sc, q):                      # forward.py:86-93
    return any(np.any(g <= 0) for g in _gaps_all(sc, q))


def scatter_elements(els, vals, n):
    """out[dofs] += vals (E, 3nv)."""
    out = np.zeros(n)
    if vals.shape[0]:
        np.add.at(out, els.dofs.ravel(), vals.ravel())
    return out


def momentum_residual(sc, A, els, es, q, q_hat, ct):
    """forward.py:101-110 with elasticity.internal_force_and_rhs (:386-396)."""
    h2 = sc.h ** 2
    gp = scatter_elements(
        els, els.w[:, None] * np.einsum("eji,ej->ei", els.G, es.p), sc.ndof)
    b = sc.mass_vector() * q_hat + h2 * gp
    r = A @ q - b
    for i, v in enumerate(sc.bind_vertex):
        lam_b = -(q[3 * v:3 * v + 3] - sc.bind_target[i]) / sc.bind_compliance[i]
        r[3 * v:3 * v + 3] -= h2 * lam_b
    if len(ct):
        f = np.einsum("cji,cj->ci", ct.frame, -h2 * ct.lam)
        np.add.at(r.reshape(-1, 3), ct.vertex, f)
    return r


def newton_matrix(sc, A, els, es, ct, transpose_contacts=False):
    """A_hat = A - DeltaA + K_b + K_c (forward.py:113-149)."""
    h2 = sc.h ** 2
    n = sc.ndof
    rows, cols, vals = [], [], []
    if els.G.shape[0]:
        blk = -h2 * els.w[:, None, None] * (
            np.swapaxes(els.G, 1, 2) @ es.J @ els.G)
        k = els.dofs.shape[1]
        rows.append(np.repeat(els.dofs[:, :, None], k, axis=2).ravel())
        cols.append(np.repeat(els.dofs[:, None, :], k, axis=1).ravel())
        vals.append(blk.ravel())
    for i, v in enumerate(sc.bind_vertex):
        d = np.arange(3 * v, 3 * v + 3)
        rows.append(d)
        cols.append(d)
        vals.append(np.full(3, h2 / sc.bind_compliance[i]))
    if len(ct):
        Kc, _ = contact_blocks(ct)
        if transpose_contacts:
            Kc = np.swapaxes(Kc, 1, 2)
        gb = h2 * np.swapaxes(ct.frame, 1, 2) @ Kc @ ct.frame
        d = 3 * ct.vertex[:, None] + np.arange(3)
        rows.append(np.repeat(d[:, :, None], 3, axis=2).ravel())
        cols.append(np.repeat(d[:, None, :], 3, axis=1).ravel())
        vals.append(gb.ravel())
    if rows:
        D = sp.csr_matrix((np.concatenate(vals),
                           (np.concatenate(rows), np.concatenate(cols))),
                          shape=(n, n))
        return sp.csr_matrix(A + D)
    return sp.csr_matrix(A)


@dataclass
class StepResult:
    q_bar: np.ndarray
    v_bar: np.ndarray
    q_hat: np.ndarray
    q_new: np.ndarray
    v_new: np.ndarray
    es: ElemState
    contacts: Contacts
    residual_history: list = field(default_factory=list)
    converged: bool = False
    iterations: int = 0


def forward_step(sc, A, els, q0, v0, cfg=None):
    """forward_step (forward.py:174-248)."""
    cfg = cfg or ForwardConfig()
    q_bar = q0.copy()
    v_bar = v0.copy()
    q_hat = predict(sc, q_bar, v_bar)
    q = pullback(sc, q_hat.copy(), cfg.pullback_margin, q_bar)
    scale = max(1.0, float(np.max(np.abs(sc.mass_vector() * q_hat))))
    hist = []

    def evaluate(qc, ct, jac):
        es = project_elements(els, qc, jac)
        solve_multipliers(ct, qc, q_bar)
        return es, momentum_residual(sc, A, els, es, qc, q_hat, ct)

    dense = sc.ndof <= 300
    converged = False
    ct = es = None
    for _ in range(cfg.max_iter):
        ct = detect_contacts(sc, q)
        es, r = evaluate(q, ct, True)
        rmax = float(np.max(np.abs(r)))
        hist.append(rmax / scale)
        if hist[-1] <= cfg.tol:
            converged = True
            break
        Ah = newton_matrix(sc, A, els, es, ct)
        if dense:
            dq = np.linalg.solve(Ah.toarray(), -r)
        else:
            dq = spla.spsolve(sp.csc_matrix(Ah), -r)
        t = 1.0
        accepted = False
        for _ls in range(cfg.max_line_search):
            qt = q + t * dq
            if not any_penetration(sc, qt):
                try:
                    _, rt = evaluate(qt, ct, False)
                    if np.max(np.abs(rt)) < rmax:
                        q = qt
                        accepted = True
                        break
                except ValueError:
                    pass
            t *= 0.5
        if not accepted and not any_penetration(sc, q + t * dq):
            q = q + t * dq
    return StepResult(q_bar, v_bar, q_hat, q, (q - q_bar) / sc.h, es, ct,
                      hist, converged, len(hist))


def rollout(sc, q0, v0, n_steps, cfg=None, raise_on_failure=True):
    """rollout (forward.py:251-267)."""
    els = build_elements(sc)
    A = assemble_A(sc, els)
    steps = []
    q, v = q0.copy(), v0.copy()
    for k in range(n_steps):
        st = forward_step(sc, A, els, q, v, cfg)
        if raise_on_failure and not st.converged:
            raise RuntimeError(f"forward step {k} did not converge "
                               f"(residual {st.residual_history[-1]:.3e})")
        steps.append(st)
        q, v = st.q_new, st.v_new
    return els, A, steps


# ---------------------------------------------------------------------------
# Krylov solvers (linsolve.py:62-197)


def cg(apply, rhs, dinv, tol=1e-10, max_iter=2000):
    """Jacobi-PCG with a true residual per iteration (linsolve.py:62-105)."""
    nb = np.linalg.norm(rhs)
    x = np.zeros_like(rhs)
    if nb == 0:
        return x, True, [0.0]
    r = rhs.copy()
    z = dinv * r
    p = z.copy()
    rz = r @ z
    hist = []
    for _ in range(max_iter):
        rel = np.linalg.norm(rhs - apply(x)) / nb
        hist.append(rel)
        if rel <= tol:
            return x, True, hist
        ap = apply(p)
        pap = p @ ap
        if pap <= 0:
            raise RuntimeError("cg breakdown")
        al = rz / pap
        x = x + al * p
        r = r - al * ap
        z = dinv * r
        rzn = r @ z
        p = z + (rzn / rz) * p
        rz = rzn
    rel = np.linalg.norm(rhs - apply(x)) / nb
    hist.append(rel)
    return x, rel <= tol, hist


def gmres(apply, rhs, dinv, tol=1e-10, max_iter=2000, restart=50):
    """Left-preconditioned restarted GMRES (linsolve.py:108-197)."""
    n = rhs.shape[0]
    m = min(restart, n)
    nb = np.linalg.norm(rhs)
    x = np.zeros_like(rhs)
    hist = []
    if nb == 0:
        return x, True, [0.0]
    nMb = np.linalg.norm(dinv * rhs) or 1.0
    total = 0
    while total < max_iter:
        r = rhs - apply(x)
        rel = np.linalg.norm(r) / nb
        hist.append(rel)
        if rel <= tol:
            break
        start = rel
        z = dinv * r
        beta = np.linalg.norm(z)
        if beta == 0:
            break
        Vb = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        Vb[0] = z / beta
        used = 0
        for j in range(m):
            if total >= max_iter:
                break
            w = dinv * apply(Vb[j])
            for i in range(j + 1):
                H[i, j] = w @ Vb[i]
                w = w - H[i, j] * Vb[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] > 1e-300:
                Vb[j + 1] = w / H[j + 1, j]
            for i in range(j):
                tmp = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = tmp
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / den if den else 1.0
            sn[j] = H[j + 1, j] / den if den else 0.0
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            used = j + 1
            total += 1
            est = abs(g[j + 1]) / nMb
            hist.append(est)
            if est <= 0.1 * tol:
                break
        if used:
            y = sla.solve_triangular(H[:used, :used], g[:used])
            x = x + Vb[:used].T @ y
        rel = np.linalg.norm(rhs - apply(x)) / nb
        hist[-1] = rel
        if rel <= tol:
            break
        if rel >= start * (1.0 - 1e-12):
            break
    final = np.linalg.norm(rhs - apply(x)) / nb
    if hist[-1] != final:
        hist.append(final)
    return x, final <= tol, hist


# ---------------------------------------------------------------------------
# adjoint (adjoint.py)


@dataclass
class Grads:
    """GradientReport fields (adjoint.py:70-90)."""

    dL_dqbar: np.ndarray = None
    dL_dvbar: np.ndarray = None
    dL_dfext: list = field(default_factory=list)
    dL_dmu_friction: float = 0.0
    dL_dEb: np.ndarray = None
    dL_ddb: np.ndarray = None
    dL_dw: np.ndarray = None
    dL_dstiffness: float = 0.0
    dL_dE: float = 0.0
    dL_dnu: float = 0.0


def adjoint_solve(sc, A, els, st, rhs, tol=1e-10, max_iter=2000, restart=50, direct=False):
    """assemble_adjoint_operator + solve_adjoint (adjoint.py:93-139).

    direct=True (test infrastructure): solve A_hat^T z = rhs with SuperLU
    instead of the reference's Jacobi-preconditioned Krylov method, for
    operators where that method does not reach its tolerance (compressed
    cloth) - the solution, not the solver, is the parity target."""
    Ah = newton_matrix(sc, A, els, st.es, st.contacts)
    AhT = sp.csr_matrix(Ah.T)
    if direct:
        return spla.spsolve(sp.csc_matrix(AhT), rhs)
    d = Ah.diagonal()
    if np.any(np.abs(d) < 1e-300):
        raise ValueError("jacobi preconditioner requires nonzero diagonal")
    dinv = 1.0 / d
    symmetric = bool(np.all(st.contacts.mu == 0.0))
    if symmetric:
        z, ok, hist = cg(lambda x: Ah @ x, rhs, dinv, tol, max_iter)
    else:
        z, ok, hist = gmres(lambda x: AhT @ x, rhs, dinv, tol, max_iter,
                            restart)
    if not ok:
        raise RuntimeError("adjoint solve did not converge")
    return z


def backprop_step(sc, els, st, z, dL_dv, g):
    """backprop_step (adjoint.py:154-219), batched over elements."""
    h = sc.h
    h2 = h * h
    m = sc.mass_vector()
    ct = st.contacts
    dqbar = m * z - dL_dv / h
    if len(ct):
        Kc, kmu = contact_blocks(ct)
        zc = np.einsum("cij,cj->ci", ct.frame, z.reshape(-1, 3)[ct.vertex])
        t = np.einsum("cji,cj->ci", Kc, zc)          # Kc^T zc
        t[:, 0] = 0.0                                  # P_f = diag(0,1,1)
        add = h2 * np.einsum("cji,cj->ci", ct.frame, t)
        np.add.at(dqbar.reshape(-1, 3), ct.vertex, add)
        g.dL_dmu_friction += float(np.sum(-h2 * np.sum(kmu * zc, axis=1)))
    dvbar = h * (m * z)
    g.dL_dfext.append(h2 * z)
    q = st.q_new
    for i, v in enumerate(sc.bind_vertex):
        Eb = sc.bind_compliance[i]
        lam_b = -(q[3 * v:3 * v + 3] - sc.bind_target[i]) / Eb
        zb = z[3 * v:3 * v + 3]
        g.dL_dEb[i] += float(zb @ (-h2 * lam_b / Eb))
        g.dL_ddb[i] += h2 / Eb * zb
    ne = els.G.shape[0]
    if ne:
        gz = np.einsum("eij,ej->ei", els.G, z[els.dofs])
        gq = np.einsum("eij,ej->ei", els.G, q[els.dofs])
        base = np.sum(gz * (st.es.p - gq), axis=1)
        ar = els.model == 0
        g.dL_dw[ar] += h2 * base[ar]
        g.dL_dstiffness += float(np.sum(h2 * base[ar] * els.vol[ar]))
        nh = np.nonzero(els.model == 1)[0]
        if nh.size:
            es = st.es
            pmu, plam = dP_dlame(es.U[nh], es.s[nh], es.V[nh], es.theta[nh],
                                 els.mu[nh], els.lam[nh])
            dmu = np.sum(h2 * (2.0 * els.vol[nh] * base[nh]
                               + els.w[nh] * np.sum(gz[nh] * _vecF(pmu), 1)))
            dlam = np.sum(h2 * els.w[nh] * np.sum(gz[nh] * _vecF(plam), 1))
            if dmu or dlam:
                f = nh[0]
                Jl = lame_jacobian(sc.mat_E[f], sc.mat_nu[f])
                dE, dnu = Jl.T @ np.array([dmu, dlam])
                g.dL_dE += float(dE)
                g.dL_dnu += float(dnu)
    return g, dqbar, dvbar


def backprop_rollout(sc, els, A, steps, target=None, loss_fn=None,
                     tol=1e-10, direct=False):
    """backprop_rollout (adjoint.py:228-271) for a final-state loss
    (adjoint.py:222-225) or a callable loss."""
    n = sc.ndof
    T = len(steps)
    if T == 0:
        raise ValueError("empty rollout")
    g = Grads(dL_dEb=np.zeros(len(sc.bind_vertex)),
              dL_ddb=np.zeros((len(sc.bind_vertex), 3)),
              dL_dw=np.zeros(els.G.shape[0]))
    dq = np.zeros(n)
    dv = np.zeros(n)
    fx = []
    for k in range(T, 0, -1):
        st = steps[k - 1]
        if loss_fn is not None:
            gq, gv = loss_fn(k, st.q_new, (st.q_new - st.q_bar) / sc.h)
        elif k == T:
            gq, gv = 2.0 * (st.q_new - target), np.zeros(n)
        else:
            gq, gv = np.zeros(n), np.zeros(n)
        dq = dq + gq
        dv = dv + gv
        z = adjoint_solve(sc, A, els, st, dq + dv / sc.h, tol=tol, direct=direct)
        g.dL_dfext = []
        g, dq, dv = backprop_step(sc, els, st, z, dv, g)
        fx.append(g.dL_dfext[0])
    g.dL_dfext = list(reversed(fx))
    g.dL_dqbar = dq
    g.dL_dvbar = dv
    return g
