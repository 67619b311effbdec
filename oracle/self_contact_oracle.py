"""CPU oracle for self-contact detection.

TEST INFRASTRUCTURE ONLY (tests/ use it as the checker of the CUDA path).

The reference (arXiv 2603.16478 `diffproj`) has no self-contact
(/root/reference/SPEC.md: non-goal), so this is a brute-force restatement of
the rule the CUDA path implements (paper_2603_16478_b200/csrc/dp_contact.cu,
SelfContact in dp_internal.h): every vertex's q_bar position against every
surface triangle frozen at q_bar, skipping triangles with a vertex in the
vertex's 1-ring (vertices sharing an element, incl. itself); the candidate is
the triangle with the smallest closest-point distance^2 <= R^2, R =
activation + |q_hat - q_bar| (ties to the lower triangle index); its
half-space is the triangle's unit normal at q_bar turned to the side the
vertex was on at q_bar, active when the gap is <= activation.  Arithmetic mirrors the
CUDA code operation by operation (no FMA; dot products ((x0 y0 + x1 y1) +
x2 y2)), so pair sets and distances compare bit for bit: no broad phase here,
all V x T pairs.
"""

from __future__ import annotations

import numpy as np


def surface_triangles(elements):
    """Boundary faces of a tet mesh (faces of exactly one tet) or every
    triangle of a triangle mesh, in the CUDA path's order."""
    el = np.asarray(elements, dtype=np.int64)
    if el.shape[1] == 3:
        return el.astype(np.int32)
    faces = np.concatenate([el[:, [0, 1, 2]], el[:, [0, 1, 3]], el[:, [0, 2, 3]], el[:, [1, 2, 3]]])
    key = np.sort(faces, axis=1)
    _, inv, cnt = np.unique(key, axis=0, return_inverse=True, return_counts=True)
    return faces[cnt[inv.reshape(-1)] == 1].astype(np.int32)


def rings(n_verts, elements):
    """1-ring (incl. the vertex) of every vertex: vertices sharing an element."""
    r = [set([v]) for v in range(n_verts)]
    for e in np.asarray(elements, dtype=np.int64):
        for a in e:
            r[a].update(int(b) for b in e)
    return r


def _sdot(a, b):
    return (a[..., 0] * b[..., 0] + a[..., 1] * b[..., 1]) + a[..., 2] * b[..., 2]


def tri_dist2(p, a, b, c):
    """Squared distance point p -> triangle (a, b, c), broadcast over leading
    axes; the CUDA tri_dist2's case order and arithmetic."""
    ab, ac, ap = b - a, c - a, p - a
    d1, d2 = _sdot(ab, ap), _sdot(ac, ap)
    bp = p - b
    d3, d4 = _sdot(ab, bp), _sdot(ac, bp)
    vc = d1 * d4 - d3 * d2
    cp = p - c
    d5, d6 = _sdot(ab, cp), _sdot(ac, cp)
    vb = d5 * d2 - d1 * d6
    va = d3 * d6 - d5 * d4
    with np.errstate(divide="ignore", invalid="ignore"):
        q_ab = a + (d1 / (d1 - d3))[..., None] * ab
        q_ac = a + (d2 / (d2 - d6))[..., None] * ac
        q_bc = b + ((d4 - d3) / ((d4 - d3) + (d5 - d6)))[..., None] * (c - b)
        denom = 1.0 / (va + vb + vc)
        q_in = (a + ab * (vb * denom)[..., None]) + ac * (vc * denom)[..., None]
    c1 = (d1 <= 0.0) & (d2 <= 0.0)
    c2 = (d3 >= 0.0) & (d4 <= d3)
    c3 = (vc <= 0.0) & (d1 >= 0.0) & (d3 <= 0.0)
    c4 = (d6 >= 0.0) & (d5 <= d6)
    c5 = (vb <= 0.0) & (d2 >= 0.0) & (d6 <= 0.0)
    c6 = (va <= 0.0) & ((d4 - d3) >= 0.0) & ((d5 - d6) >= 0.0)
    q = np.where(c1[..., None], a,
        np.where(c2[..., None], b,
        np.where(c3[..., None], q_ab,
        np.where(c4[..., None], c,
        np.where(c5[..., None], q_ac,
        np.where(c6[..., None], q_bc, q_in))))))
    d = p - q
    return _sdot(d, d)


def tri_normals(qb, tris):
    """Unit normals at q_bar (cross((b-a), (c-a)) / |.|)."""
    P = qb.reshape(-1, 3)
    a, b, c = P[tris[:, 0]], P[tris[:, 1]], P[tris[:, 2]]
    e1, e2 = b - a, c - a
    n = np.stack([e1[:, 1] * e2[:, 2] - e1[:, 2] * e2[:, 1],
                  e1[:, 2] * e2[:, 0] - e1[:, 0] * e2[:, 2],
                  e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]], axis=1)
    ln = np.sqrt(_sdot(n, n))
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(ln[:, None] > 0.0, n / ln[:, None], 0.0)


def self_candidates(q_bar, q_pred, elements, act, tris=None):
    """Per vertex, once per step: the candidate triangle (nearest non-ring
    surface triangle to the q_bar position within R = act + |q_pred - q_bar|;
    -1 if none), its distance^2 at q_bar (-1), the oriented plane normal and
    offset (gap(x) = n . x - offset); the CUDA k_self_candidates."""
    Pb = np.asarray(q_bar, np.float64).reshape(-1, 3)
    Pp = np.asarray(q_pred, np.float64).reshape(-1, 3)
    V = Pb.shape[0]
    tris = surface_triangles(elements) if tris is None else np.asarray(tris, np.int32).reshape(-1, 3)
    ring = rings(V, elements)
    a, b, c = Pb[tris[:, 0]], Pb[tris[:, 1]], Pb[tris[:, 2]]
    d2 = tri_dist2(Pb[:, None, :], a[None], b[None], c[None])          # (V, T)
    dp = Pp - Pb
    R = act + np.sqrt(_sdot(dp, dp))
    lim = R * R
    excl = np.zeros(d2.shape, bool)
    for v in range(V):
        rv = ring[v]
        excl[v] = [(int(t0) in rv) or (int(t1) in rv) or (int(t2) in rv) for t0, t1, t2 in tris]
    d2m = np.where(excl | ~(d2 <= lim[:, None]), np.inf, d2)
    t = np.argmin(d2m, axis=1)                      # first minimum = lowest index on ties
    has = np.isfinite(d2m[np.arange(V), t])
    tri = np.where(has, t, -1)
    dist2 = np.where(has, d2m[np.arange(V), t], -1.0)
    tn = tri_normals(q_bar, tris)
    nrm = np.zeros((V, 3))
    off = np.zeros(V)
    for v in np.nonzero(has)[0]:
        m = tn[tri[v]]
        av = Pb[tris[tri[v], 0]]
        n = (-1.0 if _sdot(m, Pb[v] - av) < 0.0 else 1.0) * m
        nrm[v] = n
        off[v] = _sdot(n, av)
    return tri, dist2, nrm, off


def active_self_contacts(tri, nrm, off, q, act):
    """Vertices whose candidate plane gap at q is <= act (HalfSpace rule,
    contact.py:124-136) and those gaps."""
    P = np.asarray(q, np.float64).reshape(-1, 3)
    gap = _sdot(nrm, P) - off
    return np.nonzero((tri >= 0) & ~(gap > act))[0], gap
