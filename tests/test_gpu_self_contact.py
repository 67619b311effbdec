"""Self-contact (no reference implementation): the GPU
spatial-hash detection against the brute-force CPU oracle
(oracle/self_contact_oracle.py) - pair sets and distances bit-exact - and
the coupled Newton step / adjoint with self contacts: no interpenetration,
and analytic gradients against central finite differences (one step from a
fixed start state, where the frozen contact triangles do not depend on the
parameters)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2603_16478_b200 as p
    from paper_2603_16478_b200 import _lib
    _lib.lib()
    return p


def _query(scene, q_bar, q_pred):
    from paper_2603_16478_b200 import _lib, core
    sm = core.assemble_system_matrix(scene)
    dev = sm.dev
    dev.sync(scene, force=True)
    V = scene.n_verts
    tri = np.empty(V, np.int32)
    d2 = np.empty(V)
    nrm = np.empty(3 * V)
    off = np.empty(V)
    _lib.check(dev.lib.dp_self_contact_query(dev.handle, _lib.ptr(_lib.f64(q_bar)), _lib.ptr(_lib.f64(q_pred)),
                                             _lib.PTR_HOST, _lib.ptr(tri), _lib.ptr(d2), _lib.ptr(nrm),
                                             _lib.ptr(off)))
    return tri, d2, nrm.reshape(-1, 3), off


def _folded_sheet(n=12, gap=6e-4, seed=0):
    """A cloth sheet whose right half is folded over its left half, gap
    apart, with seeded jitter (q_bar), and a perturbed current state q."""
    from paper_2603_16478_b200 import core, ident
    edge = 0.1 / n
    v, t = ident.horizontal_sheet(n, n, edge)
    xc = 0.5 * n * edge
    qb = v.copy()
    right = qb[:, 0] > xc + 1e-12
    qb[right, 0] = 2 * xc - qb[right, 0]
    qb[right, 2] = gap + 0.2 * edge * (qb[right, 0] - xc) ** 2 / edge
    rng = np.random.default_rng(seed)
    qb += rng.uniform(-1e-4, 1e-4, qb.shape)
    q = qb + rng.uniform(-2e-4, 2e-4, qb.shape)
    sc = core.Scene(v, t, core.lumped_masses(v, t, 0.3), [core.MaterialParams("arap", stiffness=50.0)] * len(t),
                    self_contact=True, self_mu=0.2)
    return sc, qb.reshape(-1), q.reshape(-1)


def _stacked_cubes(n=3, gap=5e-4, seed=1):
    """Two tet cubes in one mesh, the upper gap above the lower."""
    from paper_2603_16478_b200 import core, ident
    size = 0.02 / n
    v1, t1 = ident.box_tet_mesh(n, n, n, size=size, origin=(0.0, 0.0, 5e-4))
    v2, t2 = ident.box_tet_mesh(n, n, n, size=size, origin=(0.002, 0.001, 5e-4 + 0.02 + gap))
    v = np.concatenate([v1, v2])
    t = np.concatenate([t1, t2 + len(v1)])
    sc = core.Scene(v, t, core.lumped_masses(v, t, 1000.0),
                    [core.MaterialParams("neohookean", E=2e4, nu=0.3)] * len(t),
                    colliders=[core.HalfSpace([0, 0, 1], 0.0, mu=0.0)], eps_fb=1e-7,
                    self_contact=True, self_mu=0.0)
    rng = np.random.default_rng(seed)
    q = v.reshape(-1) + rng.uniform(-1e-4, 1e-4, 3 * len(v))
    return sc, v.reshape(-1).copy(), q


@pytest.mark.parametrize("make", [_folded_sheet, _stacked_cubes], ids=["folded-sheet", "stacked-cubes"])
def test_self_candidates_bit_exact_vs_bruteforce(pkg, make):
    """Per-vertex candidate triangle, its distance^2 and the oriented plane:
    GPU spatial hash vs all-pairs brute force, bitwise."""
    import self_contact_oracle as SO
    scene, qb, q = make()
    tri, d2, nrm, off = _query(scene, qb, q)
    otri, od2, onrm, ooff = SO.self_candidates(qb, q, scene.elements, scene.contact_activation)
    assert (otri >= 0).sum() > 10                      # the configuration has candidates
    assert np.array_equal(tri, otri)
    assert np.array_equal(d2, od2)
    m = otri >= 0
    assert np.array_equal(nrm[m], onrm[m])
    assert np.array_equal(off[m], ooff[m])


def test_stacked_cubes_step_no_interpenetration_and_fd_gradient(pkg):
    """The upper cube falls onto the lower one (its predicted motion in one
    step is larger than the activation distance): self contacts (collider
    index = n_colliders) appear, the step converges, the self-contact vertex
    set equals the oracle's at the converged point, no vertex ends behind its
    contact plane, and dL/dE of the step matches central differences (from
    a fixed start state the frozen planes do not depend on E)."""
    import self_contact_oracle as SO
    from paper_2603_16478_b200 import adjoint as aj, core, forward as fw
    scene, q0, _ = _stacked_cubes(gap=4e-4)
    scene.eps_fb = 1e-9
    st0 = scene.rest_state()
    st0.v[2::3] = -0.05
    cfg = fw.ForwardConfig(tol=1e-11)
    sm = core.assemble_system_matrix(scene)
    st, rep = fw.forward_step(scene, st0, sm, cfg)
    assert rep.converged
    cps = rep.cache.contacts
    ncol = len(scene.colliders)
    got = np.array([c.vertex for c in cps if c.collider == ncol])
    assert got.size > 5
    q_hat = rep.cache.q_hat
    tri, _, nrm, off = SO.self_candidates(q0, q_hat, scene.elements, scene.contact_activation)
    act_v, gap = SO.active_self_contacts(tri, nrm, off, rep.cache.q_new, scene.contact_activation)
    assert np.array_equal(got, act_v)
    assert np.all(gap[tri >= 0] > 0.0)

    target = st.q + 1e-4

    def loss(E):
        sc = scene.copy()
        for m in sc.materials:
            m.E = E
        s1, r1 = fw.forward_step(sc, st0, core.assemble_system_matrix(sc), cfg)
        assert r1.converged
        return float(np.sum((s1.q - target) ** 2))

    g = aj.backprop_rollout([rep.cache], target)
    E0, eta = 2e4, 2e4 * 1e-3
    fd = (loss(E0 + eta) - loss(E0 - eta)) / (2 * eta)
    assert abs(g.dL_dE - fd) <= 1e-3 * abs(fd)


def test_c2_fold_converges_with_self_contact(pkg):
    """The bench's C2 fold (3,200-triangle ARAP sheet folded over its centre
    line in 120 steps, bench.py CONFIGS['c2fold']): every step converges, the
    folded halves end in hundreds of self contacts, and at the final state no
    vertex lies behind its self-contact plane (planes from the oracle's
    brute-force candidates at the last step's q_bar)."""
    import sys
    import os
    import self_contact_oracle as SO
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2603_16478_b200 import core, forward as fw
    scene = bench.make_scene("c2fold")
    sm = core.assemble_system_matrix(scene)
    cfg = fw.ForwardConfig(tol=bench.CONFIGS["c2fold"]["tol"])
    st = scene.rest_state()
    rep = None
    for k in range(bench.CONFIGS["c2fold"]["steps"]):
        bench.move_fingers(scene, k)
        st_prev = st
        st, rep = fw.forward_step(scene, st, sm, cfg)
        assert rep.converged, k
    ncol = len(scene.colliders)
    n_self = sum(1 for c in rep.cache.contacts if c.collider == ncol)
    assert n_self > 100
    tri, _, nrm, off = SO.self_candidates(st_prev.q, rep.cache.q_hat, scene.elements, scene.contact_activation)
    _, gap = SO.active_self_contacts(tri, nrm, off, st.q, scene.contact_activation)
    assert np.all(gap[tri >= 0] > 0.0)
