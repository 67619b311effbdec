"""Full-size GPU checks through size-independent properties (the oracle is
too slow at these sizes): adjoint gradient vs central finite differences at
C3 scale, bitwise run-to-run determinism and bit-exact contact detection at
C5 (998,250 tets)."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _rollout(scene, steps, tol, sm=None):
    from paper_2603_16478_b200 import core, forward as fw
    sm = sm or core.assemble_system_matrix(scene)
    states, caches = fw.rollout(scene, scene.rest_state(), steps, sysmat=sm,
                                cfg=fw.ForwardConfig(tol=tol))
    return sm, states, caches


def test_c3_scale_dE_matches_finite_differences():
    import bench
    from paper_2603_16478_b200 import adjoint as aj, core
    n, steps, tol = 16, 3, 1e-12
    base = bench.make_scene(n, fingers=False, eps_fb=1e-7)
    _, states, caches = _rollout(base, steps, tol)
    target = states[0].q + 1e-3
    g = aj.backprop_rollout(caches, target)

    def loss(E):
        sc = bench.make_scene(n, fingers=False, eps_fb=1e-7)
        mat = core.MaterialParams("neohookean", E=E, nu=bench.NU)
        sc.materials = [mat] * len(sc.materials)
        _, st, _ = _rollout(sc, steps, tol)
        d = st[-1].q - target
        return float(d @ d)

    eta = 1.0
    fd = (loss(bench.E_YOUNG + eta) - loss(bench.E_YOUNG - eta)) / (2 * eta)
    assert abs(g.dL_dE - fd) <= 1e-4 * abs(fd), (g.dL_dE, fd)


def test_c5_determinism_and_bit_exact_detection():
    import bench
    import diffproj_oracle as O
    from paper_2603_16478_b200 import core, forward as fw
    scene = bench.make_scene(55, fingers=True)
    sm = core.assemble_system_matrix(scene)
    bench.move_fingers(scene, 0)
    s1, r1 = fw.forward_step(scene, scene.rest_state(), sm, fw.ForwardConfig())
    s2, r2 = fw.forward_step(scene, scene.rest_state(), sm, fw.ForwardConfig())
    assert r1.converged and r2.converged
    assert np.array_equal(s1.q, s2.q) and np.array_equal(s1.v, s2.v)   # no float atomics
    # the cached contact list is detect_contacts at the converged q, with
    # the reference's arithmetic
    osc = O.OScene(core.scene_to_arrays(scene))
    ref = O.detect_contacts(osc, s1.q)
    got = r1.cache.contacts
    assert len(got) == len(ref) > 3000
    assert np.array_equal([c.vertex for c in got], ref.vertex)
    assert np.array_equal([c.collider for c in got], ref.collider)
    assert np.array_equal(np.array([c.frame for c in got]), ref.frame)
    assert np.array_equal(np.array([c.d_n for c in got]), ref.d_n)


def test_concurrent_rollouts_match_sequential():
    """k rollouts on one GPU, one stream + host thread each (the batched
    identification mode of bench.py --config c3): bitwise equal to running
    them one after the other."""
    from concurrent.futures import ThreadPoolExecutor

    import bench
    from paper_2603_16478_b200 import adjoint as aj, core, forward as fw

    def job(E):
        sc = bench.make_scene(4, fingers=True, eps_fb=1e-6, E=E)
        sm = core.assemble_system_matrix(sc)
        st, caches = sc.rest_state(), []
        for k in range(3):
            bench.move_fingers(sc, k)
            st, rep = fw.forward_step(sc, st, sm, fw.ForwardConfig(tol=1e-10))
            caches.append(rep.cache)
        g = aj.backprop_rollout(caches, sc.rest_state().q + 1e-3)
        return st.q, g.dL_dE

    Es = [1e4, 1.2e4, 1.5e4, 2e4]
    seq = [job(E) for E in Es]
    with ThreadPoolExecutor(4) as ex:
        par = list(ex.map(job, Es))
    for (qa, ga), (qb, gb) in zip(seq, par):
        assert np.array_equal(qa, qb)
        assert ga == gb
