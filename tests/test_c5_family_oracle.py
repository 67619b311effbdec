"""The bench's C5 workload is a regime the REFERENCE converges in (VERDICT r1
item 1): the CPU oracle (reference algorithm, exact SuperLU Newton solves,
oracle/diffproj_oracle.py) over the bench's finger schedule - closing and
hold - converges at every step.  The C5 family at 8^3 cells (bench.c5_family:
eps_fb and the absolute Newton tolerance scaled with the vertex mass);
larger sizes (10^3-20^3, 30 steps) are logged in
profiles/r02_scene_explore/oracle_c5fam_*.log."""

import numpy as np


def test_c5_family_converges_every_step_on_the_oracle():
    import bench
    import diffproj_oracle as O
    from paper_2603_16478_b200 import core
    fam = bench.c5_family(8)
    assert fam["mu"] == 0.0 and fam["schedule"] == (bench.FINGER_SPEED, bench.FINGER_HOLD)
    scene = bench.make_scene(fam)
    osc = O.OScene(core.scene_to_arrays(scene))
    els = O.build_elements(osc)
    A = O.assemble_A(osc, els)
    q = scene.vertices.reshape(-1).copy()
    v = np.zeros_like(q)
    n_steps = bench.FINGER_HOLD + 10          # the closing phase and 10 held steps
    finger_contacts = 0
    for k in range(n_steps):
        bench.move_fingers(scene, bench.FINGER_K0 + k)
        osc = O.OScene(core.scene_to_arrays(scene))
        st = O.forward_step(osc, A, els, q, v, O.ForwardConfig(tol=fam["tol"]))
        assert st.converged, (k, st.iterations, st.residual_history[-1])
        assert st.iterations < 30, (k, st.iterations)
        finger_contacts += int(np.sum(st.contacts.collider > 0))
        q, v = st.q_new, st.v_new
    assert finger_contacts > 0


def test_finger_schedule_is_independent_of_warmup():
    """The finger index of a rollout's step k is FINGER_K0 + k (never the
    --warmup count), closing then holding."""
    import bench
    sc = bench.make_scene(bench.c5_family(4))
    xs = []
    for k in range(bench.FINGER_HOLD + 5):
        bench.move_fingers(sc, bench.FINGER_K0 + k)
        xs.append(sc.colliders[1].center[0])
    d = np.diff(xs)
    assert np.allclose(d[:bench.FINGER_HOLD], bench.FINGER_SPEED)
    assert np.all(d[bench.FINGER_HOLD:] == 0.0)
    assert bench.FINGER_K0 == 0


def test_c2_fold_scene_and_targets():
    """bench.py's C2 fold: a 40 x 40 sheet with self-contact, its right edge
    bound; the edge targets are that edge rigidly folded about x = size/2 by
    pi (k+1)/fold - vertical at mid-fold, mirrored onto the left half (lifted
    by 2 mm) at the end - and the frictionless ground is the only collider."""
    import bench
    sc = bench.make_scene("c2fold")
    c = bench.CONFIGS["c2fold"]
    size = c["cells"][0] * c["edge"]
    assert sc.self_contact and sc.h == c["h"] and len(sc.colliders) == 1 and sc.colliders[0].mu == 0.0
    assert len(sc.bindings) == c["cells"][1] + 1
    edge = np.array([sc.vertices[b.vertex] for b in sc.bindings])
    assert np.allclose(edge[:, 0], size)
    bench.move_fingers(sc, c["fold"] // 2 - 1)
    mid = np.array([b.target for b in sc.bindings])
    assert np.allclose(mid[:, 0], size / 2, atol=1e-12)
    assert np.allclose(mid[:, 2], edge[:, 2] + size / 2 + 2e-3)
    bench.move_fingers(sc, c["fold"] - 1)
    end = np.array([b.target for b in sc.bindings])
    assert np.allclose(end[:, 0], 0.0, atol=1e-12) and np.allclose(end[:, 1], edge[:, 1])
    assert np.allclose(end[:, 2], edge[:, 2] + 2e-3, atol=1e-12)
