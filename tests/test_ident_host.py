"""Identification driver around the hot path (ident.py:100-316): problem
validation and the convergence metrics on CPU; gradient descent with
analytic vs (concurrent) finite-difference gradients on the GPU."""
import numpy as np
import pytest


def test_opt_problem_validation():
    from paper_2603_16478_b200 import ident
    sc = ident.scene_library()["bar_neohookean"]
    with pytest.raises(ValueError):
        ident.OptProblem(sc, 3, "E", 1e4, learning_rate=0.0, iterations=1)
    with pytest.raises(ValueError):
        ident.OptProblem(sc, 3, "Young", 1e4, learning_rate=1.0, iterations=1)
    with pytest.raises(ValueError):
        ident.OptProblem(sc, 3, " , ", 1e4, learning_rate=1.0, iterations=1)
    p = ident.OptProblem(sc, 3, "E, nu", np.array([1e4, 0.3]), learning_rate=1.0, iterations=1)
    assert p.names() == ["E", "nu"] and not p.scalar
    with pytest.raises(ValueError):
        ident.resolve_target(p)                      # neither target given


def test_metrics_known_trace():
    from paper_2603_16478_b200 import ident
    tr = ident.OptTrace(losses=[10.0, 6.0, 4.0, 2.0, 1.0], params=[0] * 5, grads_ana=[1.0, 2.0, 1.0, 1.0, 1.0],
                        grads_fd=[1.1, None, 1.0, None, 0.5])
    m = ident.metrics(tr)
    # total drop 9: 50% (4.5) first reached at i=2 (drop 6), 90% (8.1) at i=4 (drop 9)
    assert m.t50 == pytest.approx(2 / 4) and m.t90 == pytest.approx(4 / 4)
    assert m.auc_e == pytest.approx(np.mean([(10 - 1) / 9, (6 - 1) / 9]))
    assert m.auc_m == pytest.approx(np.mean([(4 - 1) / 9, (2 - 1) / 9]))
    assert m.auc_l == pytest.approx(0.0)
    assert m.mre_e == pytest.approx(abs(1.0 - 1.1) / (1.1 + 1e-12))
    assert m.mre_m == pytest.approx(0.0)
    assert m.mre_l == pytest.approx(abs(1.0 - 0.5) / (0.5 + 1e-12))
    assert not m.degenerate
    assert ident.metrics(ident.OptTrace(losses=[1.0])).degenerate
    assert ident.metrics(ident.OptTrace(losses=[1.0, 2.0])).degenerate
    with pytest.raises(ValueError):
        ident.metrics(ident.OptTrace())


@pytest.mark.gpu
def test_optimize_with_fd_check():
    """Three gradient steps on E of the NH bar (scene_library) with an FD
    check every iteration: the loss decreases, analytic and concurrent
    central-difference gradients agree, and the concurrent FD equals the
    sequential one bitwise."""
    from paper_2603_16478_b200 import forward as fw, ident
    sc = ident.scene_library()["bar_neohookean"]
    cfg = fw.ForwardConfig(tol=1e-12)
    prob = ident.OptProblem(sc, 4, "E", 4.0e4, learning_rate=1.0, iterations=3, target_value=5.0e4,
                            fd_every=1, fd_eta=1e-4)
    L0, g0 = ident.rollout_loss(prob, 4.0e4, with_grad=True, cfg=cfg)
    prob.learning_rate = 0.2 * 4.0e4 / abs(g0)        # a stable step for this problem
    tr = ident.optimize(prob, cfg=cfg)
    assert not tr.diverged and len(tr.losses) == 3
    assert tr.losses[-1] < tr.losses[0]
    for ga, gf in zip(tr.grads_ana, tr.grads_fd):
        assert abs(ga - gf) <= 1e-4 * abs(gf)
    seq = ident.fd_gradient(prob, 4.0e4, cfg=cfg, workers=1)
    par = ident.fd_gradient(prob, 4.0e4, cfg=cfg, workers=2)
    assert seq == par
    m = ident.metrics(tr)
    assert m.mre_e <= 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("var,x0,target", [("E", 4.0e4, 5.0e4), ("E,nu", [4.0e4, 0.3], [5.0e4, 0.32])])
def test_batched_fd_on_pooled_device_scenes(var, x0, target):
    """finite differences evaluated on pooled device scenes
    (FDPool: parameters pushed in place with dp_scene_set_materials, no scene
    copy or device-scene rebuild per rollout) equal, bitwise, the per-rollout
    rebuild path (the reference's rollout_loss), for one and several
    variables; a reused pool gives the same result again."""
    from paper_2603_16478_b200 import forward as fw, ident
    sc = ident.scene_library()["bar_neohookean"]
    cfg = fw.ForwardConfig(tol=1e-12)
    prob = ident.OptProblem(sc, 4, var, np.asarray(x0), learning_rate=1.0, iterations=1,
                            target_value=np.asarray(target))
    ref = ident.fd_gradient(prob, x0, cfg=cfg, workers=2, batched=False)
    pool = ident.FDPool(prob, 2)
    got = ident.fd_gradient(prob, x0, cfg=cfg, workers=2, pool=pool)
    again = ident.fd_gradient(prob, x0, cfg=cfg, workers=2, pool=pool)
    assert np.array_equal(np.atleast_1d(got), np.atleast_1d(ref))
    assert np.array_equal(np.atleast_1d(again), np.atleast_1d(ref))
    _, g_ana = ident.rollout_loss(prob, x0, with_grad=True, cfg=cfg)
    assert np.allclose(np.atleast_1d(g_ana), np.atleast_1d(got), rtol=1e-4)
