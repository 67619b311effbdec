"""N>1 data-parallel path with REAL rollouts: two ranks
(gloo, both on cuda:0 - this box has one GPU; never a measurement) each run
their round-robin share of C3-family E candidates (a 12x3x3-cell NH beam on
a frictional ground), pack the full GradientReport (scalars + dL/dw, dL/dE_b,
dL/dd_b, dL/dfext[T], dL/dq_bar, dL/dv_bar) and all-reduce it once.  The
reduced vector must equal, bitwise, the sum of the same packed vectors
computed by a single process in the same order."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_CAND = 4
BLOCKS = ("dL_dw", "dL_dEb", "dL_ddb", "dL_dfext", "dL_dqbar", "dL_dvbar")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _candidate_vector(i):
    """Packed gradient of rollout candidate i (E = 1e4 (1 + 0.05 i))."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    from paper_2603_16478_b200 import adjoint as aj, forward as fw
    from paper_2603_16478_b200.parallel import pack_gradients
    c = dict(bench.CONFIGS["c3"], cells=(12, 3, 3))
    scene = bench.make_scene(c, E=1e4 * (1 + 0.05 * i))
    states, caches = fw.rollout(scene, scene.rest_state(), 4, cfg=fw.ForwardConfig(tol=c["tol"]))
    target = states[0].q + 1e-3
    g = aj.backprop_rollout(caches, target)
    loss = float(np.sum((states[-1].q - target) ** 2))
    return pack_gradients(g, loss, "cpu", blocks=BLOCKS, layout=True)


def _rank(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    from paper_2603_16478_b200.parallel import allreduce_gradients, shard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tot = None
    for i in shard(N_CAND, rank, world):
        v, _ = _candidate_vector(i)
        tot = v if tot is None else tot + v
    allreduce_gradients(tot, world)
    q.put((rank, tot.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_allreduce_equals_single_process_sum():
    import torch.multiprocessing as mp
    from paper_2603_16478_b200.parallel import unpack_gradients
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    vecs, lay = [], None
    for i in range(N_CAND):
        v, lay = _candidate_vector(i)
        vecs.append(v.numpy())
    ref = (vecs[0] + vecs[2]) + (vecs[1] + vecs[3])     # rank 0 owns 0, 2; rank 1 owns 1, 3
    assert np.array_equal(res[0], res[1])
    assert np.array_equal(res[0], ref)
    out = unpack_gradients(ref, lay)
    assert out["dL_dfext"].shape[0] == 4 and np.abs(out["dL_dfext"]).max() > 0
    assert out["dL_dw"].shape == (12 * 3 * 3 * 6,)
    assert np.abs(out["dL_dqbar"]).max() > 0 and out["dL_dE"] != 0.0
