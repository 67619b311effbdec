"""Multi-rank host logic of the data-parallel rollouts on CPU (gloo, world 2):
round-robin sharding of rollouts and the one all-reduce of the packed
parameter gradient per optimisation iteration."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_16478_b200.adjoint import GradientReport
    from paper_2603_16478_b200.parallel import allreduce_gradients, pack_gradients, shard, unpack_gradients
    mine = shard(7, rank, world)
    g = GradientReport(dL_dE=0.0, dL_dnu=0.0)
    loss = 0.0
    for i in mine:              # fake per-rollout gradients: rollout i contributes i+1
        g.dL_dE += i + 1.0
        g.dL_dnu += 0.5 * (i + 1.0)
        g.dL_dmu_friction += 2.0
        loss += 10.0 * i
    v = pack_gradients(g, loss, extra=[rank + 1.0])
    allreduce_gradients(v, world)
    q.put((rank, mine, unpack_gradients(v)))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_partitions_all_rollouts():
    from paper_2603_16478_b200.parallel import shard
    for world in (1, 2, 3, 8):
        got = sorted(i for r in range(world) for i in shard(13, r, world))
        assert got == list(range(13))


def test_gloo_world2_allreduce_of_packed_gradient():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == [0, 2, 4, 6] and res[1][1] == [1, 3, 5]
    for _, _, out in res:
        assert out["dL_dE"] == pytest.approx(sum(range(1, 8)))
        assert out["dL_dnu"] == pytest.approx(0.5 * sum(range(1, 8)))
        assert out["dL_dmu_friction"] == pytest.approx(14.0)
        assert out["loss"] == pytest.approx(10.0 * sum(range(7)))
        assert np.allclose(out["extra"], [3.0])


def test_allreduce_noop_without_process_group():
    from paper_2603_16478_b200.parallel import allreduce_gradients
    v = torch.tensor([1.0, 2.0], dtype=torch.float64)
    assert torch.equal(allreduce_gradients(v), v)


def _fake_report(i, E=5, B=2, T=3, n=6):
    """Deterministic per-rollout GradientReport with every array block."""
    from paper_2603_16478_b200.adjoint import GradientReport
    r = np.random.default_rng(100 + i)
    return GradientReport(dL_dqbar=r.standard_normal(n), dL_dvbar=r.standard_normal(n),
                          dL_dfext=[r.standard_normal(n) for _ in range(T)],
                          dL_dmu_friction=float(r.standard_normal()), dL_dEb=r.standard_normal(B),
                          dL_ddb=r.standard_normal((B, 3)), dL_dw=r.standard_normal(E),
                          dL_dstiffness=float(r.standard_normal()), dL_dE=float(r.standard_normal()),
                          dL_dnu=float(r.standard_normal()))


BLOCKS = ("dL_dw", "dL_dEb", "dL_ddb", "dL_dfext", "dL_dqbar", "dL_dvbar")


def _worker_blocks(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_16478_b200.parallel import allreduce_gradients, pack_gradients, shard, unpack_gradients
    tot = lay = None
    for i in shard(5, rank, world):
        v, lay = pack_gradients(_fake_report(i), float(i), blocks=BLOCKS, layout=True)
        tot = v if tot is None else tot + v
    allreduce_gradients(tot, world)
    q.put((rank, unpack_gradients(tot, lay)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_allreduce_of_full_packed_gradient():
    """the packed vector carries dL/dw, dL/dE_b, dL/dd_b,
    the shared controls dL/dfext and the state gradients; the all-reduced
    blocks equal the sum over all rollouts of every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_blocks, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    reps = [_fake_report(i) for i in range(5)]
    for _, out in res:
        assert out["loss"] == pytest.approx(sum(range(5)))
        assert out["dL_dE"] == pytest.approx(sum(r.dL_dE for r in reps))
        for name in BLOCKS:
            ref = sum(np.asarray(getattr(r, name)) for r in reps)
            assert out[name].shape == np.asarray(ref).shape, name
            assert np.allclose(out[name], ref, rtol=1e-14, atol=1e-14), name


def test_pack_roundtrip_and_layout():
    from paper_2603_16478_b200.parallel import PackLayout, pack_gradients, unpack_gradients
    g = _fake_report(0)
    v, lay = pack_gradients(g, 2.5, blocks=BLOCKS, extra=[7.0, 8.0], layout=True)
    assert v.numel() == lay.size == 5 + 5 + 2 + 6 + 3 * 6 + 6 + 6 + 2
    out = unpack_gradients(v, lay)
    assert out["loss"] == 2.5
    assert np.array_equal(out["dL_dfext"], np.array(g.dL_dfext))
    assert np.array_equal(out["dL_ddb"], g.dL_ddb)
    assert np.array_equal(out["extra"], [7.0, 8.0])
    with pytest.raises(ValueError):
        PackLayout(("not_a_field",))
