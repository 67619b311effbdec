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
