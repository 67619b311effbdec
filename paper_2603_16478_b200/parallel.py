"""Data-parallel batched rollouts.

Work is partitioned by independent rollouts - a batch of parameter candidates
or environments, candidate ``i`` on rank ``i % world`` - with no data-path
collective.  The only exchange is one all-reduce (sum) of the packed
parameter gradient per optimisation iteration, over NCCL (NVLink/NVSwitch)
when the tensors are on CUDA and gloo on CPU.
"""

from __future__ import annotations

import numpy as np

# order of the packed gradient vector (GradientReport fields, adjoint.py:70-90)
PACKED_FIELDS = ("loss", "dL_dE", "dL_dnu", "dL_dmu_friction", "dL_dstiffness")


def shard(n_items, rank, world):
    """Indices of the rollouts this rank owns (round robin)."""
    return list(range(rank, n_items, world))


def pack_gradients(grads, loss, device="cpu", extra=None):
    """[loss, dL/dE, dL/dnu, dL/dmu, dL/dstiffness, extra...] as float64."""
    import torch
    vals = [float(loss), float(grads.dL_dE), float(grads.dL_dnu),
            float(grads.dL_dmu_friction), float(grads.dL_dstiffness)]
    if extra is not None:
        vals.extend(np.asarray(extra, dtype=np.float64).ravel().tolist())
    return torch.tensor(vals, dtype=torch.float64, device=device)


def unpack_gradients(vec):
    v = vec.detach().cpu().numpy()
    out = dict(zip(PACKED_FIELDS, v[:len(PACKED_FIELDS)].tolist()))
    out["extra"] = v[len(PACKED_FIELDS):]
    return out


def allreduce_gradients(vec, world=None):
    """Sum the packed gradient across ranks (in place).  No-op when not
    distributed."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return vec
    if world is not None and world <= 1:
        return vec
    dist.all_reduce(vec, op=dist.ReduceOp.SUM)
    return vec


def batched_loss_and_grad(problems_x, problem, rank, world, device="cpu"):
    """Evaluate rollout_loss(with_grad) for this rank's share of candidate
    parameter vectors and all-reduce the summed [loss, grad...] vector."""
    from . import ident
    import torch
    names = problem.names()
    total = torch.zeros(1 + len(names), dtype=torch.float64, device=device)
    for i in shard(len(problems_x), rank, world):
        L, g = ident.rollout_loss(problem, problems_x[i], with_grad=True)
        total += torch.tensor([L] + list(np.atleast_1d(g)), dtype=torch.float64, device=device)
    return allreduce_gradients(total, world)
