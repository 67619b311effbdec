"""Data-parallel batched rollouts.

Work is partitioned by independent rollouts - a batch of parameter candidates
or environments, candidate ``i`` on rank ``i % world`` - with no data-path
collective.  The only exchange is one all-reduce (sum) of the packed
parameter gradient per optimisation iteration, over NCCL (NVLink/NVSwitch)
when the tensors are on CUDA and gloo on CPU.

The packed vector is one contiguous float64 tensor: the scalar fields
(``SCALAR_FIELDS``) followed by the optional per-element / per-binding /
per-step blocks of ``GradientReport`` (adjoint.py:70-90) a caller asks for
(``BLOCK_FIELDS``): dL/dw[E], dL/dE_b[B], dL/dd_b[B,3], the shared controls
dL/dfext[T,3V] and the initial-state gradients dL/dq_bar, dL/dv_bar[3V].
Device-resident inputs (torch CUDA tensors) are packed on the device, so the
all-reduce never touches the host.
"""

from __future__ import annotations

import numpy as np

# order of the packed gradient vector (GradientReport fields, adjoint.py:70-90)
SCALAR_FIELDS = ("loss", "dL_dE", "dL_dnu", "dL_dmu_friction", "dL_dstiffness")
PACKED_FIELDS = SCALAR_FIELDS
BLOCK_FIELDS = ("dL_dw", "dL_dEb", "dL_ddb", "dL_dfext", "dL_dqbar", "dL_dvbar")


def shard(n_items, rank, world):
    """Indices of the rollouts this rank owns (round robin)."""
    return list(range(rank, n_items, world))


class PackLayout:
    """Names, shapes and offsets of the packed gradient vector."""

    def __init__(self, blocks=(), extra=0):
        self.entries = [(f, ()) for f in SCALAR_FIELDS]
        self.blocks = tuple(blocks)
        for b in self.blocks:
            name, shape = b if isinstance(b, tuple) else (b, None)
            if name not in BLOCK_FIELDS:
                raise ValueError(f"unknown gradient block {name!r}")
            self.entries.append((name, shape))
        self.extra = int(extra)

    def bind(self, grads):
        """Fix the block shapes from a GradientReport (first pack)."""
        out = []
        for name, shape in self.entries:
            if shape is None:
                shape = tuple(_as_array_shape(getattr(grads, name)))
            out.append((name, shape))
        self.entries = out
        return self

    @property
    def size(self):
        return sum(int(np.prod(s)) if s else 1 for _, s in self.entries) + self.extra


def _as_array_shape(v):
    if isinstance(v, list):
        if not v:
            return (0,)
        return (len(v),) + tuple(_shape(v[0]))
    return _shape(v)


def _shape(v):
    return tuple(v.shape) if hasattr(v, "shape") else np.shape(v)


def _flat(torch, v, device):
    if isinstance(v, list):
        if not v:
            return torch.zeros(0, dtype=torch.float64, device=device)
        return torch.cat([_flat(torch, x, device) for x in v])
    if isinstance(v, torch.Tensor):
        return v.reshape(-1).to(device=device, dtype=torch.float64)
    return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64).reshape(-1)).to(device)


def pack_gradients(grads, loss, device="cpu", extra=None, blocks=(), layout=None):
    """[loss, dL/dE, dL/dnu, dL/dmu, dL/dstiffness, blocks..., extra...] as
    one float64 tensor on `device`.  `blocks` names GradientReport array
    fields to append (BLOCK_FIELDS); a field may hold a torch CUDA tensor (then
    nothing goes through the host).  Returns the tensor, or (tensor, layout)
    when `layout` is True."""
    import torch
    lay = PackLayout(blocks, 0 if extra is None else np.size(extra)).bind(grads) if blocks else None
    scal = torch.tensor([float(loss), float(grads.dL_dE), float(grads.dL_dnu),
                         float(grads.dL_dmu_friction), float(grads.dL_dstiffness)],
                        dtype=torch.float64, device=device)
    parts = [scal]
    for name in (lay.blocks if lay else ()):
        name = name[0] if isinstance(name, tuple) else name
        parts.append(_flat(torch, getattr(grads, name), device))
    if extra is not None:
        parts.append(_flat(torch, np.asarray(extra, dtype=np.float64), device))
    vec = torch.cat(parts) if len(parts) > 1 else scal
    if layout:
        return vec, (lay or PackLayout((), 0 if extra is None else np.size(extra)))
    return vec


def unpack_gradients(vec, layout=None):
    """Inverse of pack_gradients: scalars as floats, blocks as NumPy arrays
    of their shapes, the rest as `extra`."""
    v = vec.detach().cpu().numpy() if hasattr(vec, "detach") else np.asarray(vec)
    lay = layout or PackLayout()
    out, o = {}, 0
    for name, shape in lay.entries:
        if not shape:
            out[name] = float(v[o])
            o += 1
        else:
            n = int(np.prod(shape))
            out[name] = v[o:o + n].reshape(shape)
            o += n
    out["extra"] = v[o:]
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
