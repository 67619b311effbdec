"""Trajectory output of a rollout (the reference CLI's ``simulate`` artefacts,
cli.py:81-110): ``trajectory.csv`` (schema "trajectory v1": step, vid, x, y,
z with 17 significant digits) and ``forward.json`` (per-step iterations,
convergence, final residual, contact count).

B200 side: ``TrajectoryRecorder`` streams the states of a device-resident
rollout (``forward_step(..., device_io=...)``) to page-locked host memory on a
second CUDA stream while the next steps compute: one event per step orders
the copy after the step's kernels, the copy engine does the transfer, and the
rollout never waits for it (the host buffers are one pinned slab allocated
up front, so no per-step cudaHostAlloc).  ``simulate`` is the public-API
equivalent of the reference's ``cmd_simulate``.
"""

from __future__ import annotations

import json
import os

import numpy as np

from . import forward as fw

CSV_HEADER = "# schema: trajectory v1\n"


def write_trajectory_csv(path, positions):
    """positions: sequence (or array [T+1, V, 3]) of per-step vertex
    positions, step 0 = the initial state.  Byte-identical to the reference
    writer (cli.py:92-100: csv rows `step, vid, x, y, z`, f"{c:.17g}")."""
    with open(path, "w", newline="") as f:
        f.write(CSV_HEADER)
        f.write("step,vid,x,y,z\r\n")
        for s, pos in enumerate(positions):
            p = np.asarray(pos, dtype=np.float64).reshape(-1, 3)
            rows = [f"{s},{v},{x:.17g},{y:.17g},{z:.17g}\r\n" for v, (x, y, z) in enumerate(p.tolist())]
            f.write("".join(rows))


def forward_summaries(reports):
    """forward.json rows (cli.py:101-106) from ForwardReports."""
    return [{"step": i + 1, "iterations": r.iterations, "converged": r.converged,
             "final_residual": r.residual_history[-1] if r.residual_history else None,
             "n_contacts": r.n_contacts} for i, r in enumerate(reports)]


class TrajectoryRecorder:
    """Asynchronous device-to-host recording of a device-resident rollout.

    rec = TrajectoryRecorder(n_dofs, n_steps, device)
    rec.record(k, q_tensor)        # after forward_step k wrote q_tensor
    positions = rec.finish()       # [n_steps + 1, V, 3] NumPy (waits once)
    """

    def __init__(self, n_dofs, n_steps, device="cuda:0", stride=1):
        import torch
        self.torch = torch
        self.stride = max(1, int(stride))
        self.n_slots = n_steps // self.stride + 1
        self.host = torch.empty((self.n_slots, n_dofs), dtype=torch.float64, pin_memory=True)
        self.copy_stream = torch.cuda.Stream(device=device)
        self.filled = []

    def record(self, k, q, producer_stream=None):
        """Enqueue the copy of step k's positions (device tensor) once the
        producer stream (default: the current stream) has written them."""
        if k % self.stride:
            return
        torch = self.torch
        ev = torch.cuda.Event()
        ev.record(producer_stream or torch.cuda.current_stream())
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(ev)
            self.host[k // self.stride].copy_(q, non_blocking=True)
            q.record_stream(self.copy_stream)
        self.filled.append(k // self.stride)

    def finish(self):
        """Wait for the copies once; positions [slots, V, 3] (NumPy view of
        the pinned slab)."""
        self.copy_stream.synchronize()
        n = max(self.filled) + 1 if self.filled else 0
        return self.host[:n].numpy().reshape(n, -1, 3)


def simulate(scene, n_steps, out_dir, cfg=None, state0=None):
    """Public-API equivalent of the reference's ``simulate`` command
    (cli.py:81-110): rollout, trajectory.csv, forward.json.  Raises the
    reference's RuntimeError on a non-converged step (forward.py:261-264).
    Returns (states, caches)."""
    os.makedirs(out_dir, exist_ok=True)
    states, caches = fw.rollout(scene, state0 or scene.rest_state(), n_steps, cfg=cfg)
    write_trajectory_csv(os.path.join(out_dir, "trajectory.csv"), [st.q for st in states])
    with open(os.path.join(out_dir, "forward.json"), "w") as f:
        json.dump(forward_summaries([c.report for c in caches]), f, indent=1)
    return states, caches


__all__ = ["write_trajectory_csv", "forward_summaries", "TrajectoryRecorder", "simulate"]
