"""Probe: per-step wall time of forward_step through host NumPy buffers vs
device tensors on the C5 scene (where does the e2e gap come from?)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_16478_b200 import _lib, core, forward as fw  # noqa: E402

scene = bench.make_scene("c5")
cfg = fw.ForwardConfig(tol=bench.CONFIGS["c5"]["tol"])
sm = core.assemble_system_matrix(scene)
n = scene.ndof
K = 12
orig = _lib.check


def run(host):
    st = scene.rest_state()
    q = torch.zeros((K + 1, n), dtype=torch.float64, device="cuda")
    v = torch.zeros_like(q)
    q[0] = torch.from_numpy(st.q)
    ts = []
    for k in range(K):
        bench.move_fingers(scene, bench.FINGER_K0 + k)
        t0 = time.perf_counter()
        if host:
            st, rep = fw.forward_step(scene, st, sm, cfg)
        else:
            _, rep = fw.forward_step(scene, None, sm, cfg, device_io=dict(q_bar=q[k], v_bar=v[k], q_out=q[k + 1], v_out=v[k + 1]))
        ts.append(1e3 * (time.perf_counter() - t0))
    return ts


for rep_ in range(2):
    d = run(False)
    h = run(True)
    print("device", [round(x, 2) for x in d])
    print("host  ", [round(x, 2) for x in h])
    print("diff  ", [round(b - a, 2) for a, b in zip(d, h)])
# timing of the C call alone in host mode
import ctypes as C  # noqa: E402
st = scene.rest_state()
L = sm.dev.lib
calls = []
real = L.dp_forward_step


def timed(*a):
    t0 = time.perf_counter()
    r = real(*a)
    calls.append(1e3 * (time.perf_counter() - t0))
    return r


L.dp_forward_step = timed
for k in range(K):
    bench.move_fingers(scene, bench.FINGER_K0 + k)
    t0 = time.perf_counter()
    st, rep = fw.forward_step(scene, st, sm, cfg)
    tot = 1e3 * (time.perf_counter() - t0)
    print(f"host step {k}: total {tot:.2f} ms, C call {calls[-1]:.2f} ms, python {tot - calls[-1]:.2f} ms")
