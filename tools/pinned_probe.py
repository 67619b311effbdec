"""Probe: are the public API's output arrays page-locked on this box, and
what H2D / D2H bandwidth do they get (vs pageable NumPy)?"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_16478_b200 import _pinned  # noqa: E402

n = 3 * 175616
d = torch.empty(n, dtype=torch.float64, device="cuda")
for label, mk in (("pinned", lambda: _pinned.pool().empty(n)), ("numpy", lambda: np.empty(n))):
    a = mk()
    a[:] = 1.0
    t = torch.from_numpy(a)
    print(label, "is_pinned", t.is_pinned(), type(a.base).__name__)
    for _ in range(3):
        d.copy_(t, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        d.copy_(t, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for _ in range(20):
        t.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(label, f"H2D {20 * 8 * n / (t1 - t0) / 1e9:.1f} GB/s, D2H {20 * 8 * n / (t2 - t1) / 1e9:.1f} GB/s")
t0 = time.perf_counter()
for _ in range(100):
    _pinned.empty(n)
print(f"_pinned.empty {1e6 * (time.perf_counter() - t0) / 100:.1f} us/call")
