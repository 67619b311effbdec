"""Host logic of the page-locked output pool (paper_2603_16478_b200/_pinned.py):
carved arrays never overlap while alive, a slab is reused only after every
array (and every view of one) carved from it is gone.  The slab allocation is
replaced by ordinary memory here (pinning needs a GPU)."""
import gc

import numpy as np


class _FakeSlab:
    def __init__(self, nbytes):
        self.buf = np.empty(nbytes, dtype=np.uint8)
        self.size = nbytes
        self.off = 0
        self.live = 0


def test_pool_carves_disjoint_and_recycles(monkeypatch):
    from paper_2603_16478_b200 import _pinned
    monkeypatch.setattr(_pinned, "_Slab", _FakeSlab)
    p = _pinned.PinnedPool(slab_bytes=8 << 20)
    n = (1 << 20) // 8 + 5                      # > 1 MB: pooled
    a, b = p.empty(n), p.empty(n)
    a[:] = 1.0
    b[:] = 2.0
    assert np.all(a == 1.0) and np.all(b == 2.0)
    slab = p.cur
    assert slab.live == 2
    view = a[::7]                               # a view keeps a's memory alive
    del a
    gc.collect()
    assert slab.live == 2 and np.all(view == 1.0)
    del view, b
    gc.collect()
    assert slab.live == 0
    c = p.empty(n)                              # slab reused from offset 0
    assert p.cur is slab and slab.live == 1
    c[:] = 3.0
    small = p.empty(10)                         # small requests: plain NumPy
    assert small.base is None
