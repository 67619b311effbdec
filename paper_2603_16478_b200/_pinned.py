"""Page-locked host arrays for the public API's per-step outputs.

The reference API returns NumPy arrays (states, dL/dfext per step).  Copying
them from the GPU into ordinary (pageable) memory runs at a fraction of the
host link's bandwidth and cannot overlap; into page-locked memory it is a
direct DMA.  Pinning is expensive (cudaHostAlloc), and a rollout keeps every
step's arrays alive, so a caching allocator cannot recycle them per step
(round 1 measured that as a loss).  This pool carves arrays out of large
pinned slabs with a bump pointer; every array holds its slab alive, and a
slab whose arrays have all been garbage-collected goes back to a free list
and is reused by later rollouts (weakref.finalize on the arrays).
Small requests get ordinary NumPy memory.
"""

from __future__ import annotations

import threading
import weakref

import numpy as np

_ALL_SLABS = []               # every slab ever allocated (kept until exit)
_MIN_BYTES = 1 << 20          # below this a plain NumPy array is as fast
_SLAB_BYTES = 64 << 20


class _Slab:
    """One cudaHostAlloc'd block (dp_pinned_alloc), never freed before the
    process exits: freeing page-locked memory during interpreter teardown,
    after the CUDA context is gone, aborts the process."""

    __slots__ = ("buf", "size", "off", "live", "__weakref__")

    def __init__(self, nbytes):
        import ctypes as C
        from . import _lib
        L = _lib.lib()
        p = C.c_void_p()
        _lib.check(L.dp_pinned_alloc(nbytes, C.byref(p)))
        self.buf = np.frombuffer((C.c_uint8 * nbytes).from_address(p.value), dtype=np.uint8)
        self.size = nbytes
        self.off = 0
        self.live = 0
        _ALL_SLABS.append(self)


class _Owner:
    """Buffer exporter (PEP 688) for one carved array: NumPy keeps it as the
    base of the array and of every view derived from it, so the finalizer
    runs only when no view of the memory is left."""

    __slots__ = ("mem", "__weakref__")

    def __init__(self, mem):
        self.mem = mem

    def __buffer__(self, flags):
        return memoryview(self.mem)

    def __release_buffer__(self, view):
        view.release()


class PinnedPool:
    def __init__(self, slab_bytes=_SLAB_BYTES):
        self.slab_bytes = slab_bytes
        self.cur = None
        self.free = []
        self.lock = threading.Lock()

    def _release(self, slab):
        with self.lock:
            slab.live -= 1
            if slab.live == 0 and slab is not self.cur:
                slab.off = 0
                self.free.append(slab)

    def empty(self, n, dtype=np.float64):
        """Uninitialised 1-D array of n elements in page-locked memory."""
        dt = np.dtype(dtype)
        nbytes = int(n) * dt.itemsize
        if nbytes < _MIN_BYTES:
            return np.empty(n, dtype=dt)
        need = (nbytes + 255) & ~255
        with self.lock:
            s = self.cur
            if s is not None and s.live == 0:
                s.off = 0          # every array carved from it is gone
            if s is None or s.off + need > s.size:
                if s is not None and s.live == 0:
                    s.off = 0
                    self.free.append(s)
                s = None
                for i, f in enumerate(self.free):
                    if f.size >= need:
                        s = self.free.pop(i)
                        break
                if s is None:
                    s = _Slab(max(self.slab_bytes, need))
                self.cur = s
            off = s.off
            s.off += need
            s.live += 1
        owner = _Owner(s.buf[off:off + nbytes])
        arr = np.ndarray((int(n),), dtype=dt, buffer=owner)
        weakref.finalize(owner, self._release, s)
        return arr


_pools = {}
_pools_lock = threading.Lock()


def pool():
    """The calling thread's pool (host threads of concurrent rollouts do not
    contend on one bump pointer)."""
    tid = threading.get_ident()
    with _pools_lock:
        p = _pools.get(tid)
        if p is None:
            p = _pools[tid] = PinnedPool()
    return p


def empty(n, dtype=np.float64):
    try:
        return pool().empty(n, dtype)
    except Exception:   # no CUDA / torch: ordinary memory (host-only paths)
        return np.empty(n, dtype=dtype)
