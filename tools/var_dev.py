"""Variance probe: device-only work (SpMV chains, no host syncs inside a
chunk) timed per chunk from process start."""
import ctypes as C, os, sys, time
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, '.')
import torch
import bench
from paper_2603_16478_b200 import core, forward as fw, _lib
torch.cuda.set_device(0)
sc = bench.make_scene("c5"); sm = core.assemble_system_matrix(sc)
st, rep = fw.forward_step(sc, sc.rest_state(), sm, fw.ForwardConfig(tol=1e-11))   # assembles val_fwd
L = sm.dev.lib
n3 = 3 * sc.n_verts
x = torch.randn(n3, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
ms = C.c_float()
t0 = time.perf_counter()
out = []
for rep in range(40):
    L.dp_bench_spmv(sm.dev.handle, 1, _lib.ptr(x), _lib.ptr(y), 300, C.byref(ms))
    out.append((round(time.perf_counter() - t0, 1), round(ms.value, 2)))
print(out)
