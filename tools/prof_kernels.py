"""Profile helper: the C5 bench's roofline kernels on a real operator (after
2 bench steps): one fine-level smoother sweep (dp_bench_smoother) and one
FP64 SpMV (dp_bench_spmv), bracketed by cudaProfilerStart/Stop so that
`ncu --profile-from-start off` captures exactly these launches."""
import sys, ctypes as C
sys.path.insert(0, '.')
import torch
import bench
from paper_2603_16478_b200 import core, forward as fw, _lib
sc = bench.make_scene("c5")
sm = core.assemble_system_matrix(sc)
st = sc.rest_state()
for k in range(2):
    bench.move_fingers(sc, k)
    st, rep = fw.forward_step(sc, st, sm, fw.ForwardConfig(tol=bench.CONFIGS["c5"]["tol"]))
n3 = 3 * sc.n_verts
dd = dict(device="cuda:0", dtype=torch.float64)
x, b, o = torch.randn(n3, **dd), torch.randn(n3, **dd), torch.empty(n3, **dd)
torch.cuda.synchronize()
ms = C.c_float()
L, h = sm.dev.lib, sm.dev.handle
torch.cuda.profiler.start()
_lib.check(L.dp_bench_smoother(h, _lib.ptr(x), _lib.ptr(b), _lib.ptr(o), 2, C.byref(ms)))
_lib.check(L.dp_bench_spmv(h, 1, _lib.ptr(x), _lib.ptr(o), 2, C.byref(ms)))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
