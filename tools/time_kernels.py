"""Standalone per-launch times of the bench's roofline kernels on a real C5
operator (after 2 bench steps): fine-level smoother sweep, FP64 SpMV,
element kernel (residual-only / with Jacobian)."""
import sys, ctypes as C, json
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
q = torch.from_numpy(st.q).cuda()
torch.cuda.synchronize()
ms = C.c_float()
L, h = sm.dev.lib, sm.dev.handle
out = {}
for name, fn in (("smoother", lambda r: L.dp_bench_smoother(h, _lib.ptr(x), _lib.ptr(b), _lib.ptr(o), r, C.byref(ms))),
                 ("spmv", lambda r: L.dp_bench_spmv(h, 1, _lib.ptr(x), _lib.ptr(o), r, C.byref(ms))),
                 ("elem_res", lambda r: L.dp_bench_elements(h, _lib.ptr(q), 0, r, C.byref(ms))),
                 ("elem_jac", lambda r: L.dp_bench_elements(h, _lib.ptr(q), 1, r, C.byref(ms)))):
    _lib.check(fn(3))
    _lib.check(fn(20))
    out[name + "_us"] = round(1e3 * ms.value / 20, 2)
print(json.dumps(out))
