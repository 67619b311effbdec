"""Profile helper: the C5 element kernel at a deformed state (after 3 bench
steps): one residual-only and one Jacobian launch via dp_bench_elements.
Run under ncu with the DFMA/DMUL/DADD instruction metrics to get FP64 FLOPs
per element."""
import sys, ctypes as C
sys.path.insert(0, '.')
import torch
import bench
from paper_2603_16478_b200 import core, forward as fw, _lib
sc = bench.make_scene("c5")
sm = core.assemble_system_matrix(sc)
st = sc.rest_state()
for k in range(3):
    bench.move_fingers(sc, k)
    st, rep = fw.forward_step(sc, st, sm, fw.ForwardConfig(tol=bench.CONFIGS["c5"]["tol"]))
q = torch.from_numpy(st.q).cuda()
torch.cuda.synchronize()
ms = C.c_float()
for jac in (0, 1):
    _lib.check(sm.dev.lib.dp_bench_elements(sm.dev.handle, _lib.ptr(q), jac, 1, C.byref(ms)))
    print("jac", jac, "ms", ms.value)
