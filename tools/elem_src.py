"""Profile helper: one residual-only element launch at a C5 state, between
cudaProfilerStart/Stop (ncu --profile-from-start off --import-source on)."""
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
q = torch.from_numpy(st.q).cuda()
torch.cuda.synchronize()
ms = C.c_float()
torch.cuda.profiler.start()
_lib.check(sm.dev.lib.dp_bench_elements(sm.dev.handle, _lib.ptr(q), int(sys.argv[1]) if len(sys.argv) > 1 else 0, 1, C.byref(ms)))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
