"""Profile helper: one C5 forward step, then the adjoint inside an NVTX range
"adjoint" (ncu --nvtx --nvtx-include adjoint/)."""
import sys
import torch
sys.path.insert(0, '.')
import bench
from paper_2603_16478_b200 import forward as fw, core, adjoint as aj
sc = bench.make_scene(int(sys.argv[1]), fingers=True)
sm = core.assemble_system_matrix(sc)
st = sc.rest_state()
caches = []
for k in range(int(sys.argv[2])):
    bench.move_fingers(sc, k)
    st, rep = fw.forward_step(sc, st, sm, fw.ForwardConfig())
    caches.append(rep.cache)
torch.cuda.nvtx.range_push("adjoint")
g = aj.backprop_rollout(caches, st.q + 1e-3)
torch.cuda.nvtx.range_pop()
print("dE", g.dL_dE)
