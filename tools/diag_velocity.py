import sys, os
sys.path.insert(0, '.')
import numpy as np, bench
from paper_2603_16478_b200 import forward as fw, core
sc = bench.make_scene("c5", eps_fb=1e-9)
sm = core.assemble_system_matrix(sc)
st = sc.rest_state()
cfg = fw.ForwardConfig(tol=1e-10)
for k in range(7):
    bench.move_fingers(sc, k)
    st, rep = fw.forward_step(sc, st, sm, cfg)
    v = st.v.reshape(-1, 3); q = st.q.reshape(-1, 3)
    sp = np.linalg.norm(v, axis=1); i = np.argsort(-sp)[:4]
    print(k, rep.iterations, "vmax", sp[i], "at", q[i].round(5).tolist(), "median", np.median(sp), flush=True)
