"""The CPU oracle (reference semantics, exact SuperLU Newton solves) over the
C5 family schedule at n cells per side: per-step convergence / iterations /
time.  argv: n steps.  Test infrastructure / measurement only."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import diffproj_oracle as O  # noqa: E402
from paper_2603_16478_b200 import core  # noqa: E402

n = int(sys.argv[1])
steps = int(sys.argv[2])
fam = bench.c5_family(n)
scene = bench.make_scene(fam)
osc = O.OScene(core.scene_to_arrays(scene))
els = O.build_elements(osc)
A = O.assemble_A(osc, els)
q = scene.vertices.reshape(-1).copy()
v = np.zeros_like(q)
out = []
t0 = time.perf_counter()
for k in range(steps):
    bench.move_fingers(scene, bench.FINGER_K0 + k)
    osc = O.OScene(core.scene_to_arrays(scene))
    a = time.perf_counter()
    st = O.forward_step(osc, A, els, q, v, O.ForwardConfig(tol=fam["tol"]))
    out.append(dict(k=k, conv=st.converged, it=st.iterations, nc=len(st.contacts.vertex),
                    t=round(time.perf_counter() - a, 2), r=st.residual_history[-1]))
    print(json.dumps(out[-1]), flush=True)
    if not st.converged:
        break
    q, v = st.q_new, st.v_new
print("total", round(time.perf_counter() - t0, 1), "s", flush=True)
