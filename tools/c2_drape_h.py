"""C2 drape (100 x 100 ARAP cloth over a frictional sphere): how many steps
converge at h = 10 ms vs 5 ms / 2.5 ms (the reference's Newton fails at step
6 at h = 10 ms)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_16478_b200 import core, forward as fw  # noqa: E402

for h, steps in ((0.01, 12), (0.005, 24), (0.0025, 48)):
    sc = bench.make_scene("c2")
    sc.h = h
    sm = core.assemble_system_matrix(sc)
    st = sc.rest_state()
    cfg = fw.ForwardConfig(tol=bench.CONFIGS["c2"]["tol"])
    its, t0 = [], time.time()
    for k in range(steps):
        try:
            st, rep = fw.forward_step(sc, st, sm, cfg)
        except Exception as ex:  # noqa: BLE001
            its.append(f"EXC@{k}:{str(ex)[:40]}")
            break
        if not rep.converged:
            its.append(f"NC@{k}:{rep.residual_history[-1]:.1e}")
            break
        its.append(rep.iterations)
    print(json.dumps(dict(h=h, steps=steps, its=its, t=round(time.time() - t0, 1))), flush=True)
