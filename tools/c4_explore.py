"""C4 trunk over a long horizon on the GPU: per-step Newton iterations for
cable amplitude / wall-gap variants.  argv: JSON list of {amp, gap, steps, tol}."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_16478_b200 import core, forward as fw  # noqa: E402

for d in json.loads(sys.argv[1]):
    c = dict(bench.CONFIGS["c4"], wall_gap=d.get("gap", 5e-3))
    sc = bench.make_scene(c)
    sc._cable_amp = d.get("amp", 2e-3)
    sm = core.assemble_system_matrix(sc)
    st = sc.rest_state()
    cfg = fw.ForwardConfig(tol=d.get("tol", c["tol"]))
    its, t0, ok = [], time.time(), True
    for k in range(d.get("steps", 200)):
        bench.move_fingers(sc, k)
        try:
            st, rep = fw.forward_step(sc, st, sm, cfg)
        except Exception as ex:  # noqa: BLE001
            its.append(f"EXC@{k}:{str(ex)[:40]}")
            ok = False
            break
        its.append(rep.iterations if rep.converged else f"NC@{k}")
        if not rep.converged:
            ok = False
            break
    xmax = float(st.q[0::3].max())
    print(json.dumps(dict(d=d, ok=ok, n=len(its), its=its[-12:], maxit=max([i for i in its if isinstance(i, int)] or [0]),
                          nc=rep.n_contacts, xmax=xmax, t=round(time.time() - t0, 1))), flush=True)
