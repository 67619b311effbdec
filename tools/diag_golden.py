"""Replay a reference fixture scene (tests/golden/scene_<name>.npz) on the GPU
step by step with the fixture's tolerance; print Newton iterations vs the
reference's and the state error.  argv: name [steps] [lin_rtol]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_16478_b200 import core, forward as fw  # noqa: E402

name = sys.argv[1]
g = dict(np.load(os.path.join(ROOT, "tests", "golden", f"scene_{name}.npz")))
T = int(sys.argv[2]) if len(sys.argv) > 2 else int(g["T"])
eta = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
scene = core.scene_from_arrays(g)
sm = core.assemble_system_matrix(scene)
st = core.SimState(g["q"][0], g["v0"])
cfg = fw.ForwardConfig(tol=float(g["tol"]), lin_rtol_max=eta, lin_rtol_min=eta)
for k in range(T):
    if "finger_x" in g:
        scene.colliders[1].center[0], scene.colliders[2].center[0] = g["finger_x"][k]
    st, rep = fw.forward_step(scene, st, sm, cfg)
    err = np.max(np.abs(st.q - g["q"][k + 1])) / np.max(np.abs(g["q"][k + 1]))
    print(f"step {k}: conv {rep.converged} its {rep.iterations} (ref {g['iterations'][k]}) err {err:.2e} "
          f"hist {[f'{h:.1e}' for h in rep.residual_history[-6:]]}", flush=True)
    if not rep.converged:
        break
