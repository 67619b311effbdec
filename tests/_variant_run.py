"""Helper for tests/test_gpu_variants.py: a C5-family rollout (12^3 cells: a 3-level hierarchy, two
moving sphere fingers, frictional ground) forward + reverse sweep; prints a
bitwise digest of the final state and the gradient.  Solver switches come in
through the environment (read once when the library loads)."""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_16478_b200 import adjoint as aj, core, forward as fw  # noqa: E402

scene = bench.make_scene(int(os.environ.get("VARIANT_CELLS", "12")), fingers=True)
sm = core.assemble_system_matrix(scene)
st = scene.rest_state()
caches = []
for k in range(3):
    bench.move_fingers(scene, k)
    st, rep = fw.forward_step(scene, st, sm, fw.ForwardConfig(tol=1e-11))
    assert rep.converged
    caches.append(rep.cache)
g = aj.backprop_rollout(caches, st.q + 1e-3)
h = hashlib.sha256(np.ascontiguousarray(st.q).tobytes() + np.float64(g.dL_dE).tobytes()
                   + np.ascontiguousarray(g.dL_dqbar).tobytes()).hexdigest()
print("DIGEST", h, repr(float(g.dL_dE)))
if os.environ.get("VARIANT_OUT"):
    np.savez(os.environ["VARIANT_OUT"], q=st.q, dL_dE=g.dL_dE, dL_dqbar=g.dL_dqbar)
