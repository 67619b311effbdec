import sys; sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import numpy as np, bench, diffproj_oracle as O
from paper_2603_16478_b200 import core, forward as fw
c = dict(cells=(2, 2, 40), edge=2.5e-3, eps_fb=1e-10, wall_gap=5e-4)
scene = bench.make_trunk(c, 1e5)
osc = O.OScene(core.scene_to_arrays(scene)); els = O.build_elements(osc); A = O.assemble_A(osc, els)
sm = core.assemble_system_matrix(scene)
st = scene.rest_state(); q, v = st.q.copy(), st.v.copy()
f = np.zeros(3 * scene.n_verts)
for ci, line in enumerate(scene._cable_lines):
    f[3 * line] += (1.0 if ci in (1, 3) else -0.2) * 3e-4 * (1/3.)
scene.fext = f; osc.fext = f.copy()
for tol in (1e-11, 1e-13):
    st1, rep = fw.forward_step(scene, st, sm, fw.ForwardConfig(tol=tol))
    o = O.forward_step(osc, A, els, q, v, O.ForwardConfig(tol=tol))
    print("tol", tol, "gpu it", rep.iterations, rep.converged, rep.residual_history[-3:], "oracle it", o.iterations, o.converged, o.residual_history[-3:])
    d = np.abs(st1.q - o.q_new); i = np.argmax(d)
    print("  max dq", d.max(), "at dof", i, "vertex", i//3)
    # oracle residual at the GPU's q
    q_hat = O.predict(osc, q, v)
    ct = O.detect_contacts(osc, st1.q)
    es = O.project_elements(els, st1.q, False)
    O.solve_multipliers(ct, st1.q, q)
    r = O.momentum_residual(osc, A, els, es, st1.q, q_hat, ct)
    print("  oracle residual at gpu q", np.abs(r).max(), "at", np.argmax(np.abs(r)))
