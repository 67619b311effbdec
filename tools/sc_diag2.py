import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests'); sys.path.insert(0,'oracle')
import test_gpu_self_contact as T
import self_contact_oracle as SO
from paper_2603_16478_b200 import core, forward as fw
scene, q0, _ = T._stacked_cubes(gap=4e-4)
scene.eps_fb = 1e-9
st0 = scene.rest_state(); st0.v[2::3] = -0.05
sm = core.assemble_system_matrix(scene)
st, rep = fw.forward_step(scene, st0, sm, fw.ForwardConfig(tol=1e-10))
P = st.q.reshape(-1, 3); nv = len(P) // 2
print("lower top z", P[:nv, 2].max(), "upper bottom z", P[nv:, 2].min(), "lower bottom", P[:nv,2].min())
P0 = q0.reshape(-1,3)
print("q0: lower top", P0[:nv,2].max(), "upper bottom", P0[nv:,2].min())
tri, d2, gap, n = SO.self_contacts(q0, st.q, scene.elements, scene.contact_activation)
print("oracle self contacts at final q vs frozen q0:", (tri>=0).sum(), "min gap", gap[tri>=0].min() if (tri>=0).any() else None)
qh = st0.q + 0.01*st0.v + 1e-4*np.tile([0,0,-9.8], scene.n_verts)
tri, d2, gap, n = SO.self_contacts(q0, qh, scene.elements, scene.contact_activation)
print("oracle self contacts at q_hat:", (tri>=0).sum(), "min gap", gap[tri>=0].min() if (tri>=0).any() else None)
