import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests'); sys.path.insert(0,'oracle')
import test_gpu_self_contact as T
from paper_2603_16478_b200 import core, forward as fw
for eps, tol in ((1e-7, 1e-12), (1e-7, 1e-9), (1e-9, 1e-10), (1e-9, 1e-11)):
    scene, q0, _ = T._stacked_cubes(gap=4e-4)
    scene.eps_fb = eps
    st0 = scene.rest_state(); st0.v[2::3] = -0.05
    sm = core.assemble_system_matrix(scene)
    st, rep = fw.forward_step(scene, st0, sm, fw.ForwardConfig(tol=tol))
    cols = np.array([c.collider for c in rep.cache.contacts])
    print(eps, tol, rep.converged, rep.iterations, (cols == 1).sum(), (cols==0).sum(), ['%.1e' % h for h in rep.residual_history[-5:]], flush=True)
