"""Diagnostic: C2-family cloth (n x n sheet over a sphere) on the GPU next to
the oracle (same input state every step).  argv: n steps eps tol [oracle]."""
import sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np, bench
from paper_2603_16478_b200 import core, forward as fw
n = int(sys.argv[1]); steps = int(sys.argv[2]); eps = float(sys.argv[3]); tol = float(sys.argv[4])
use_oracle = len(sys.argv) > 5 and sys.argv[5] == "1"
bench.CONFIGS["c2s"] = dict(bench.CONFIGS["c2"], cells=(n, n, 0), edge=1.0 / n)
sc = bench.make_scene("c2s", eps_fb=eps)
sm = core.assemble_system_matrix(sc)
st = sc.rest_state()
cfg = fw.ForwardConfig(tol=tol)
if use_oracle:
    import diffproj_oracle as O
    osc = O.OScene(core.scene_to_arrays(sc))
    els = O.build_elements(osc)
    A = O.assemble_A(osc, els)
for k in range(steps):
    t0 = time.time()
    st1, rep = fw.forward_step(sc, st, sm, cfg)
    line = f"{k} gpu conv={rep.converged} it={rep.iterations} kry={rep.krylov_iterations} C={rep.n_contacts} r={rep.residual_history[-1]:.3e} t={time.time()-t0:.2f}"
    if use_oracle:
        res = O.forward_step(osc, A, els, st.q, st.v, O.ForwardConfig(tol=tol))
        d = np.max(np.abs(res.q_new - st1.q)) / np.max(np.abs(res.q_new))
        line += f" | oracle conv={res.converged} it={res.iterations} C={len(res.contacts.vertex)} dq_rel={d:.2e}"
    print(line, flush=True)
    st = st1
