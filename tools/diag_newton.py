"""Diagnostic: per-step Newton residual histories of the bench scene family."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.')
import bench
from paper_2603_16478_b200 import forward as fw, core

def run(n, steps, fingers=True, tol=1e-9, rmax=1e-3, eps=None):
    sc = bench.make_scene(n, fingers=fingers, eps_fb=eps)
    sm = core.assemble_system_matrix(sc)
    st = sc.rest_state()
    cfg = fw.ForwardConfig(tol=tol, lin_rtol_max=rmax)
    out = []
    for k in range(steps):
        bench.move_fingers(sc, k)
        t0 = time.time()
        st, rep = fw.forward_step(sc, st, sm, cfg)
        out.append(dict(k=k, conv=rep.converged, it=rep.iterations, kry=rep.krylov_iterations,
                        ls=rep.line_search_trials, nc=rep.n_contacts, t=round(time.time()-t0, 3),
                        hist=[float('%.3e' % h) for h in rep.residual_history[:12]] + (['...'] + [float('%.3e' % h) for h in rep.residual_history[-5:]] if rep.iterations > 12 else [])))
        print(json.dumps(out[-1]), flush=True)
    return out

if __name__ == '__main__':
    n = int(sys.argv[1]); steps = int(sys.argv[2]); fingers = sys.argv[3] == '1'
    rmax = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-3
    eps = float(sys.argv[5]) if len(sys.argv) > 5 else None
    run(n, steps, fingers, rmax=rmax, eps=eps)
