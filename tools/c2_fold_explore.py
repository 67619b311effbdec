"""C2 fold exploration on the GPU: an ARAP cloth sheet on the ground, its
right edge bound to targets that swing over the centre line (a half fold),
with self-contact.  argv: JSON list of {n, steps, fold, eps, tol, mu, mus,
comp, stiff, h, max_iter, th0, lift}."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_16478_b200 import core, forward as fw, ident  # noqa: E402


def fold_scene(d):
    n = d.get("n", 40)
    size = d.get("size", 0.4)
    edge = size / n
    v, t = ident.horizontal_sheet(n, n, edge, origin=(0.0, 0.0, 5e-4))
    m = core.lumped_masses(v, t, 0.3)
    right = np.nonzero(np.abs(v[:, 0] - size) < 1e-12)[0]
    binds = [core.BindingSpec(int(i), v[i].copy(), d.get("comp", 1e-6)) for i in right]
    sc = core.Scene(v, t, m, [core.MaterialParams("arap", stiffness=d.get("stiff", 50.0))] * len(t),
                    colliders=[core.HalfSpace([0, 0, 1], 0.0, mu=d.get("mu", 0.0))], bindings=binds, h=d.get("h", 0.01),
                    eps_fb=d.get("eps", 1e-9), self_contact=True, self_mu=d.get("mus", 0.0))
    return sc, size


def fold_angle(k, fold, th0):
    return th0 + (np.pi - th0) * min(1.0, (k + 1) / fold)


def folded(v, size, th, lift):
    """The sheet with its right half rotated by th about the crease line
    x = size/2 (a rigid fold; the crease row stays), lifted by `lift`."""
    q = v.copy()
    xc = 0.5 * size
    r = q[:, 0] > xc + 1e-12
    d = q[r, 0] - xc
    q[r, 0] = xc + d * np.cos(th)
    q[r, 2] = q[r, 2] + d * np.sin(th) + lift * np.minimum(1.0, d / (0.1 * size))
    return q


def set_fold(sc, size, k, fold, th0=0.0, lift=2e-3):
    """targets of the bound edge at step k: the edge of the rigidly folded
    sheet at angle th(k) = th0 + (pi - th0) min(1, (k+1)/fold)."""
    th = fold_angle(k, fold, th0)
    tgt = folded(sc.vertices, size, th, lift)
    for b in sc.bindings:
        b.target = tgt[b.vertex].copy()


for d in json.loads(sys.argv[1]):
    sc, size = fold_scene(d)
    sm = core.assemble_system_matrix(sc)
    st = sc.rest_state()
    th0 = d.get("th0", 0.0)
    if th0:
        st.q[:] = folded(sc.vertices, size, th0, d.get("lift", 2e-3)).reshape(-1)
    cfg = fw.ForwardConfig(tol=d.get("tol", 1e-10), max_iter=d.get("max_iter", 100))
    its, t0, ok, nself = [], time.time(), True, []
    for k in range(d.get("steps", 60)):
        set_fold(sc, size, k, d.get("fold", 40), th0, d.get("lift", 2e-3))
        try:
            st, rep = fw.forward_step(sc, st, sm, cfg)
        except Exception as ex:  # noqa: BLE001
            its.append(f"EXC@{k}:{str(ex)[:40]}")
            ok = False
            break
        if not rep.converged:
            its.append(f"NC@{k}:{rep.residual_history[-1]:.1e}")
            ok = False
            break
        its.append(rep.iterations)
        cols = [c.collider for c in rep.cache.contacts]
        nself.append(int(sum(1 for c in cols if c == len(sc.colliders))))
    P = st.q.reshape(-1, 3)
    print(json.dumps(dict(d=d, ok=ok, n=len(its), its=its, self_contacts=nself[-5:], zmax=float(P[:, 2].max()),
                          xmin=float(P[:, 0].min()), xmax=float(P[:, 0].max()), t=round(time.time() - t0, 1))),
          flush=True)
