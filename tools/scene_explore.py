"""Scene-design exploration for the C5 workload: per design, run the GPU
forward rollout and print the Newton iteration count / convergence of every
step (stops a design at its first non-converged step).

argv[1]: JSON list of designs, each a dict with keys
  n (cells/side), eps, tol, speed (m/step), hold (finger index where closing
  stops), muf (finger mu), mug (ground mu), steps, gap0 (initial finger gap),
  r (finger radius)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2603_16478_b200 import core, forward as fw, ident  # noqa: E402


def scene_of(d):
    n = d.get("n", 55)
    edge = 0.1 / n
    v, t = ident.box_tet_mesh(n, n, n, size=edge, origin=(0.0, 0.0, 5e-4))
    mat = core.MaterialParams("neohookean", E=d.get("E", 1e4), nu=0.3)
    cols = [core.HalfSpace([0, 0, 1], 0.0, mu=d.get("mug", 0.5))]
    r = d.get("r", 0.02)
    gap0 = d.get("gap0", 5e-4)
    L = n * edge
    zc = 5e-4 + L / 2
    cols.append(core.Sphere([-r - gap0, L / 2, zc], r, mu=d.get("muf", 0.5)))
    cols.append(core.Sphere([L + r + gap0, L / 2, zc], r, mu=d.get("muf", 0.5)))
    if d.get("push"):
        # kinematic pusher plate behind the cube (frictionless by default)
        cols.append(core.HalfSpace([0, 1, 0], -gap0, mu=d.get("mup", 0.0)))
    sc = core.Scene(v, t, core.lumped_masses(v, t, 1000.0), [mat] * len(t), colliders=cols, h=0.01,
                    eps_fb=d.get("eps", 1e-9))
    return sc, L, r, gap0


def main():
    designs = json.loads(sys.argv[1])
    for d in designs:
        if d.get("mscale"):
            # eps^2 and the (absolute, kg m) Newton tolerance scaled with the
            # vertex mass relative to the 55^3 workload
            f = (55.0 / d.get("n", 55)) ** 3
            d["eps"] = d.get("eps", 1e-9) * f
            d["tol"] = d.get("tol", 1e-11) * f
        sc, L, r, gap0 = scene_of(d)
        sm = core.assemble_system_matrix(sc)
        st = sc.rest_state()
        vp = d.get("push", 0.0)
        st.v[1::3] = d.get("v0", vp)
        cfg = fw.ForwardConfig(tol=d.get("tol", 1e-11))
        its, ok = [], True
        t0 = time.time()
        for k in range(d.get("steps", 40)):
            p = min(k, d.get("hold", 10 ** 9)) * d.get("speed", 2e-5)
            sc.colliders[1].center[0] = -r - gap0 + p
            sc.colliders[2].center[0] = L + r + gap0 - p
            if vp:
                y = vp * sc.h * k
                sc.colliders[1].center[1] = L / 2 + y
                sc.colliders[2].center[1] = L / 2 + y
                sc.colliders[3].offset = -gap0 + y
            try:
                st, rep = fw.forward_step(sc, st, sm, cfg)
            except Exception as ex:   # noqa: BLE001
                its.append(f"EXC:{type(ex).__name__}:{str(ex)[:80]}")
                ok = False
                break
            its.append(rep.iterations)
            if not rep.converged:
                its[-1] = f"NC{rep.residual_history[-1]:.1e}"
                ok = False
                break
        print(json.dumps(dict(design=d, ok=ok, its=its, nc=rep.n_contacts if ok else None,
                              t=round(time.time() - t0, 1))), flush=True)


if __name__ == "__main__":
    main()
