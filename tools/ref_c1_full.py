"""C1 in full on the CPU with the REFERENCE package itself (SURVEY.md §8(d)
item 1): box_tet_mesh(9,9,9) = 4,374 NH tets (E=1e4,
nu=0.3) dropped 0.5 mm onto a mu=0.3 ground, 100 implicit steps + the full
reverse sweep, dL/dE.  Runs only in the build container (imports
/root/reference read-only); writes profiles/r02_cpu_reference_c1.json.

argv: [steps] [impl]  impl = "reference" (default) or "oracle"."""
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
impl = sys.argv[2] if len(sys.argv) > 2 else "reference"

if impl == "reference":
    sys.path.insert(0, "/root/reference/pkg/src")
    from diffproj import adjoint as aj, core, forward as fw, ident  # noqa: E402
    v, t = ident.box_tet_mesh(9, 9, 9, size=0.1 / 9, origin=(0.0, 0.0, 5e-4))
    mats = [core.MaterialParams(model="neohookean", E=1e4, nu=0.3) for _ in range(len(t))]
    scene = core.Scene(vertices=v, elements=t, masses=core.lumped_masses(v, t, density=1000.0),
                       materials=mats, colliders=[core.HalfSpace([0, 0, 1], 0.0, mu=0.3)], h=0.01)
    sysmat = core.assemble_system_matrix(scene)
    state = scene.rest_state()
    caches, fwd_t, its = [], [], []
    t0 = time.perf_counter()
    for k in range(steps):
        a = time.perf_counter()
        state, rep = fw.forward_step(scene, state, sysmat, fw.ForwardConfig())
        fwd_t.append(time.perf_counter() - a)
        its.append(rep.iterations)
        if not rep.converged:
            raise RuntimeError(f"reference forward step {k} did not converge ({rep.residual_history[-1]:.3e})")
        caches.append(rep.cache)
        print(f"step {k}: {its[-1]} its {fwd_t[-1]:.2f} s", file=sys.stderr, flush=True)
    t_f = time.perf_counter() - t0
    target = scene.vertices.reshape(-1) + 1e-3
    a = time.perf_counter()
    g = aj.backprop_rollout(caches, target)
    t_b = time.perf_counter() - a
    out = dict(impl="reference (/root/reference/pkg/src/diffproj, unmodified)", steps=steps, tets=len(t),
               verts=len(v), fwd_s=t_f, bwd_s=t_b, fwd_s_per_step=t_f / steps, bwd_s_per_step=t_b / steps,
               steps_per_s=steps / (t_f + t_b), newton_iterations=its, dL_dE=float(g.dL_dE),
               dL_dnu=float(g.dL_dnu), dL_dmu=float(g.dL_dmu_friction),
               cpu=platform.processor() or platform.machine(), nproc=os.cpu_count(),
               blas_threads=os.environ.get("OPENBLAS_NUM_THREADS", "default"))
    path = os.path.join(ROOT, "profiles", f"r02_cpu_reference_c1_{steps}.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))
