"""Variance probe on the C3 beam: 20 repeats of a 6-step fwd rollout through
the public API; prints ms per repeat."""
import os, sys, time
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, '.')
import bench
from paper_2603_16478_b200 import core, forward as fw
if os.environ.get("PIN"):
    os.sched_setaffinity(0, {int(os.environ["PIN"])})
sc = bench.make_scene("c3"); sm = core.assemble_system_matrix(sc)
cfg = fw.ForwardConfig(tol=1e-9)
out = []
for rep in range(20):
    t0 = time.perf_counter()
    st = sc.rest_state()
    for k in range(6):
        st, rep_ = fw.forward_step(sc, st, sm, cfg)
    out.append(round((time.perf_counter() - t0) * 1e3, 1))
print(out)
