"""Variance probe: repeated 3-step C5 forward rollouts (public API) in one
process; prints per-repeat ms."""
import os, sys, time
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, '.')
import bench  # noqa (applies the heap settings)
from paper_2603_16478_b200 import core, forward as fw
sc = bench.make_scene("c5"); sm = core.assemble_system_matrix(sc)
cfg = fw.ForwardConfig(tol=1e-11)
out = []
t_start = time.perf_counter()
for rep in range(int(os.environ.get("REPS", "30"))):
    t0 = time.perf_counter()
    st = sc.rest_state()
    for k in range(3):
        bench.move_fingers(sc, k)
        st, rep_ = fw.forward_step(sc, st, sm, cfg)
    out.append((round(time.perf_counter() - t_start, 1), round((time.perf_counter() - t0) * 1e3, 1)))
print(out)
