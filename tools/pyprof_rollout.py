import sys, time, os
sys.path.insert(0, '.')
import numpy as np
from paper_2603_16478_b200 import forward as fw, core, _lib
orig_check = _lib.check
T = {}
D = {}
def timed(name, f):
    def g(*a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); dt = time.perf_counter() - t0
        T[name] = T.get(name, 0) + dt; D.setdefault(name, []).append(round(dt * 1e3, 2)); return r
    return g
core.DeviceScene.sync = timed("sync", core.DeviceScene.sync)
fw.DeviceCache.__init__ = timed("cache_create", fw.DeviceCache.__init__)
import gc
gcs = []
def cb(phase, info):
    if phase == "start": cb.t = time.perf_counter()
    else: gcs.append((info["generation"], time.perf_counter() - cb.t))
gc.callbacks.append(cb)
import runpy
sys.argv = ["tools/time_rollout.py", "c5", "6", "15", "1"]
try:
    runpy.run_path("tools/time_rollout.py", run_name="__main__")
finally:
    print("T", {k: round(v, 4) for k, v in T.items()})
    print("cache_create ms", D.get("cache_create"))
    big = sorted(gcs, key=lambda x: -x[1])[:5]
    print("gc", len(gcs), "max", [(g, round(t * 1e3, 2)) for g, t in big])
