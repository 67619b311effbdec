"""Variance probe: repeat the device-resident C5 rollout (3 steps fwd+bwd) and
print per-repeat ms (CUDA events on the scene stream) and host wall."""
import os, sys, time
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, '.')
import torch
import bench
from paper_2603_16478_b200 import core, forward as fw, adjoint as aj, _lib
torch.cuda.set_device(0)
cpus = sorted(os.sched_getaffinity(0))
PIN = int(os.environ.get('PIN', '1'))
if PIN: os.sched_setaffinity(0, set(cpus[1:1 + PIN]))
sc = bench.make_scene(55); sm = core.assemble_system_matrix(sc)
L = sm.dev.lib
cfg = fw.ForwardConfig(tol=1e-11)
n3 = 3 * sc.n_verts
dd = dict(device="cuda:0", dtype=torch.float64)
stream = torch.cuda.ExternalStream(L.dp_scene_stream(sm.dev.handle))
import gc
if os.environ.get("GCFREEZE"):
    gc.collect(); gc.freeze()
for rep in range(int(os.environ.get('REPS', '8'))):
    q = [torch.empty(n3, **dd) for _ in range(4)]; v = [torch.empty(n3, **dd) for _ in range(4)]
    q[0].copy_(torch.from_numpy(sc.vertices.reshape(-1))); v[0].zero_(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(stream)
    tf = []
    for k in range(3):
        bench.move_fingers(sc, 3 + k)
        t1 = time.perf_counter()
        fw.forward_step(sc, None, sm, cfg, device_io=dict(q_bar=q[k], v_bar=v[k], q_out=q[k+1], v_out=v[k+1]))
        tf.append(round((time.perf_counter() - t1) * 1e3, 1))
    e1.record(stream); torch.cuda.synchronize()
    print(rep, "fwd ms", round(e0.elapsed_time(e1), 1), "host", round((time.perf_counter() - t0) * 1e3, 1), tf, flush=True)

# pure device loop: 2000 SpMVs, repeated
import ctypes as C
x = torch.randn(n3, **dd); y = torch.empty(n3, **dd); ms = C.c_float()
for rep in range(0):
    L.dp_bench_spmv(sm.dev.handle, 1, _lib.ptr(x), _lib.ptr(y), 2000, C.byref(ms))
    print("spmv x2000 ms", round(ms.value, 1), flush=True)
# sync-heavy loop: 2000 x (spmv + sync)
for rep in range(0):
    t0 = time.perf_counter()
    for i in range(500):
        L.dp_bench_spmv(sm.dev.handle, 1, _lib.ptr(x), _lib.ptr(y), 1, C.byref(ms))
    print("500 x (spmv+sync) ms", round((time.perf_counter() - t0) * 1e3, 1), flush=True)
