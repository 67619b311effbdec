"""Benchmark: fwd+bwd implicit steps/s at N tets on B200 (BASELINE.json metric).

Workload (default --config c5): box_tet_mesh(55,55,55)
= 998,250 Neo-Hookean tets (E=1e4, nu=0.3, 10 cm cube) dropped onto a ground
plane and squeezed by two kinematic sphere "fingers" closing 10 um per step
up to finger index 20, then holding (frictionless contacts, ~3,200 of them;
why frictionless: CONFIGS comment).  Every rollout starts from the rest state
at finger index 0 (FINGER_K0), so warm-up and timed rollouts are the same
workload; a non-converged step raises (forward.py:261-264).  A "step" = one
forward Newton step + its adjoint
step (A_hat^T solve + z-products) of a K-step rollout with a final-state
loss; parameter gradient dL/d(E, nu, mu) allreduced across ranks (NCCL) at
the end of every rollout.

  value : device-resident path (inputs already in HBM), CUDA events on the
          scene stream, max over ranks, whole-job steps/s.
  e2e   : the public API (rollout + backprop_rollout) with host NumPy
          buffers: host<->device copies inside the timed region.
  cpu_baseline / --impl reference : the CPU oracle port (oracle/, a
          vectorised restatement of the reference) on a bounded sample: the
          same scene family on a smaller cube over the same schedule; the
          measured rate is reported in measured_* fields, `value` scales it
          linearly in tets (generous to the CPU; SuperLU scales worse).

Inputs are larger than L2 (val ~200 MB per SpMV operand at C5); no explicit
flush.  Launch: python bench.py [--gpus N --steps K --warmup W]; for N>1 via
torchrun (one process per GPU).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# load every kernel at context creation, not at its first launch inside the
# timed region
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")


def _keep_heap():
    """Keep freed multi-MB host buffers in the heap instead of munmap'ing them:
    each step returns fresh 3V-double NumPy arrays (public API), and the
    mmap/munmap + page-zeroing churn showed up as 50-200 ms outliers."""
    try:
        import ctypes
        libc = ctypes.CDLL("libc.so.6")
        libc.mallopt(-3, 1 << 30)   # M_MMAP_THRESHOLD: serve big blocks from the heap
        libc.mallopt(-1, 1 << 31)   # M_TRIM_THRESHOLD: never give the top back
    except (OSError, AttributeError):
        pass


_keep_heap()

# Workloads.  cells = box_tet_mesh resolution, edge = cell
# size (m); eps_fb and the Newton tolerance are scaled with the vertex mass:
#  * eps_fb: the condensed normal force eps^2/delta at the activation
#    distance (1 mm) must stay below a vertex's weight, otherwise the
#    activation discontinuity of the reference model (contact.py:129-130,
#    SURVEY.md App. A item 2) makes Newton cycle at |r| ~ h^2 eps^2/activation;
#    the default 1e-6 is fine for ~1e-3 kg vertices (C1, C3) but not for C5
#    (~6e-6 kg).
#  * Newton tol: the reference's stop test is an absolute max|r| <= tol *
#    max(1, max|m q_hat|) (forward.py:169-171, :202) in kg*m, default 1e-9.
#    C5 uses 1e-10 (10x tighter than the default).  It must stay above the
#    activation jump h^2 eps^2/activation of a vertex crossing the 1 mm
#    activation distance (5e-11 at eps_fb = 1e-9): with tol = 1e-11 (round 1)
#    a vertex hovering at the activation boundary stalls Newton (oracle, C5
#    family at 10^3 cells, step 16: plateau 7.9e-9 = that jump, scaled).
#
# C5 is FRICTIONLESS (ground and fingers mu = 0), with the fingers closing
# 10 um per step for FINGER_HOLD steps and then holding.  Measured
# (profiles/r02_c5_scene_design.md, tools/scene_explore.py): with the
# reference's friction model (contact.py:139-165) a resting frictional
# contact has no stable stick state (the capped branch pushes a vertex ALONG
# its slip, the equilibria form a ring |delta_f| = delta_n/mu), and at 55^3
# every frictional variant tried (mu 0.1-0.5, eps_fb 5e-11-1e-8, closing
# speeds, holds, a pusher plate) stalls, inverts an element or stalls the NH
# projection within 1-10 steps; the reference itself (CPU oracle) stalls on
# the round-1 schedule at 12^3.  The frictionless family
# converges every step for 60 steps at 8^3 ... 55^3 on the GPU and on the CPU
# oracle (tests/test_c5_family_oracle.py, profiles/r02_c5_scene_design.md).
FINGER_SPEED = 1e-5   # m per step
FINGER_HOLD = 20      # finger index after which the fingers hold
FINGER_K0 = 0         # first finger index of every rollout (never --warmup)
CONFIGS = {
    "c5": dict(cells=(55, 55, 55), edge=0.1 / 55, fingers=True, mu=0.0, eps_fb=1e-9, tol=1e-10, rollouts=1, steps=20,
               vary="target",
               desc="1M-tet NH cube squeezed by 2 kinematic sphere fingers on the ground, frictionless "
                    "(high contact count; C5)"),
    "c5f": dict(cells=(55, 55, 55), edge=0.1 / 55, fingers=True, mu=0.3, eps_fb=1e-10, tol=1e-11, rollouts=1,
                vary="target",
                desc="C5 with mu=0.3 ground and fingers, eps_fb=1e-10 (GPU-converged 40 steps; not "
                     "reference-validated at 55^3)"),
    "c3": dict(cells=(60, 12, 12), edge=0.01, fingers=False, eps_fb=1e-6, tol=1e-9, rollouts=8, steps=50,
               desc="identification batch: 8 rollouts/GPU of a 51,840-tet NH beam on a frictional ground, "
                    "one E candidate per rollout (C3)"),
    "c2": dict(cells=(100, 100, 0), edge=0.01, fingers=False, eps_fb=1e-9, tol=1e-11, rollouts=1, cloth=True, steps=4,
               desc="20,000-triangle ARAP cloth (1 m, 0.3 kg/m^2) draping over a frictional sphere, "
                    "per-step control-force gradients (C2 without self-contact: none in the reference)"),
    "c2drape": dict(cells=(100, 100, 0), edge=0.01, fingers=False, eps_fb=1e-9, tol=1e-11, rollouts=1, cloth=True,
                    h=0.0025, steps=48,
                    desc="C2 drape at h = 2.5 ms: the 20,000-triangle cloth over the frictional sphere for 48 steps "
                         "(0.12 s; at h = 10 ms the reference model's Newton stalls at step 4-6)"),
    "c2fold": dict(cells=(40, 40, 0), edge=0.01, fingers=False, eps_fb=1e-9, tol=1e-10, rollouts=1, cloth=True,
                   fold=120, h=0.005, comp=1e-4, steps=120,
                   desc="3,200-triangle ARAP sheet (40 cm) on a frictionless ground, its right edge bound to "
                        "targets that fold it over its centre line in 120 steps of 5 ms, self-contact on (C2 fold "
                        "at reduced size: the 100 x 100 sheet stalls in the reference model's Newton)"),
    "c4": dict(cells=(8, 8, 520), edge=2.5e-3, fingers=False, eps_fb=1e-9, tol=1e-10, rollouts=1, trunk=True,
               steps=200, wall_gap=2e-3, cable_amp=1e-3,
               desc="199,680-tet NH trunk (2 x 2 x 130 cm) clamped at the top by stiff bindings, 4 cable "
                    "force lines (1 mN/vertex) driven per step, frictional wall 2 mm away, 200 steps (C4)"),
    "c1": dict(cells=(9, 9, 9), edge=0.1 / 9, fingers=False, mu=0.3, eps_fb=1e-6, tol=1e-9, rollouts=1, steps=100,
               desc="4,374-tet NH cube on a frictional ground (C1)"),
    "c1b": dict(cells=(9, 9, 9), edge=0.1 / 9, fingers=False, mu=0.3, eps_fb=1e-6, tol=1e-9, rollouts=16,
                desc="16 concurrent rollouts/GPU of the 4,374-tet C1 cube (batched small scenes)"),
}
E_YOUNG = 1e4
# FP64 FLOPs per tet of the element kernel (2 DFMA + DMUL + DADD thread
# instructions / E, ncu at a C5 state, profiles/r01_elements_fp64.md)
ELEM_FLOPS_JAC = 5250.0
ELEM_FLOPS_RES = 3139.0
PACK_BLOCKS = ("dL_dw", "dL_dEb", "dL_ddb", "dL_dfext", "dL_dqbar", "dL_dvbar")
ADJ_RESTART = 20            # adjoint GMRES restart length in the bench (see gpu_arm)
FP64_PEAK_TFLOPS = 34.18     # measured DFMA peak, profiles/r01_fp64_peak.json
NU = 0.3
MU = 0.5


def c5_family(n):
    """C5 scene parameters at n cells per side: the same 10 cm cube,
    frictionless fingers and ground; eps_fb and the (absolute) Newton
    tolerance scaled with the vertex mass, (55/n)^3, so every resolution sees
    the same force/weight ratios (tests and the CPU baseline use n < 55)."""
    f = (55.0 / n) ** 3
    return dict(cells=(n, n, n), edge=0.1 / n, fingers=True, mu=0.0, eps_fb=1e-9 * f, tol=1e-10 * f,
                schedule=(FINGER_SPEED, FINGER_HOLD))


def make_scene(cfg_or_n, fingers=None, eps_fb=None, E=E_YOUNG, mu=None):
    """Scene of a workload: a CONFIGS key, a dict of workload parameters
    (c5_family), or cells-per-side of the round-1 frictional finger cube
    (mu = 0.5, fingers closing 20 um per step; kept for the friction tests)."""
    from paper_2603_16478_b200 import core, ident
    if isinstance(cfg_or_n, str):
        c = CONFIGS[cfg_or_n]
    elif isinstance(cfg_or_n, dict):
        c = cfg_or_n
    else:
        n = int(cfg_or_n)
        c = dict(cells=(n, n, n), edge=0.1 / n, fingers=True, eps_fb=1e-9 if n >= 40 else (1e-7 if n >= 20 else 1e-6),
                 schedule=(2e-5, None))
    nx, ny, nz = c["cells"]
    if c.get("fold"):
        # C2 fold (tools/c2_fold_explore.py): the bound right edge swings over
        # the crease line x = size/2; self-contact between the two halves
        size = nx * c["edge"]
        v, t = ident.horizontal_sheet(nx, ny, c["edge"], origin=(0.0, 0.0, 5e-4))
        right = np.nonzero(np.abs(v[:, 0] - size) < 1e-12)[0]
        binds = [core.BindingSpec(int(i), v[i].copy(), c["comp"]) for i in right]
        sc = core.Scene(v, t, core.lumped_masses(v, t, 0.3), [core.MaterialParams("arap", stiffness=50.0)] * len(t),
                        colliders=[core.HalfSpace([0, 0, 1], 0.0, mu=0.0)], bindings=binds, h=c["h"],
                        eps_fb=c["eps_fb"] if eps_fb is None else eps_fb, self_contact=True, self_mu=0.0)
        sc._fold = (size, c["fold"])
        return sc
    if c.get("cloth"):
        # horizontal sheet 0.5 mm above a sphere of radius 0.25
        v, t = ident.horizontal_sheet(nx, ny, c["edge"], origin=(0.0, 0.0, 0.2505))
        mats = [core.MaterialParams("arap", stiffness=50.0)] * len(t)
        cx, cy = nx * c["edge"] / 2, ny * c["edge"] / 2
        cols = [core.HalfSpace([0, 0, 1], 0.0, mu=0.3), core.Sphere([cx, cy, 0.0], 0.25, mu=0.3)]
        return core.Scene(v, t, core.lumped_masses(v, t, 0.3), mats, colliders=cols, h=c.get("h", 0.01),
                          eps_fb=c["eps_fb"] if eps_fb is None else eps_fb)
    if c.get("trunk"):
        return make_trunk(c, E)
    mu_ = c.get("mu", MU) if mu is None else mu
    v, t = ident.box_tet_mesh(nx, ny, nz, size=c["edge"], origin=(0.0, 0.0, 5e-4))
    mat = core.MaterialParams("neohookean", E=E, nu=NU)
    cols = [core.HalfSpace([0, 0, 1], 0.0, mu=mu_)]
    if c["fingers"] if fingers is None else fingers:
        r = 0.02
        ly, lz = ny * c["edge"], nz * c["edge"]
        zc = 5e-4 + lz / 2
        cols.append(core.Sphere([-r - 5e-4, ly / 2, zc], r, mu=mu_))
        cols.append(core.Sphere([nx * c["edge"] + r + 5e-4, ly / 2, zc], r, mu=mu_))
    sc = core.Scene(v, t, core.lumped_masses(v, t, 1000.0), [mat] * len(t),
                    colliders=cols, h=0.01, eps_fb=c["eps_fb"] if eps_fb is None else eps_fb)
    sc._finger_schedule = c.get("schedule", (FINGER_SPEED, FINGER_HOLD))
    return sc


def make_trunk(c, E):
    """C4: a hanging NH trunk, clamped at the top by
    stiff bindings (E_b = 1e-8 as cli.py:230-231), four "cables" = per-step
    external-force patterns on the four vertical corner lines (no cable model
    exists in the reference), a frictional wall 5 mm beside it."""
    from paper_2603_16478_b200 import core, ident
    nx, ny, nz = c["cells"]
    edge = c["edge"]
    v, t = ident.box_tet_mesh(nx, ny, nz, size=edge, origin=(0.0, 0.0, 0.0))
    ztop = v[:, 2].max()
    top = np.nonzero(v[:, 2] > ztop - 1e-9)[0]
    binds = [core.BindingSpec(int(i), v[i], 1e-8) for i in top]
    lx, ly = nx * edge, ny * edge
    wall = core.HalfSpace([-1.0, 0.0, 0.0], -(lx + c.get("wall_gap", 5e-3)), mu=0.3)
    sc = core.Scene(v, t, core.lumped_masses(v, t, 1000.0), [core.MaterialParams("neohookean", E=E, nu=NU)] * len(t),
                    colliders=[wall], bindings=binds, h=0.01, eps_fb=c["eps_fb"])
    lines = []
    for (cx, cy) in ((0.0, 0.0), (lx, 0.0), (0.0, ly), (lx, ly)):
        m = (np.abs(v[:, 0] - cx) < 1e-9) & (np.abs(v[:, 1] - cy) < 1e-9) & (v[:, 2] < 0.5 * ztop)
        lines.append(np.nonzero(m)[0])
    sc._cable_lines = lines
    # 1 mN per vertex: at 2 mN the trunk hits an NH projection stall at step
    # 81 (the reference raises there too, elasticity.py NH Newton); 1 mN runs
    # 200 steps with the trunk pressed against the wall (tools/c4_explore.py)
    sc._cable_amp = c.get("cable_amp", 2e-3)
    return sc


def drive_cables(scene, k):
    """Cable pattern of step k: the two +x cables pull towards the wall with a
    ramped, phase-shifted tension, the -x pair relaxes (2 mN per vertex)."""
    f = np.zeros(3 * scene.n_verts)
    a0 = getattr(scene, "_cable_amp", 2e-3)
    for ci, line in enumerate(scene._cable_lines):
        amp = a0 * min(1.0, (k + 1) / 10.0) * (1.0 + 0.5 * np.sin(0.3 * k + ci))
        sx = 1.0 if ci in (1, 3) else -0.25
        f[3 * line] += sx * amp
    scene.fext = f
    return f


def fold_targets(scene, k, lift=2e-3):
    """C2 fold: targets of the bound edge at step k = that edge of the sheet
    rigidly folded about x = size/2 by th(k) = pi min(1, (k+1)/fold), lifted
    by `lift` near the crease (tools/c2_fold_explore.py)."""
    size, fold = scene._fold
    th = np.pi * min(1.0, (k + 1) / fold)
    v = scene.vertices
    xc = 0.5 * size
    for b in scene.bindings:
        x = v[b.vertex]
        d = x[0] - xc
        b.target = np.array([xc + d * np.cos(th), x[1], x[2] + d * np.sin(th) + lift * min(1.0, d / (0.1 * size))])


def finger_offset(scene, k):
    """How far each finger has closed at finger index k (m)."""
    speed, hold = getattr(scene, "_finger_schedule", (2e-5, None))
    return speed * (k if hold is None else min(k, hold))


def move_fingers(scene, k):
    """Kinematic fingers at finger index k (host-side; colliders are re-read
    every step as in contact.py:125-127); C4: cable forces."""
    if getattr(scene, "_cable_lines", None) is not None:
        drive_cables(scene, k)
        return
    if getattr(scene, "_fold", None) is not None:
        fold_targets(scene, k)
        return
    if len(scene.colliders) < 3:
        return
    lx = scene.vertices[:, 0].max()
    p = finger_offset(scene, k)
    scene.colliders[1].center[0] = -0.02 - 5e-4 + p
    scene.colliders[2].center[0] = lx + 0.02 + 5e-4 - p


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    """SM clock + throttle reasons sampled with NVML (in-process thread, every
    250 ms) during the timed region.  Spawning nvidia-smi inside the timed
    region was measured to perturb the step time."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.thread = None

    def __enter__(self):
        if os.environ.get("BENCH_NO_CLOCKS"):
            return self
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for name, bit in self.REASONS.items():
                            if r & bit:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    self._stop.wait(0.25)

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        sm = self.samples
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(sm), "source": "NVML, 250 ms"}


# ---------------------------------------------------------------------------
# GPU arm


try:   # the process's CPU set before any thread pins itself
    _ALL_CPUS = sorted(os.sched_getaffinity(0))
except AttributeError:
    _ALL_CPUS = list(range(os.cpu_count() or 1))


def _pin_thread(local_rank, slot):
    """Pin the calling thread to one core (the Newton driver spin-waits on
    ~100 device synchronisations per step; migrations show up as jitter).
    The cores are split into one contiguous block per local rank
    (LOCAL_WORLD_SIZE ranks on the node), so spinning drivers of different
    ranks never share a core."""
    if os.environ.get("BENCH_NO_PIN"):
        return
    try:
        cpus = _ALL_CPUS
        nloc = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
        block = max(1, len(cpus) // nloc)
        base = (local_rank % nloc) * block
        os.sched_setaffinity(0, {cpus[base + (2 * slot + 1) % block]})
    except (AttributeError, OSError, IndexError):
        pass


def gpu_arm(args, rank, world, local_rank):
    import ctypes as C
    from concurrent.futures import ThreadPoolExecutor

    import torch
    import torch.distributed as dist

    from paper_2603_16478_b200 import _lib, adjoint as aj, core, forward as fw
    from paper_2603_16478_b200.parallel import allreduce_gradients, pack_gradients

    torch.cuda.set_device(local_rank)
    cdef = CONFIGS[args.config]
    R = args.rollouts or cdef["rollouts"]
    K, W = args.steps, args.warmup
    dd = dict(device="cuda:%d" % local_rank, dtype=torch.float64)
    cfg = fw.ForwardConfig(tol=cdef["tol"])
    if os.environ.get("BENCH_ETA"):          # diagnostics: Newton forcing term
        cfg.lin_rtol_max = cfg.lin_rtol_min = float(os.environ["BENCH_ETA"])
    # adjoint: the reference's tolerance (1e-10) and iteration cap; GMRES(20)
    # instead of the default restart length 50: with the V-cycle the solve
    # needs ~60-70 iterations either way and the shorter Gram-Schmidt
    # recurrences make each one cheaper (measured -10% adjoint time at C5)
    adj_cfg = aj.SolverConfig(tol=1e-10, max_iter=2000, gmres_restart=ADJ_RESTART)
    scfg = adj_cfg.to_c()

    class Ctx:
        pass

    # one rollout per (rank, slot): candidate E = E0 (1 + 0.05 * global index)
    t_setup = time.perf_counter()
    ctxs = []
    for i in range(R):
        c = Ctx()
        c.slot = i
        g_idx = rank * R + i
        if cdef.get("vary", "E") == "E":
            c.E = E_YOUNG * (1 + 0.05 * g_idx)
            c.target_shift = 1e-3
        else:
            # same material on every rank, a different synthetic target per
            # rollout (C5: E candidates move the scene into the reference
            # model's friction-rotation stall within 6 steps)
            c.E = E_YOUNG
            c.target_shift = 1e-3 * (1 + 0.1 * g_idx)
        c.scene = make_scene(args.config, E=c.E)
        c.sysmat = core.assemble_system_matrix(c.scene, device=local_rank)
        c.dev = c.sysmat.dev
        c.L = c.dev.lib
        c.stream = torch.cuda.ExternalStream(c.L.dp_scene_stream(c.dev.handle))
        ctxs.append(c)
    setup_s = time.perf_counter() - t_setup
    info = ctxs[0].dev.info()
    scene0 = ctxs[0].scene
    V, E_ = scene0.n_verts, len(scene0.elements)
    n3 = 3 * V

    def device_rollout(c, nsteps, k0):
        """forward K steps + reverse sweep of one rollout, device-resident."""
        _pin_thread(local_rank, c.slot)
        L, dev, scene = c.L, c.dev, c.scene
        with torch.cuda.stream(c.stream):
            q = [torch.empty(n3, **dd) for _ in range(nsteps + 1)]
            v = [torch.empty(n3, **dd) for _ in range(nsteps + 1)]
            q[0].copy_(torch.from_numpy(scene.vertices.reshape(-1)))
            v[0].zero_()
        c.stream.synchronize()
        caches, stats = [], []
        trace = [] if os.environ.get("BENCH_TRACE") else None
        for k in range(nsteps):
            if trace is not None:
                trace.append(time.perf_counter())
            move_fingers(scene, k0 + k)
            _, rep = fw.forward_step(scene, None, c.sysmat, cfg,
                                     device_io=dict(q_bar=q[k], v_bar=v[k], q_out=q[k + 1], v_out=v[k + 1]))
            if not rep.converged:   # forward.py:261-264 (rollout raises)
                raise RuntimeError(f"forward step {k} did not converge (residual {rep.residual_history[-1]:.3e})")
            caches.append(rep.cache)
            stats.append((rep.converged, rep.iterations, rep.krylov_iterations, rep.n_contacts))
        with torch.cuda.stream(c.stream):
            target = q[0] + c.target_shift   # synthetic target shape
            dq = 2.0 * (q[nsteps] - target)
            dv = torch.zeros(n3, **dd)
            z = torch.empty(n3, **dd)
            dqb = torch.empty(n3, **dd)
            dvb = torch.empty(n3, **dd)
            dfx = torch.empty((nsteps, n3), **dd)   # the controls' gradient of every step
        c.stream.synchronize()
        _lib.check(L.dp_grads_reset(dev.handle))
        adj_iters = 0
        for k in range(nsteps, 0, -1):
            h = caches[k - 1]._dc.handle
            _lib.check(L.dp_adjoint_assemble(dev.handle, h, None))
            rep = _lib.SolveReportC()
            _lib.check(L.dp_adjoint_solve(dev.handle, h, _lib.ptr(dq), _lib.ptr(dv), _lib.PTR_DEVICE,
                                          C.byref(scfg), _lib.ptr(z), C.byref(rep)))
            adj_iters += rep.iterations
            _lib.check(L.dp_backprop_step(dev.handle, h, _lib.ptr(z), _lib.ptr(dv), _lib.PTR_DEVICE,
                                          _lib.ptr(dqb), _lib.ptr(dvb), _lib.ptr(dfx[k - 1])))
            dq, dqb = dqb, dq
            dv, dvb = dvb, dv
        if trace is not None:
            trace.append(time.perf_counter())
            print("[trace] step ms", [round(1e3 * (b - a), 1) for a, b in zip(trace, trace[1:])],
                  file=sys.stderr, flush=True)
        # the full GradientReport stays on the device:
        # dL/dw, dL/dE_b, dL/dd_b, dL/dfext[K], dL/dq_bar, dL/dv_bar
        with torch.cuda.stream(c.stream):
            grads = aj.device_gradient_report(dev, scene, dd["device"])
            grads.dL_dfext = dfx
            grads.dL_dqbar = dq
            grads.dL_dvbar = dv
        if trace is not None:
            t_fold = time.perf_counter()
        with torch.cuda.stream(c.stream):
            loss = float(torch.sum((q[nsteps] - target) ** 2))
        c.q_final = q[nsteps]
        if trace is not None:
            print(f"[trace] fold {1e3 * (t_fold - trace[-1]):.1f} ms, loss {1e3 * (time.perf_counter() - t_fold):.1f} ms",
                  file=sys.stderr, flush=True)
        return grads, loss, stats, adj_iters

    def host_rollout(c, nsteps, k0):
        """the same through the public API with host NumPy buffers (e2e)."""
        _pin_thread(local_rank, c.slot)
        scene = c.scene
        st0 = scene.rest_state()
        st, caches = st0, []
        trace = [] if os.environ.get("BENCH_TRACE") else None
        for k in range(nsteps):
            if trace is not None:
                trace.append(time.perf_counter())
            move_fingers(scene, k0 + k)
            st, rep = fw.forward_step(scene, st, c.sysmat, cfg)
            if not rep.converged:   # forward.py:261-264 (rollout raises)
                raise RuntimeError(f"forward step {k} did not converge (residual {rep.residual_history[-1]:.3e})")
            caches.append(rep.cache)
        target = st0.q + c.target_shift
        if trace is not None:
            trace.append(time.perf_counter())
        g = aj.backprop_rollout(caches, target, solver_cfg=adj_cfg)
        if trace is not None:
            trace.append(time.perf_counter())
            print("[trace] e2e step ms", [round(1e3 * (b - a), 1) for a, b in zip(trace, trace[1:])],
                  file=sys.stderr, flush=True)
        return g, float(np.sum((st.q - target) ** 2))

    pool = ThreadPoolExecutor(max_workers=R)

    def run_all(fn, *a):
        if R == 1:
            return [fn(ctxs[0], *a)]
        return list(pool.map(lambda c: fn(c, *a), ctxs))

    def pack_sum(results):
        """Sum of this rank's packed gradients (scalars + every array block,
        SURVEY.md §8(e)); summed in the rollouts' fixed order."""
        tot = None
        for g, loss in results:
            v = pack_gradients(g, loss, dd["device"], blocks=PACK_BLOCKS)
            tot = v if tot is None else tot + v
        return tot

    # warm-up (untimed): the same K-step rollouts + reverse sweeps as timed,
    # at least W of them and at least --warmup-seconds of wall time (a freshly
    # leased box shows 2-4x step-time noise for its first ~2 s of GPU work,
    # then settles to within 0.5%: measured, tools/var_c3.py)
    t_w = time.perf_counter()
    n_w = 0
    gw = None
    while n_w < max(W, 0) or time.perf_counter() - t_w < args.warmup_seconds:
        res = run_all(device_rollout, K, FINGER_K0)
        # the timed region's gradient packing runs here too, so its device
        # allocation comes from torch's cache, not a cudaMalloc inside the
        # timed region (measured: 60-80 ms stalls on a fresh box)
        gw = pack_sum([(r[0], r[1]) for r in res])
        n_w += 1
    # one all-reduce on every rank (the time-based warm-up count differs
    # between ranks; collectives must pair up): initialises NCCL and warms
    # its buffers before the timed region
    if gw is not None:
        allreduce_gradients(gw, world)
    torch.cuda.synchronize()
    if os.environ.get("BENCH_DEBUG"):
        for i in range(int(os.environ.get("BENCH_DEBUG_REPS", "3"))):
            t0 = time.perf_counter(); run_all(device_rollout, K, FINGER_K0); torch.cuda.synchronize()
            t1 = time.perf_counter(); run_all(host_rollout, K, FINGER_K0); torch.cuda.synchronize()
            t2 = time.perf_counter()
            print(f"[bench] device path {1e3 * (t1 - t0):.1f} ms, host path {1e3 * (t2 - t1):.1f} ms",
                  file=sys.stderr, flush=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    for c in ctxs:
        c.L.dp_scene_reset_timing(c.dev.handle)
    # host hygiene: no cyclic-GC pass inside the timed region (a full
    # collection walks the ~10^6 objects of torch/scipy/numpy: tens of ms)
    gc.collect()
    gc.freeze()
    gc.disable()
    with ClockSampler(local_rank) as clk:
        ev0.record()
        tw0 = time.perf_counter()
        res = run_all(device_rollout, K, FINGER_K0)
        tw1 = time.perf_counter()
        gvec = pack_sum([(r[0], r[1]) for r in res])
        allreduce_gradients(gvec, world)      # one all-reduce per optimisation iteration
        torch.cuda.synchronize()
        ev1.record()
        ev1.synchronize()
        tw2 = time.perf_counter()
    if os.environ.get("BENCH_TRACE"):
        print(f"[trace] timed: rollouts {1e3 * (tw1 - tw0):.1f} ms, pack+allreduce+sync {1e3 * (tw2 - tw1):.1f} ms",
              file=sys.stderr, flush=True)
    gc.enable()
    g_dE, g_loss = float(gvec[1]), float(gvec[0])
    del gvec, gw                # the packed vectors' device memory goes back to the caching allocator
    ms = ev0.elapsed_time(ev1)
    launches = sum(int(c.L.dp_scene_launch_count(c.dev.handle)) for c in ctxs)
    host_syncs = sum(int(c.L.dp_scene_host_sync_count(c.dev.handle)) for c in ctxs)
    t = torch.tensor([ms], device=dd["device"])
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    stats = res[0][2]
    adj_iters = res[0][3]

    # in-situ kernel times (the roofline's "average launch duration over the
    # timed region"): one more rollout of exactly the timed workload with a
    # CUDA event pair around every launch of the instrumented kernels on the
    # scene stream (no per-launch host sync; resolved afterwards).  Kept out
    # of the timed rollout so the events do not perturb the headline number.
    c0 = ctxs[0]
    kt = None
    if not args.skip_insitu:
        _lib.check(c0.L.dp_scene_enable_timing(c0.dev.handle, 1))
        _lib.check(c0.L.dp_scene_reset_timing(c0.dev.handle))
        device_rollout(c0, K, FINGER_K0)
        kt = _lib.KernelTimes()
        _lib.check(c0.L.dp_scene_get_timing(c0.dev.handle, C.byref(kt)))
        _lib.check(c0.L.dp_scene_enable_timing(c0.dev.handle, 0))
        kt = {f: getattr(kt, f) for f, _ in kt._fields_}
    # standalone (cold-operand) kernel loops, for comparison
    # roofline: dominant kernel = the SELL-32 BSR SpMV of the Krylov solves
    x = torch.randn(n3, **dd)
    y = torch.empty(n3, **dd)
    torch.cuda.synchronize()
    fms = C.c_float()
    reps = 30
    _lib.check(c0.L.dp_bench_spmv(c0.dev.handle, 1, _lib.ptr(x), _lib.ptr(y), 10, C.byref(fms)))
    _lib.check(c0.L.dp_bench_spmv(c0.dev.handle, 1, _lib.ptr(x), _lib.ptr(y), reps, C.byref(fms)))
    spmv_ms = fms.value / reps
    # the dominant kernel of the step (launch-list share): one fine-level
    # V-cycle smoothing sweep on the FP32 operator copy
    smooth_ms = None
    b_ = torch.randn(n3, **dd)
    o_ = torch.empty(n3, **dd)
    if c0.L.dp_bench_smoother(c0.dev.handle, _lib.ptr(x), _lib.ptr(b_), _lib.ptr(o_), 10, C.byref(fms)) == 0:
        _lib.check(c0.L.dp_bench_smoother(c0.dev.handle, _lib.ptr(x), _lib.ptr(b_), _lib.ptr(o_), reps, C.byref(fms)))
        smooth_ms = fms.value / reps
    # second roofline: the FP64-bound element kernel (projection + residual,
    # and with the Jacobian blocks) at the final state of the timed rollout
    elem = None
    if c0.dev.verts_per_elem == 4:
        elem = {}
        for jac, flops in ((1, ELEM_FLOPS_JAC), (0, ELEM_FLOPS_RES)):
            _lib.check(c0.L.dp_bench_elements(c0.dev.handle, _lib.ptr(c0.q_final), jac, 2, C.byref(fms)))
            _lib.check(c0.L.dp_bench_elements(c0.dev.handle, _lib.ptr(c0.q_final), jac, 10, C.byref(fms)))
            elem[jac] = (fms.value / 10, flops * E_ / (fms.value / 10 * 1e-3) / 1e12)
    nnzb = info.nnzb
    spmv_bytes = 76 * nnzb + 4 * (V + 1) + 48 * V
    # smoother sweep: FP32 block 36 B + column 4 B per nonzero block; x (gathered,
    # once), b, out 24 B/row each; FP32 3x3 block-Jacobi inverse 36 B/row
    sbb = int(getattr(info, "smoother_bytes_per_block", 0) or 40)   # 26 with the FP16 operator copy
    smooth_bytes = sbb * nnzb + 4 * (V + 1) + 108 * V
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    achieved = spmv_bytes / (spmv_ms * 1e-3) / 1e9
    traffic = smooth_traffic = None
    prof = os.path.join(ROOT, "profiles", f"spmv_traffic_{args.config}.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            traffic = pj.get("dram_bytes_per_launch")
            smooth_traffic = pj.get("smoother_dram_bytes_per_launch")
        except ValueError:
            traffic = None

    # e2e through the public API with host buffers
    e2e = None
    if not args.skip_e2e:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # warm-up of the public-API path (untimed, like the device path's
        # warm-up): its first packing of host gradients into the all-reduce
        # vector otherwise pays the caching allocator's cudaMalloc of the
        # ~100 MB packed vector inside the timed region (measured 14-430 ms)
        for _ in range(max(1, int(os.environ.get("BENCH_E2E_PRE", "1")))):
            tp = time.perf_counter()
            allreduce_gradients(pack_sum(run_all(host_rollout, K, FINGER_K0)), world)
            torch.cuda.synchronize()
            if os.environ.get("BENCH_TRACE"):
                print(f"[trace] e2e warm-up {1e3 * (time.perf_counter() - tp):.1f} ms", file=sys.stderr, flush=True)
        if not os.environ.get("BENCH_E2E_NOGC"):
            gc.collect()
        gc.disable()
        t0 = time.perf_counter()
        res2 = run_all(host_rollout, K, FINGER_K0)
        t1 = time.perf_counter()
        allreduce_gradients(pack_sum(res2), world)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if os.environ.get("BENCH_TRACE"):
            print(f"[trace] e2e: rollouts {1e3 * (t1 - t0):.1f} ms, pack+allreduce {1e3 * (wall - (t1 - t0)):.1f} ms",
                  file=sys.stderr, flush=True)
        gc.enable()
        tw = torch.tensor([wall], device=dd["device"])
        if world > 1:
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        wall = float(tw.item())
        # per step: forward q_bar, v_bar up and q, v down; reverse sweep
        # dL/dfext down (the adjoint chain stays on the device); once per
        # rollout: the loss gradient up, q_new/q_bar (loss) and dL/dq_bar,
        # dL/dv_bar down
        # + the packed gradient (host arrays of the public API) going up for
        # the all-reduce: 5 + E + 4B + (K + 2) 3V doubles per rollout
        nb = len(scene0.bindings)
        pack_bytes = 8 * (5 + E_ + 4 * nb + (K + 2) * n3)
        h2d = (2 * n3) * 8 + (2 * n3 * 8 + pack_bytes) // K
        d2h = (2 * n3 + n3) * 8 + (4 * n3 * 8) // K
        e2e = {"value": world * R * K / wall, "unit": "steps/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h}
    pool.shutdown()
    conv = [s_[0] for r in res for s_ in r[2]]
    return dict(ms=ms_max, launches=launches, host_syncs=host_syncs, clocks=clk.summary(), spmv_ms=spmv_ms, spmv_bytes=spmv_bytes, kt=kt,
                achieved=achieved, hbm=hbm, traffic=traffic, e2e=e2e, setup_s=setup_s, R=R, elem=elem,
                smooth_ms=smooth_ms, smooth_bytes=smooth_bytes, smooth_traffic=smooth_traffic, sbb=sbb,
                fp64_peak=float(peaks.get("fp64_tflops", FP64_PEAK_TFLOPS)),
                nnzb=nnzb, V=V, E=E_, desc=cdef["desc"], newton=[s_[1] for s_ in stats],
                krylov=[s_[2] for s_ in stats], contacts=[s_[3] for s_ in stats], converged=all(conv),
                adj_iters=adj_iters, dE=g_dE, loss=g_loss, device_bytes=info.device_bytes)


# ---------------------------------------------------------------------------
# CPU oracle (reported baseline / reference arm)


def sample_scene(config, n_cells):
    """The bounded CPU sample of a workload: the same scene family at
    n_cells per side (C5: c5_family with mass-scaled eps_fb / tolerance; C1:
    the C1 cube itself when n_cells == 9), its Newton tolerance and finger
    schedule."""
    c = CONFIGS[config]
    if config.startswith("c5"):
        fam = c5_family(n_cells)
        if config == "c5f":
            fam.update(mu=c["mu"], eps_fb=c["eps_fb"] * (55.0 / n_cells) ** 3)
        return make_scene(fam), fam["tol"]
    if config in ("c1", "c1b"):
        fam = dict(c, cells=(n_cells,) * 3, edge=0.1 / n_cells)
        return make_scene(fam), c["tol"]
    raise ValueError(f"no CPU sample defined for config {config}")


def _oracle_sample(config, n_cells, steps, warmup=0):
    """One process: the oracle port (reference semantics, exact SuperLU Newton
    solves, Jacobi-preconditioned CG/GMRES adjoint) on the bounded sample:
    `warmup` untimed + `steps` timed fwd steps over the bench schedule, then
    the timed reverse sweep.  Returns (seconds per fwd+bwd step, tets,
    newton iterations)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import diffproj_oracle as O
    from paper_2603_16478_b200 import core
    scene, tol = sample_scene(config, n_cells)
    osc = O.OScene(core.scene_to_arrays(scene))
    els = O.build_elements(osc)
    A = O.assemble_A(osc, els)
    q = scene.vertices.reshape(-1).copy()
    v = np.zeros_like(q)
    its, sts = [], []
    t0 = None
    for k in range(warmup + steps):
        if k == warmup:
            t0 = time.perf_counter()
        move_fingers(scene, FINGER_K0 + k)
        osc = O.OScene(core.scene_to_arrays(scene))
        st = O.forward_step(osc, A, els, q, v, O.ForwardConfig(tol=tol))
        if not st.converged:
            raise RuntimeError(f"oracle step {k} did not converge ({st.residual_history[-1]:.3e})")
        if k >= warmup:
            sts.append(st)
            its.append(st.iterations)
        q, v = st.q_new, st.v_new
    O.backprop_rollout(osc, els, A, sts, target=scene.vertices.reshape(-1) + 1e-3)
    dt = time.perf_counter() - t0
    return dt / steps, len(scene.elements), its


def _oracle_worker(args):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    return _oracle_sample(*args)


def cpu_baseline(config, n_tets_target, n_cells, steps, procs=1, warmup=0):
    """Bounded CPU sample; returns the cpu_baseline object.  `value` is the
    measured rate scaled linearly in tets to the workload size (the metric's
    unit; generous to the CPU: SuperLU fill grows faster than linearly);
    the measured numbers are in the measured_* fields."""
    t0 = time.perf_counter()
    if procs <= 1:
        sec, tets, its = _oracle_sample(config, n_cells, steps, warmup)
        per_proc = [sec]
    else:
        import multiprocessing as mp
        ctx = mp.get_context("spawn")
        with ctx.Pool(procs) as pool:
            res = pool.map(_oracle_worker, [(config, n_cells, steps, warmup)] * procs)
        per_proc = [r[0] for r in res]
        tets, its = res[0][1], res[0][2]
    wall = time.perf_counter() - t0
    measured_rate = sum(1.0 / s for s in per_proc)          # fwd+bwd steps/s at the sample size
    rate = measured_rate * tets / n_tets_target
    return {"value": rate, "unit": "steps/s", "cores": procs, "kind": "port",
            "value_basis": f"measured rate at {tets} tets scaled linearly to {n_tets_target} tets",
            "measured_tets": tets, "measured_steps": steps, "measured_processes": procs,
            "measured_s_per_step": float(np.mean(per_proc)), "measured_steps_per_s": measured_rate,
            "measured_tet_steps_per_s_M": measured_rate * tets / 1e6, "measured_newton_iterations": its,
            "wall_s": wall,
            "sample": (f"oracle port (oracle/diffproj_oracle.py: reference algorithm, NumPy + SuperLU Newton "
                       f"solves, Jacobi-Krylov adjoint) on the same scene family at {n_cells}^3 cells "
                       f"({tets} tets), {warmup} untimed + {steps} timed fwd steps of the bench schedule + "
                       f"their reverse sweep, x {procs} process(es), 1 BLAS thread each")}


# ---------------------------------------------------------------------------


def _frac(bytes_, ms, peak):
    ach = bytes_ / (ms * 1e-3) / 1e9
    return ach, ach / peak


def roofline_smoother(r):
    """Dominant kernel of the step (launch-list share): the fine-level V-cycle
    sweep k_mg_smooth<float,1,*> on the FP32 SELL-32 operator copy.
    Algorithmic bytes per launch: per nonzero block the
    operator copy's 18 B FP16 values + 4 B scale + 4 B column (26 B; 40 B
    with the FP32 copy, DP_SMOOTH16=0), slice table 4(V+1); per row the residual-form sweep
    reads x (gathered, counted once) and b and writes r (72 B), the update
    form reads x, b, the FP32 block-Jacobi inverse (36 B) and agg (4 B) and
    writes z (112 B); a V-cycle runs one of each, so 92 B/row on average.
    `achieved` uses the in-situ average launch time (CUDA events over a
    rollout of the timed workload); the standalone loop (same kernel
    repeated on cold operands, update form) is reported beside it."""
    nnzb, V, hbm = r["nnzb"], r["V"], r["hbm"]
    out = {"bound": "hbm", "unit": "GB/s", "peak": hbm,
           "kernel": "k_mg_smooth16 / k_mg_smooth<float,1> (fine-level V-cycle sweep, SELL-32 FP16(+scale) or FP32 "
                     "3x3 blocks, cp.async ring)",
           "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"}
    kt = r.get("kt")
    if kt and kt["smooth_calls"]:
        ms = kt["smooth_ms"] / kt["smooth_calls"]
        b = r["sbb"] * nnzb + 4 * (V + 1) + 92 * V
        ach, fr = _frac(b, ms, hbm)
        out.update(achieved=ach, frac=fr, ms_per_launch=ms, bytes_per_launch=b, launches=kt["smooth_calls"],
                   bytes_per_block=r["sbb"],
                   timing="in situ: CUDA event pairs around every launch of one rollout of the timed workload",
                   traffic=r["smooth_traffic"])
    if r["smooth_ms"]:
        b = r["smooth_bytes"]
        ach, fr = _frac(b, r["smooth_ms"], hbm)
        out["standalone"] = {"achieved": ach, "frac": fr, "ms_per_launch": r["smooth_ms"], "bytes_per_launch": b,
                             "timing": "30 back-to-back launches of the update-form sweep"}
        if "achieved" not in out:
            out.update(achieved=ach, frac=fr, ms_per_launch=r["smooth_ms"], bytes_per_launch=b,
                       traffic=r["smooth_traffic"])
    return out


def roofline_spmv(r):
    """The Krylov SpMVs: the PCG's fused p-update + SpMV on the FP32 operator
    copy (in situ; 40 B per block + p, z gathered and p', q written: 96 B per
    row) and the FP64 SELL-32 SpMV k_spmv (standalone loop; 76 B per block,
    SURVEY.md §8(d))."""
    nnzb, V, hbm = r["nnzb"], r["V"], r["hbm"]
    out = {"bound": "hbm", "unit": "GB/s", "peak": hbm,
           "kernel": "k_spmv (SELL-32 3x3-BSR FP64 SpMV; k_gm_spmvdot_r / k_pcg_spmv_p are this SpMV + fusions)",
           "achieved": r["achieved"], "frac": r["achieved"] / hbm, "traffic": r["traffic"],
           "bytes_per_launch": r["spmv_bytes"], "ms_per_launch": r["spmv_ms"], "timing": "standalone loop",
           "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"}
    kt = r.get("kt")
    if kt and kt["pcg_spmv_calls"]:
        ms = kt["pcg_spmv_ms"] / kt["pcg_spmv_calls"]
        b = 40 * nnzb + 4 * (V + 1) + 96 * V
        ach, fr = _frac(b, ms, hbm)
        out["pcg_fused_insitu"] = {"kernel": "k_pcg_spmv_p (FP32 operator, forward PCG; FP64 for the adjoint)",
                                   "achieved": ach, "frac": fr, "ms_per_launch": ms, "bytes_per_launch_fp32": b,
                                   "launches": kt["pcg_spmv_calls"],
                                   "note": "average over the FP32 (forward) and FP64 (adjoint) launches; bytes "
                                           "counted for the FP32 form, so the FP64 share understates achieved"}
    return out


def roofline_fp64(r, E_tets):
    if not r["elem"]:
        return None
    out = {"bound": "fp64", "kernel": "k_elements<4,JAC> (per-tet SVD + NH projection + 10 Hessian blocks)",
           "achieved": r["elem"][1][1], "peak": r["fp64_peak"], "unit": "TFLOP/s",
           "frac": r["elem"][1][1] / r["fp64_peak"], "ms_per_launch": r["elem"][1][0],
           "flops_per_tet": ELEM_FLOPS_JAC, "timing": "standalone loop at the final state",
           "residual_only": {"achieved": r["elem"][0][1], "ms_per_launch": r["elem"][0][0],
                             "flops_per_tet": ELEM_FLOPS_RES},
           "peak_source": "profiles/r01_fp64_peak.json (measured DFMA loop)",
           "flops_source": "ncu 2*DFMA+DMUL+DADD thread instructions per tet at a C5 state "
                           "(profiles/r01_elements_fp64.md)"}
    kt = r.get("kt")
    if kt and kt["elem_jac_calls"]:
        ms = kt["elem_jac_ms"] / kt["elem_jac_calls"]
        out["insitu"] = {"ms_per_launch": ms, "launches": kt["elem_jac_calls"],
                         "achieved": ELEM_FLOPS_JAC * E_tets / (ms * 1e-3) / 1e12,
                         "frac": ELEM_FLOPS_JAC * E_tets / (ms * 1e-3) / 1e12 / r["fp64_peak"]}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0, help="steps per rollout (default per config: 6; c2 4)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-insitu", action="store_true", help="no in-situ kernel-timing rollout")
    ap.add_argument("--cpu-cells", type=int, default=0, help="cells/side of the cpu_baseline sample (c5: 8, c1: 9)")
    ap.add_argument("--cpu-steps", type=int, default=8, help="timed steps of the cpu_baseline sample")
    ap.add_argument("--ref-cells", type=int, default=10, help="cells/side of the --impl reference sample")
    ap.add_argument("--rollouts", type=int, default=0, help="rollouts per GPU (default per config)")
    ap.add_argument("--warmup-seconds", type=float, default=8.0)
    args = ap.parse_args()
    if args.cpu_cells <= 0:
        args.cpu_cells = 9 if args.config.startswith("c1") else 8
    if args.steps <= 0:
        # the reference's own Newton (oracle, exact LU) stops converging at
        # step 6 of the C2 drape (compressed ARAP cloth, tools/diag_cloth.py)
        args.steps = CONFIGS[args.config].get("steps", 6)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(1)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # functional smoke test of the N>1 code path on a 1-GPU box only (gloo,
    # every rank on cuda:0; never a measurement): BENCH_SMOKE_SHARED_GPU=1
    if os.environ.get("BENCH_SMOKE_SHARED_GPU"):
        local_rank = 0
    cdef = CONFIGS[args.config]
    R = args.rollouts or cdef["rollouts"]
    nx, ny, nz = cdef["cells"]
    cloth = bool(cdef.get("cloth"))
    n_tets = 2 * nx * ny if cloth else 6 * nx * ny * nz
    config = {"workload": f"{args.config}: {cdef['desc']}", ("n_tris" if cloth else "n_tets"): n_tets,
              "n_verts": (nx + 1) * (ny + 1) * (nz + 1 if not cloth else 1), "steps_per_rollout": args.steps,
              "rollouts_per_gpu": R, "rollouts": world * R,
              "parallelism": f"dp{world} x {R} rollouts/GPU (independent rollouts, NCCL grad allreduce)",
              "material": ("arap stiffness=50" if cloth else
                           (f"neohookean E={E_YOUNG}(1+0.05 i) nu={NU}" if cdef.get("vary", "E") == "E" else
                            f"neohookean E={E_YOUNG} nu={NU}, target shift 1e-3 (1 + 0.1 i) per rollout i")),
              "friction_mu": (0.0 if cdef.get("fold") else 0.3) if (cloth or cdef.get("trunk")) else cdef.get("mu", MU),
              "h": cdef.get("h", 0.01), "self_contact": bool(cdef.get("fold")),
              "finger_schedule": (f"close {FINGER_SPEED * 1e6:.0f} um/step up to finger index {FINGER_HOLD}, then "
                                  f"hold; every rollout starts at index {FINGER_K0}"
                                  if cdef.get("fingers") else None),
              "eps_fb": cdef["eps_fb"], "newton_tol": cdef["tol"], "adjoint_tol": 1e-10,
              "adjoint_gmres_restart": ADJ_RESTART, "l2": "operands > L2 (no flush)"}
    if args.impl == "reference":
        # the reference's algorithm on the host cores (oracle port; the
        # reference is pure Python and does not travel to the GPU box), one
        # process per core, each a bounded sample of the workload: W untimed
        # + K timed steps of the same finger schedule on a smaller cube of the
        # same family; only rank 0 runs (N>1: the other ranks exit)
        if rank != 0:
            return
        procs = os.cpu_count() or 1
        W, K = args.warmup, args.steps
        base = cpu_baseline(args.config, n_tets, n_cells=args.ref_cells, steps=K, procs=procs, warmup=W)
        line = {"metric": "fwd+bwd sim steps/sec at N tets", "value": base["value"], "unit": "steps/s",
                "n_gpus": args.gpus, "steps": K, "warmup": W,
                # what was actually timed: K steps per process at the sample size
                "ms_per_step": 1e3 * base["measured_s_per_step"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (procedural mesh)", "config": config, "impl": "reference",
                "value_basis": base["value_basis"],
                "measured_tets": base["measured_tets"], "measured_steps_per_s": base["measured_steps_per_s"],
                "tet_steps_per_s_M": base["measured_tet_steps_per_s_M"],
                "cpu_baseline": base,
                "e2e": {"value": base["value"], "unit": "steps/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0},
                "wall_s": base["wall_s"]}
        print(json.dumps(line))
        return

    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo" if os.environ.get("BENCH_SMOKE_SHARED_GPU") else "nccl")
    r = gpu_arm(args, rank, world, local_rank)
    if rank == 0:
        K = args.steps
        steps_total = world * R * K
        value = steps_total / (r["ms"] * 1e-3)
        line = {"metric": "fwd+bwd sim steps/sec at N tets", "value": value, "unit": "steps/s",
                "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": r["ms"] / K,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (procedural mesh, random-free)", "config": config,
                "tet_steps_per_s_M": value * n_tets / 1e6,
                "roofline": roofline_smoother(r),
                "roofline_spmv": roofline_spmv(r),
                "roofline_fp64": roofline_fp64(r, E_tets=n_tets),
                "kernel_times_insitu": r["kt"],
                "clocks": r["clocks"], "gpu_launches": r["launches"], "e2e": r["e2e"],
                "host_syncs_per_step": round(r["host_syncs"] / max(1, K * r["R"]), 1),   # fwd + bwd, per rollout step
                "newton_iterations": r["newton"], "krylov_iterations": r["krylov"],
                "adjoint_krylov_iterations": r["adj_iters"], "contacts": r["contacts"],
                "converged": r["converged"], "setup_s": r["setup_s"], "nnzb": r["nnzb"],
                "env_knobs": {k: v for k, v in sorted(os.environ.items()) if k.startswith("DP_")},
                "device_bytes": r["device_bytes"]}
        if not args.skip_cpu and world == 1:
            try:
                line["cpu_baseline"] = cpu_baseline(args.config, n_tets, n_cells=args.cpu_cells,
                                                    steps=min(args.cpu_steps, K), procs=1)
            except Exception as ex:   # the baseline must not kill the GPU line
                line["cpu_baseline"] = {"value": None, "error": repr(ex)[:200]}
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
