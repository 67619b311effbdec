"""ctypes binding of libdiffproj_b200.so (include/diffproj_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is visible, :func:`lib` raises ``RuntimeError`` with the reason.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DP_LIB") or os.path.join(_HERE, "libdiffproj_b200.so")

DP_OK = 0
DP_ERR_VALUE = 1
DP_ERR_INVERTED = 2
DP_ERR_PENETRATION = 3
DP_ERR_NH_STALL = 4
DP_ERR_NOT_CONVERGED = 5
DP_ERR_BREAKDOWN = 6
DP_ERR_CUDA = 7
DP_ERR_NO_DEVICE = 8

PTR_DEVICE = 0
PTR_HOST = 1

c_double_p = C.POINTER(C.c_double)
c_int32_p = C.POINTER(C.c_int32)
c_int64_p = C.POINTER(C.c_int64)


class SceneDesc(C.Structure):
    _fields_ = [("n_verts", C.c_int32), ("n_elems", C.c_int32),
                ("verts_per_elem", C.c_int32), ("device", C.c_int32),
                ("vertices", c_double_p), ("elements", c_int64_p),
                ("masses", c_double_p), ("mat_model", c_int32_p),
                ("mat_E", c_double_p), ("mat_nu", c_double_p),
                ("mat_stiffness", c_double_p), ("gravity", C.c_double * 3),
                ("h", C.c_double), ("eps_fb", C.c_double),
                ("contact_activation", C.c_double)]


class SceneInfo(C.Structure):
    _fields_ = [("n_verts", C.c_int32), ("n_elems", C.c_int32),
                ("verts_per_elem", C.c_int32), ("nnzb", C.c_int64),
                ("n_slots", C.c_int64), ("device_bytes", C.c_int64),
                ("n_colliders", C.c_int32), ("n_bindings", C.c_int32),
                ("smoother_bytes_per_block", C.c_int32), ("pad_", C.c_int32)]


class ForwardCfg(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int32),
                ("max_line_search", C.c_int32), ("pullback_margin", C.c_double),
                ("lin_rtol_max", C.c_double), ("lin_rtol_min", C.c_double),
                ("lin_max_iter", C.c_int32), ("gmres_restart", C.c_int32)]


class ForwardReportC(C.Structure):
    _fields_ = [("converged", C.c_int32), ("iterations", C.c_int32),
                ("n_contacts", C.c_int32), ("krylov_iterations", C.c_int32),
                ("line_search_trials", C.c_int32), ("symmetric", C.c_int32)]


class SolverCfgC(C.Structure):
    _fields_ = [("method", C.c_int32), ("tol", C.c_double),
                ("max_iter", C.c_int32), ("gmres_restart", C.c_int32)]


class SolveReportC(C.Structure):
    _fields_ = [("converged", C.c_int32), ("iterations", C.c_int32),
                ("rel_residual", C.c_double), ("symmetric", C.c_int32)]


class GradScalars(C.Structure):
    _fields_ = [("dL_dmu_friction", C.c_double), ("dL_dstiffness", C.c_double),
                ("dmu_lame", C.c_double), ("dlam_lame", C.c_double)]


class KernelTimes(C.Structure):
    _fields_ = [("spmv_ms", C.c_double), ("spmv_calls", C.c_int64),
                ("elem_jac_ms", C.c_double), ("elem_jac_calls", C.c_int64),
                ("elem_res_ms", C.c_double), ("elem_res_calls", C.c_int64),
                ("assemble_ms", C.c_double), ("assemble_calls", C.c_int64),
                ("smooth_ms", C.c_double), ("smooth_calls", C.c_int64),
                ("pcg_spmv_ms", C.c_double), ("pcg_spmv_calls", C.c_int64)]


_P = C.c_void_p
# name -> (restype, argtypes); every symbol declared in include/diffproj_b200.h
SIGNATURES = {
    "dp_last_error": (C.c_char_p, []),
    "dp_version": (C.c_char_p, []),
    "dp_device_count": (C.c_int, []),
    "dp_set_spin_wait": (C.c_int, [C.c_int32, C.c_int32]),
    "dp_scene_create": (C.c_int, [C.POINTER(SceneDesc), C.POINTER(_P)]),
    "dp_scene_destroy": (C.c_int, [_P]),
    "dp_scene_get_info": (C.c_int, [_P, C.POINTER(SceneInfo)]),
    "dp_scene_set_colliders": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P]),
    "dp_scene_set_bindings": (C.c_int, [_P, C.c_int32, _P, _P, _P]),
    "dp_scene_set_fext": (C.c_int, [_P, _P, C.c_int32]),
    "dp_scene_set_params": (C.c_int, [_P, C.c_double, C.c_double, C.c_double, _P]),
    "dp_scene_set_solver_options": (C.c_int, [_P, C.c_int32, C.c_double, C.c_int32]),
    "dp_scene_set_materials": (C.c_int, [_P, _P, _P, _P]),
    "dp_pinned_alloc": (C.c_int, [C.c_int64, C.POINTER(C.c_void_p)]),
    "dp_pinned_free": (C.c_int, [_P]),
    "dp_scene_set_self_contact": (C.c_int, [_P, C.c_int32, _P, C.c_double, C.c_int32]),
    "dp_self_contact_query": (C.c_int, [_P, _P, _P, C.c_int32, _P, _P, _P, _P]),
    "dp_scene_get_mg_levels": (C.c_int, [_P, c_int32_p, _P, C.c_int32]),
    "dp_scene_get_element_data": (C.c_int, [_P, _P, _P]),
    "dp_scene_export_bsr": (C.c_int, [_P, C.c_int32, _P, _P, _P]),
    "dp_forward_cfg_default": (None, [C.POINTER(ForwardCfg)]),
    "dp_forward_step": (C.c_int, [_P, _P, _P, C.c_int32, C.POINTER(ForwardCfg), _P, _P,
                                  _P, C.POINTER(ForwardReportC), _P, C.c_int32]),
    "dp_cache_create": (C.c_int, [_P, C.POINTER(_P)]),
    "dp_cache_destroy": (C.c_int, [_P]),
    "dp_cache_n_contacts": (C.c_int, [_P, c_int32_p]),
    "dp_cache_get_contacts": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "dp_cache_get_states": (C.c_int, [_P, _P, _P, _P, _P]),
    "dp_cache_get_projections": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "dp_solver_cfg_default": (None, [C.POINTER(SolverCfgC)]),
    "dp_adjoint_assemble": (C.c_int, [_P, _P, c_int32_p]),
    "dp_adjoint_solve": (C.c_int, [_P, _P, _P, _P, C.c_int32, C.POINTER(SolverCfgC), _P,
                                   C.POINTER(SolveReportC)]),
    "dp_backprop_step": (C.c_int, [_P, _P, _P, _P, C.c_int32, _P, _P, _P]),
    "dp_grads_reset": (C.c_int, [_P]),
    "dp_grads_get": (C.c_int, [_P, C.POINTER(GradScalars)]),
    "dp_grads_get_arrays": (C.c_int, [_P, _P, _P, _P]),
    "dp_project_batch": (C.c_int, [C.c_int32, C.c_int32, _P, _P, _P, _P, C.c_double, _P, _P,
                                   _P, _P, _P, _P, _P, _P]),
    "dp_contact_batch": (C.c_int, [C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                   _P, _P]),
    "dp_detect_contacts": (C.c_int, [_P, _P, C.c_int32, C.c_int32, c_int32_p, _P, _P, _P, _P]),
    "dp_bench_spmv": (C.c_int, [_P, C.c_int32, _P, _P, C.c_int32, C.POINTER(C.c_float)]),
    "dp_bench_elements": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.POINTER(C.c_float)]),
    "dp_bench_smoother": (C.c_int, [_P, _P, _P, _P, C.c_int32, C.POINTER(C.c_float)]),
    "dp_scene_enable_timing": (C.c_int, [_P, C.c_int32]),
    "dp_scene_get_timing": (C.c_int, [_P, C.POINTER(KernelTimes)]),
    "dp_scene_reset_timing": (C.c_int, [_P]),
    "dp_scene_launch_count": (C.c_int64, [_P]),
    "dp_scene_host_sync_count": (C.c_int64, [_P]),
    "dp_scene_stream": (_P, [_P]),
    "dp_scene_synchronize": (C.c_int, [_P]),
}

_lock = threading.Lock()
_lib = None


def load(path=LIB_PATH):
    """Load the shared library and declare every ABI symbol (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"libdiffproj_b200.so not found at {path}; run "
                    "`python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            lib_ = C.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib_, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib_
    return _lib


def lib():
    """The loaded library, asserting that a CUDA device is present."""
    L = load()
    if L.dp_device_count() <= 0:
        raise RuntimeError("diffproj_b200 needs a CUDA GPU (B200); none is "
                           "visible and there is no CPU fallback")
    return L


def last_error():
    return load().dp_last_error().decode()


def check(rc):
    """Map a dp_status to the reference's exception types."""
    if rc == DP_OK:
        return
    msg = last_error()
    if rc in (DP_ERR_VALUE, DP_ERR_INVERTED, DP_ERR_PENETRATION):
        raise ValueError(msg)
    if rc in (DP_ERR_NH_STALL, DP_ERR_NOT_CONVERGED, DP_ERR_BREAKDOWN):
        raise RuntimeError(msg)
    raise RuntimeError(f"diffproj_b200 error {rc}: {msg}")


def ptr(a):
    """Raw pointer of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()   # torch tensor


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)
