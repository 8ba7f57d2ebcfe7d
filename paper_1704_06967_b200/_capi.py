"""ctypes declarations of include/pba_gpu.h and the loader of the product library.

``backend("gpu")`` binds ``lib/libpba_gpu.so`` (prefix ``pba_gpu_``); it fails loudly when the
library has not been built — there is no CPU fallback and this package loads no other library.
``_COMMON`` is the call set of the C ABI; the test suite binds its CPU checkers
(tests/_oracle.py) with the same declarations and hands them to ``solver.Handle`` as library
objects, so the parity tests drive every implementation through identical calls.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
REPO = _PKG.parent
GPU_LIB = Path(os.environ.get("PBA_GPU_LIB", str(_PKG / "lib" / "libpba_gpu.so")))  # override: experiments only

# status codes (pba_gpu.h)
PBA_OK = 0
PBA_E_EMPTY_PROBLEM = 1
PBA_E_OUT_OF_BOUNDS = 2
PBA_E_INVALID_DEPTH = 3
PBA_E_DEGENERATE_DEPTH = 4
PBA_E_SINGULAR_HESSIAN = 5
PBA_E_CUDA = 6
PBA_E_ARG = 7
PBA_E_STATE = 8
PBA_E_SPEC_INFEASIBLE = 9

PBA_K_NAMES = ["obs_pass", "schur", "cholesky", "trisolve", "ic_build", "reduce"]

i32, i64, f64, u8, u64 = C.c_int32, C.c_int64, C.c_double, C.c_uint8, C.c_uint64
P = C.POINTER


class pba_image(C.Structure):
    _fields_ = [("width", i32), ("height", i32), ("fx", f64), ("fy", f64), ("cx", f64), ("cy", f64),
                ("data", P(C.c_float))]


class pba_problem(C.Structure):
    _fields_ = [("ref", pba_image), ("num_frames", i32), ("targets", P(pba_image)), ("pose_R", P(f64)),
                ("pose_t", P(f64)), ("num_points", i32), ("anchors_px", P(f64)), ("inv_depths", P(f64)),
                ("pattern_size", i32), ("pattern", P(i32)), ("obs_ptr", P(i64)), ("obs_frame", P(i32))]


class pba_config(C.Structure):
    _fields_ = [("gamma", f64), ("threshold_px", f64), ("max_iters", i32), ("lambda0", f64),
                ("max_bad_steps", i32), ("normalize_depth_gauge", i32), ("refresh_ic_hessian", i32),
                ("record_snapshots", i32)]


class pba_iter_stats(C.Structure):
    _fields_ = [("iter", i32), ("energy", f64), ("max_update_px", f64), ("wall_ms", f64),
                ("hessian_builds", i32), ("hessian_factorizations", i32), ("num_active", i64),
                ("accepted", i32)]


class pba_report(C.Structure):
    _fields_ = [("converged", i32), ("diverged", i32), ("iterations", i32), ("hessian_builds", i32),
                ("hessian_factorizations", i32), ("rejected_steps", i32), ("final_energy", f64),
                ("total_wall_ms", f64), ("masked_residuals", i64), ("final_R", P(f64)), ("final_t", P(f64)),
                ("final_inv_depths", P(f64)), ("iters", P(pba_iter_stats)), ("iters_capacity", i32),
                ("num_iters", i32), ("snap_R", P(f64)), ("snap_t", P(f64)), ("snap_d", P(f64)),
                ("message", C.c_char * 256)]


class pba_mh_problem(C.Structure):
    _fields_ = [("num_frames", i32), ("images", P(pba_image)), ("pose_R", P(f64)), ("pose_t", P(f64)),
                ("affine_a", P(f64)), ("affine_b", P(f64)), ("num_points", i32), ("host", P(i32)),
                ("anchors_px", P(f64)), ("inv_depths", P(f64)), ("pattern_size", i32), ("pattern", P(i32)),
                ("obs_ptr", P(i64)), ("obs_frame", P(i32)), ("optimize_affine", i32)]


class pba_energy_result(C.Structure):
    _fields_ = [("energy", f64), ("num_active", i64), ("num_out_of_bounds", i64)]


VP = C.c_void_p
_COMMON = {
    # name: (restype, argtypes)
    "create": (C.c_int, [P(pba_problem), P(VP)]),
    "destroy": (None, [VP]),
    "last_error": (C.c_char_p, [VP]),
    "num_observations": (i64, [VP]),
    "set_params": (C.c_int, [VP, P(f64), P(f64), P(f64)]),
    "get_params": (C.c_int, [VP, P(f64), P(f64), P(f64)]),
    "energy": (C.c_int, [VP, f64, P(u8), P(pba_energy_result), P(f64), P(u8)]),
    "ic_build": (C.c_int, [VP, P(pba_config)]),
    "ic_gradient": (C.c_int, [VP, P(f64)]),
    "ic_compute_step": (C.c_int, [VP, P(f64)]),
    "ic_solve_step": (C.c_int, [VP, P(f64), P(f64)]),
    "ic_factorize": (C.c_int, [VP, f64]),
    "ic_hessian": (C.c_int, [VP, P(f64), P(f64), P(f64), P(f64)]),
    "warning_count": (C.c_int, [VP]),
    "warning": (C.c_int, [VP, C.c_int, C.c_char_p, C.c_int]),
    "warnings_text": (C.c_int64, [VP, C.c_char_p, C.c_int64]),
    "warning_points": (C.c_int64, [VP, P(i32), C.c_int64]),
    "ic_run": (C.c_int, [VP, P(pba_config), P(pba_report)]),
    "fc_build": (C.c_int, [VP, f64, P(f64), P(f64), P(f64), P(f64)]),
    "fc_run": (C.c_int, [VP, P(pba_config), P(pba_report)]),
    "solve_normal_equations_schur": (C.c_int, [i32, i32, P(i64), P(i32), P(f64), P(f64), P(f64), P(f64), f64,
                                                P(f64)]),
    "apply_update": (C.c_int, [VP, C.c_int, P(f64), P(f64), P(f64), P(f64), P(C.c_int)]),
    "max_reproj_update": (C.c_int, [VP, P(f64), P(f64), P(f64), P(f64)]),
    "normalize_gauge": (C.c_int, [VP]),
    # joint multi-host window (pba_gpu_mh_*)
    "mh_create": (C.c_int, [P(pba_mh_problem), P(VP)]),
    "mh_destroy": (None, [VP]),
    "mh_last_error": (C.c_char_p, [VP]),
    "mh_energy": (C.c_int, [VP, f64, P(pba_energy_result)]),
    "mh_fc_run": (C.c_int, [VP, P(pba_config), P(pba_report), P(f64), P(f64)]),
}
_GPU_ONLY = {
    "create_deferred": (C.c_int, [P(pba_problem), P(VP)]),
    "nccl_unique_id": (C.c_int, [VP]),
    "set_exchange_nccl": (C.c_int, [VP, VP, i32, i32, i64]),
    "ic_begin": (C.c_int, [VP, P(pba_config)]),
    "fc_begin": (C.c_int, [VP, P(pba_config)]),
    "iterate": (C.c_int, [VP, P(pba_iter_stats), P(C.c_int)]),
    "end": (C.c_int, [VP, P(pba_report)]),
    "stream": (VP, [VP]),
    "set_profiling": (C.c_int, [VP, C.c_int]),
    "kernel_times": (C.c_int, [VP, P(i64), P(f64)]),
    "device_bytes": (i64, [VP]),
    "launch_count": (i64, []),
}

_cache: dict = {}


class Backend:
    """The loaded product library with uniformly named functions (``self.create`` ...)."""

    def __init__(self):
        self.kind = "gpu"
        path = GPU_LIB
        if not path.exists():
            raise RuntimeError(
                f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                f"(the product has no fallback)")
        self.lib = C.CDLL(str(path))
        self.path = path
        for name, (res, args) in {**_COMMON, **_GPU_ONLY}.items():
            fn = getattr(self.lib, "pba_gpu_" + name)
            fn.restype = res
            fn.argtypes = args
            setattr(self, name, fn)
        self.status_string = self.lib.pba_status_string
        self.status_string.restype = C.c_char_p
        self.status_string.argtypes = [C.c_int]
        # host-only utility of the CLI (synth.cpp:308-320); no device work
        self.perturb_parameters = self.lib.pba_perturb_parameters
        self.perturb_parameters.restype = C.c_int
        self.perturb_parameters.argtypes = [i32, P(f64), P(f64), i32, P(f64), f64, u64]
        self.config_default = self.lib.pba_config_default


def backend(kind="gpu"):
    """The product library for ``"gpu"``; a library object built elsewhere with the same call set
    (the test suite's CPU checkers) is passed through unchanged."""
    if isinstance(kind, str):
        if kind != "gpu":
            raise ValueError(f"unknown library {kind!r}: this package binds only libpba_gpu.so")
        if "gpu" not in _cache:
            _cache["gpu"] = Backend()
        return _cache["gpu"]
    if not hasattr(kind, "create"):
        raise TypeError(f"{kind!r} is not a bound PBA library")
    return kind


def default_config() -> pba_config:
    """SolverConfig{} (solver.hpp:45-54)."""
    return pba_config(gamma=0.03, threshold_px=5e-3, max_iters=200, lambda0=1e-6, max_bad_steps=8,
                      normalize_depth_gauge=1, refresh_ic_hessian=0, record_snapshots=0)


def lib_paths() -> dict:
    return {"gpu": str(GPU_LIB), "exists_gpu": GPU_LIB.exists(), "pid": os.getpid()}
