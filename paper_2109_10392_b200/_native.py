"""ctypes binding of the C ABI in include/batchmpc_b200.h.

There is no CPU fallback: if the sm_100a library is missing or no CUDA device
is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, Structure, c_double, c_int, c_longlong, c_ubyte, c_void_p
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libbatchmpc_b200.so"
if os.environ.get("BMPC_LIB"):  # e.g. the phase-profiling build (tools/phase_prof.py)
    LIB_PATH = Path(os.environ["BMPC_LIB"]).resolve()

BMPC_OK, BMPC_EINVAL, BMPC_ECUDA, BMPC_ESINGULAR = 0, 1, 2, 3

_dp = POINTER(c_double)


class Problem(Structure):
    _fields_ = [
        ("m", c_int), ("l", c_int), ("S", c_int),
        ("xi_x", c_void_p), ("xi_y", c_void_p), ("b_xy", c_void_p), ("b_psi", c_void_p),
        ("a", c_double), ("b", c_double), ("v_min", c_double), ("v_max", c_double),
        ("a_max", c_double),
    ]


class SolveOpts(Structure):
    _fields_ = [
        ("max_iter", c_int), ("tol", c_double), ("keep_multipliers", c_int),
        ("warps_per_block", c_int), ("want_v", c_int), ("precision", c_int),
        ("w_alpha", c_void_p), ("w_d", c_void_p), ("w_alpha_a", c_void_p), ("w_d_a", c_void_p),
        ("w_v", c_void_p), ("w_c_psi", c_void_p),
        ("w_l_x", c_void_p), ("w_l_y", c_void_p), ("w_l_psi", c_void_p),
        ("status_dev", c_void_p), ("w_mask", c_void_p), ("team_warps", c_int),
    ]


class SolveOut(Structure):
    _fields_ = [
        ("c_x", c_void_p), ("c_y", c_void_p), ("c_psi", c_void_p),
        ("l_x", c_void_p), ("l_y", c_void_p), ("l_psi", c_void_p),
        ("v", c_void_p), ("history", c_void_p), ("res_final", c_void_p),
        ("iterations", c_int), ("converged", c_int),
    ]


class ScoreSpec(Structure):
    _fields_ = [
        ("kind", c_int), ("v_cruise", c_double), ("v_max", c_double), ("y_rl", c_double),
        ("w1", c_double), ("w2", c_double),
        ("heading_limit", c_double), ("residual_tol", c_double), ("collision_margin", c_double),
    ]


class ScoreOut(Structure):
    _fields_ = [
        ("meta_cost", c_void_p), ("min_ratio", c_void_p), ("heading_max", c_void_p),
        ("flags", c_void_p),
        ("best_index", c_void_p), ("argmin_all", c_void_p), ("argmin_hc", c_void_p),
        ("n_feasible", c_void_p),
    ]


EXPORTS = {
    # name: (argtypes, restype)
    "bmpc_abi_version": ([], c_int),
    "bmpc_abi_layout": ([POINTER(c_longlong), c_int], c_int),
    "bmpc_last_error": ([], ctypes.c_char_p),
    "bmpc_ctx_create": ([c_int, c_int, c_double] + [_dp] * 9 + [POINTER(c_void_p)], c_int),
    "bmpc_ctx_destroy": ([c_void_p], c_int),
    "bmpc_carry_doubles": ([c_void_p], c_int),
    "bmpc_ctx_info": ([c_void_p, POINTER(c_int), POINTER(c_int), POINTER(c_int), POINTER(c_void_p)], c_int),
    "bmpc_ctx_qp_info": ([c_void_p, POINTER(c_double), POINTER(c_double), POINTER(c_int)], c_int),
    "bmpc_reduced_qp": ([c_int, c_int, _dp, _dp, _dp, POINTER(c_double)], c_int),
    "bmpc_solve": ([c_void_p, POINTER(Problem), POINTER(SolveOpts), POINTER(SolveOut), c_void_p], c_int),
    "bmpc_sweeps": ([c_void_p, POINTER(Problem), POINTER(SolveOpts), c_int, c_int, c_int, c_void_p,
                     c_int, POINTER(SolveOut), c_void_p], c_int),
    "bmpc_score": ([c_void_p, POINTER(Problem), c_void_p, c_void_p, c_void_p, c_void_p,
                    POINTER(ScoreSpec), POINTER(ScoreOut), c_void_p], c_int),
    "bmpc_score_samples": ([POINTER(Problem), c_int] + [c_void_p] * 5 + [POINTER(ScoreSpec),
                                                                       POINTER(ScoreOut), c_void_p], c_int),
    "bmpc_plan_host_layout": ([c_void_p, c_int, c_int, c_int, POINTER(c_longlong), c_int], c_int),
    "bmpc_plan_host": ([c_void_p, POINTER(Problem), POINTER(SolveOpts), POINTER(SolveOut),
                        POINTER(ScoreSpec), POINTER(ScoreOut), c_void_p], c_int),
    "bmpc_plan": ([c_void_p, POINTER(Problem), POINTER(SolveOpts), POINTER(SolveOut),
                   POINTER(ScoreSpec), POINTER(ScoreOut), c_void_p], c_int),
    "bmpc_sample": ([c_void_p, c_int] + [c_void_p] * 12 + [c_void_p], c_int),
    "bmpc_assemble": ([c_void_p, c_int, c_int, c_int, c_int] + [c_void_p] * 9 + [c_void_p], c_int),
    "bmpc_op_obstacle_update": ([c_int, c_int, c_int] + [c_void_p] * 4 + [c_double, c_double]
                                + [c_void_p] * 2 + [c_void_p], c_int),
    "bmpc_op_accel_update": ([c_int, c_int, c_void_p, c_void_p, c_double, c_void_p, c_void_p, c_void_p], c_int),
    "bmpc_op_v_update": ([c_int, c_int, c_void_p, c_void_p, c_double, c_double, c_void_p, c_void_p], c_int),
    "bmpc_op_assemble_g": ([c_int, c_int, c_int] + [c_void_p] * 8 + [c_double, c_double]
                           + [c_void_p] * 2 + [c_void_p], c_int),
    "bmpc_op_residual_vectors": ([c_int, c_int, c_int] + [c_void_p] * 14 + [c_double, c_double]
                                 + [c_void_p] * 2 + [c_void_p], c_int),
    "bmpc_op_tail": ([c_int, c_int, c_int] + [c_void_p] * 9 + [c_double] * 5 + [c_void_p] * 12
                     + [c_void_p], c_int),
    "bmpc_dfma_peak": ([c_int, _dp, c_void_p], c_int),
    "bmpc_math_check": ([c_int, c_longlong, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p], c_int),
    "bmpc_latency_probe": ([c_int, _dp, c_void_p], c_int),
    "bmpc_project": ([c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p], c_int),
    "bmpc_kkt_apply": ([c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p], c_int),
    "bmpc_heading": ([c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p], c_int),
    "bmpc_op_d_obs": ([c_int, c_int, c_int] + [c_void_p] * 5 + [c_double, c_double, c_void_p,
                                                                 c_void_p], c_int),
    "bmpc_block_norms": ([c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p], c_int),
    "bmpc_op_collision_ratios": ([c_int, c_int, c_int] + [c_void_p] * 4 + [c_double, c_double, c_void_p,
                                                                            c_void_p], c_int),
}

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load the sm_100a library (raises when it has not been built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                    " (there is no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (argtypes, restype) in EXPORTS.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = restype
            _lib = lib
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == BMPC_OK:
        return
    msg = load().bmpc_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == BMPC_EINVAL:
        raise ValueError(msg)
    if rc == BMPC_ESINGULAR:
        raise np.linalg.LinAlgError(msg)
    raise RuntimeError(msg)


def host_ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags.c_contiguous, "host buffers must be C-contiguous"
    return a.ctypes.data


def c_double_ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


__all__ = ["load", "check", "Problem", "SolveOpts", "SolveOut", "ScoreSpec", "ScoreOut",
           "EXPORTS", "LIB_PATH", "host_ptr", "c_double_ptr", "c_longlong", "c_ubyte"]
