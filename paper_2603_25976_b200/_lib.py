"""ctypes binding of libcurvopt_b200.so (the C ABI in include/curvopt_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every device entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import ContractError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libcurvopt_b200.so")

CV_OK, CV_E_CONTRACT, CV_E_NOT_PD, CV_E_CUDA, CV_E_NCCL, CV_E_UNSUPPORTED = range(6)
ACT = {"relu": 0, "tanh": 1}
LOSS = {"mse": 0, "ce": 1}
KIND_GGN, KIND_HESSIAN = 0, 1
ENGINE = {"auto": 0, "simt": 1, "tc": 2}


class CgStats(C.Structure):
    _fields_ = [("relres", C.c_double), ("bnorm", C.c_double), ("iterations", C.c_int32),
                ("converged", C.c_int32), ("neg_curv", C.c_int32), ("gv_count", C.c_int32),
                ("done", C.c_int32), ("x0_nonzero", C.c_int32), ("pad", C.c_int32 * 2)]


CG_STATS_BYTES = C.sizeof(CgStats)

LINK = {"scale": 0, "scale_by_schedule": 0, "trace_momentum": 1, "add_decayed_weights": 2, "scale_by_adam": 3,
        "sophia_clip": 4, "clip_global_norm": 5}


class CvLink(C.Structure):
    """cv_link (include/curvopt_b200.h): one pre-evaluated transform link."""
    _fields_ = [("kind", C.c_int32), ("pad", C.c_int32), ("p", C.c_double * 7), ("state_in", C.c_void_p * 2),
                ("state_out", C.c_void_p * 2)]

_P = C.c_void_p
# cv_comm_fn: int (*)(void* user, int dtype, void* buf, int64_t count, void* stream)
COMM_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p)
_SIGS = {
    "cv_version": (C.c_char_p, []),
    "cv_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, _P, C.POINTER(_P)]),
    "cv_ctx_destroy": (C.c_int, [_P]),
    "cv_ctx_set_comm": (C.c_int, [_P, COMM_FN, _P]),
    "cv_ctx_set_stream": (C.c_int, [_P, _P]),
    "cv_ctx_set_engine": (C.c_int, [_P, C.c_int]),
    "cv_last_error": (C.c_char_p, [_P]),
    "cv_ctx_capture_begin": (C.c_int, [_P]),
    "cv_ctx_capture_end": (C.c_int, [_P, C.POINTER(_P)]),
    "cv_arena_free": (C.c_int, [_P, _P]),
    "cv_nccl_unique_id": (C.c_int, [_P]),
    "cv_kernel_launches": (C.c_int64, [_P]),
    "cv_linearize": (C.c_int, [_P, C.c_int, _P, C.c_int, C.c_int, _P, _P, _P, C.c_int, C.c_int,
                               C.POINTER(_P), _P, _P]),
    "cv_snap_free": (C.c_int, [_P]),
    "cv_snap_dim": (C.c_int64, [_P]),
    "cv_snap_outputs": (C.c_int, [_P, _P]),
    "cv_snap_activation": (C.c_int, [_P, C.c_int, _P]),
    "cv_matvec": (C.c_int, [_P, C.c_int, _P, _P]),
    "cv_jvp": (C.c_int, [_P, _P, _P]),
    "cv_vjp": (C.c_int, [_P, _P, _P]),
    "cv_cg_solve": (C.c_int, [_P, C.c_int, _P, C.c_double, C.c_double, C.c_int, C.c_int, _P, C.c_double,
                              _P, _P, _P]),
    "cv_rademacher": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_int64, _P]),
    "cv_hutchinson": (C.c_int, [_P, C.c_int, C.c_uint64, C.c_uint64, C.c_int, _P, _P]),
    "cv_power_iter": (C.c_int, [_P, C.c_int, C.c_uint64, C.c_uint64, C.c_int, _P]),
    "cv_diag_ema": (C.c_int, [_P, _P, _P, C.c_double, C.c_int64, C.c_int, _P]),
    "cv_loss_at": (C.c_int, [_P, _P, _P]),
    "cv_rho_terms": (C.c_int, [_P, C.c_int, _P, _P, _P, _P]),
    "cv_apply_update": (C.c_int, [_P, _P, _P, C.c_double, C.c_int64, _P, _P, _P]),
    "cv_norm_check": (C.c_int, [_P, _P, C.c_int64, _P]),
    "cv_chain_apply": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, C.c_int64, _P, _P, _P]),
    "cv_gnb_diag": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_int, C.c_int64, _P]),
    "cv_gemm_test": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, _P, C.c_int64, C.c_int, _P, C.c_int64,
                               C.c_int, _P, C.c_int64]),
    "cv_gemm_bench": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    "cv_gemm_test_seg2": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, _P, _P, C.c_float, _P]),
    "cv_row_dim": (C.c_int64, [_P]),
    "cv_row_rhs": (C.c_int, [_P, _P]),
    "cv_row_gram": (C.c_int, [_P, _P]),
    "cv_row_solve_cholesky": (C.c_int, [_P, C.c_double, _P, _P]),
    "cv_row_solve_cholesky_dist": (C.c_int, [_P, _P, C.c_double, _P, _P]),
    "cv_row_solve_cg_dist": (C.c_int, [_P, _P, C.c_double, _P, C.c_double, C.c_int, C.c_int, _P, _P, _P]),
    "cv_backproject": (C.c_int, [_P, _P, _P]),
    "cv_row_solve_cg": (C.c_int, [_P, C.c_double, _P, C.c_double, C.c_int, C.c_int, _P, _P, _P]),
    "cv_dense_cholesky_solve": (C.c_int, [_P, _P, C.c_int64, C.c_double, _P, _P]),
    "cv_dense_cg_solve": (C.c_int, [_P, _P, C.c_int64, C.c_double, _P, C.c_double, C.c_int, C.c_int, _P, _P, _P]),
}

_lib = None
_lock = threading.Lock()


class DeviceError(RuntimeError):
    """A CUDA / NCCL failure inside the native library."""


class NotPositiveDefinite(ContractError):
    pass


def lib():
    """Load (once) and return the native library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"curvopt_b200 native library not built: {LIB_PATH} (run __graft_entry__.build())")
            h = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def exported_symbols():
    return tuple(_SIGS)


def check(rc: int, ctx_handle) -> None:
    if rc == CV_OK:
        return
    msg = lib().cv_last_error(ctx_handle)
    msg = msg.decode() if msg else "error"
    if rc == CV_E_CONTRACT:
        raise ContractError(msg)
    if rc == CV_E_NOT_PD:
        raise ContractError(msg)
    if rc == CV_E_UNSUPPORTED:
        raise ContractError("unsupported: " + msg)
    raise DeviceError(f"curvopt_b200 error {rc}: {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()
