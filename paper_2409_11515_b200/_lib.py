"""ctypes binding of the native library (include/condkit_b200.h).

The library is built in-tree (``paper_2409_11515_b200/libcondkit_b200.so``).
There is no fallback: if the library is missing or no sm_100 device is visible,
calls that need the GPU raise ``DeviceUnavailable``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CK_LIB") or os.path.join(_HERE, "libcondkit_b200.so")

dp = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
u64p = C.POINTER(C.c_uint64)


class AdamCfg(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps_stab", C.c_double), ("max_iter", C.c_uint64), ("seed", C.c_uint64),
                ("rel_tol", C.c_double), ("patience", C.c_uint64)]


class NormResult(C.Structure):
    _fields_ = [("value", C.c_double), ("iterations", C.c_uint64), ("converged", C.c_int32),
                ("_pad", C.c_int32)]


class StepInfo(C.Structure):
    _fields_ = [("t", C.c_uint64), ("loss", C.c_double), ("loss_min", C.c_double),
                ("x_dot_delta", C.c_double), ("delta_norm", C.c_double), ("phase", C.c_int32),
                ("_pad", C.c_int32)]


class MatrixInfo(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("sell_entries_a", C.c_int64), ("sell_entries_at", C.c_int64),
                ("device_bytes", C.c_int64), ("device", C.c_int32), ("col_format", C.c_int32)]


# name -> (restype, argtypes)
_SIGS = {
    "ck_last_error": (C.c_char_p, []),
    "ck_abi_version": (C.c_int32, []),
    "ck_device_count": (C.c_int, [i32p]),
    "ck_device_memory": (C.c_int, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), i32p]),
    "ck_set_device": (C.c_int, [C.c_int32]),
    "ck_device_synchronize": (C.c_int, []),
    "ck_host_register": (C.c_int, [C.c_void_p, C.c_uint64]),
    "ck_start_vector_prefetch": (C.c_int, [C.c_uint64, C.c_int64]),
    "ck_start_vector_prefetch_cancel": (C.c_int, []),
    "ck_start_vector_prefetch_stats": (C.c_int, [u64p, u64p]),
    "ck_host_unregister": (C.c_int, [C.c_void_p]),
    "ck_adam_default": (None, [C.POINTER(AdamCfg)]),
    "ck_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "ck_random_unit_vectors": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, dp]),
    "ck_uniform_in": (C.c_int, [C.c_uint64, C.c_int64, C.c_double, C.c_double, dp]),
    "ck_loose_bounds": (C.c_int, [C.c_double, C.c_double, C.c_double, dp, dp]),
    "ck_tight_bounds": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, dp, dp]),
    "ck_propagate_bound": (C.c_int, [C.c_double, dp]),
    "ck_singularity_bound": (C.c_int, [C.c_double, C.c_double, dp]),
    "ck_matrix_upload": (C.c_int, [C.c_int64, C.c_int64, i64p, i32p, dp, C.POINTER(C.c_void_p)]),
    "ck_matrix_free": (C.c_int, [C.c_void_p]),
    "ck_matrix_get_info": (C.c_int, [C.c_void_p, C.POINTER(MatrixInfo)]),
    "ck_spmv": (C.c_int, [C.c_void_p, dp, dp]),
    "ck_spmv_t": (C.c_int, [C.c_void_p, dp, dp]),
    "ck_residual_norms": (C.c_int, [C.c_void_p, dp, dp, dp, dp, dp]),
    "ck_loss_explicit": (C.c_int, [C.c_void_p, dp, dp]),
    "ck_grad_explicit": (C.c_int, [C.c_void_p, dp, dp]),
    "ck_projected_adam": (C.c_int, [C.c_void_p, C.POINTER(AdamCfg), C.POINTER(NormResult), dp]),
    "ck_estimate_norm": (C.c_int, [C.c_void_p, C.POINTER(AdamCfg), C.c_uint64,
                                   C.POINTER(NormResult), dp]),
    "ck_session_create": (C.c_int, [C.c_void_p, C.POINTER(AdamCfg), u64p, C.c_int32,
                                    C.POINTER(C.c_void_p)]),
    "ck_session_run": (C.c_int, [C.c_void_p, C.c_uint64, i32p]),
    "ck_session_step_observed": (C.c_int, [C.c_void_p, C.POINTER(StepInfo), dp, dp]),
    "ck_session_time": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int32, dp, dp, dp]),
    "ck_session_result": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(NormResult), dp]),
    "ck_session_free": (C.c_int, [C.c_void_p]),
    "ck_lu_factorize": (C.c_int, [C.c_void_p, C.c_double, C.POINTER(C.c_void_p), i64p, dp]),
    "ck_lu_free": (C.c_int, [C.c_void_p]),
    "ck_lu_get_info": (C.c_int, [C.c_void_p, i64p, i64p, i64p, dp, i64p]),
    "ck_lu_factorize_batch": (C.c_int, [C.c_void_p, C.c_int32, C.c_double, C.c_void_p, i32p, i64p, dp]),
    "ck_lu_export": (C.c_int, [C.c_void_p, dp, i32p]),
    "ck_lu_csr_info": (C.c_int, [C.c_void_p, i64p, i64p]),
    "ck_lu_export_csr": (C.c_int, [C.c_void_p, i64p, i32p, dp, i64p, i32p, dp, i64p]),
    "ck_lu_solve": (C.c_int, [C.c_void_p, dp, dp]),
    "ck_restart_group": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int32, C.POINTER(C.c_int32)]),
    "ck_lu_dense_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), dp]),
    "ck_lu_dense_solve": (C.c_int, [C.c_void_p, C.c_int32, dp, dp]),
    "ck_lu_transpose_solve": (C.c_int, [C.c_void_p, dp, dp]),
    "ck_loss_inverse": (C.c_int, [C.c_void_p, dp, dp]),
    "ck_grad_inverse": (C.c_int, [C.c_void_p, dp, dp]),
    "ck_inv_projected_adam": (C.c_int, [C.c_void_p, C.POINTER(AdamCfg), C.POINTER(NormResult), dp]),
    "ck_inv_estimate_norm": (C.c_int, [C.c_void_p, C.POINTER(AdamCfg), C.c_uint64,
                                       C.POINTER(NormResult), dp]),
    "ck_session_create_inverse": (C.c_int, [C.c_void_p, C.POINTER(AdamCfg), u64p, C.c_int32,
                                            C.POINTER(C.c_void_p)]),
    "ck_cond2": (C.c_int, [C.c_void_p, C.POINTER(AdamCfg), C.c_uint64, C.c_double, dp,
                           C.POINTER(NormResult), C.POINTER(NormResult), i32p]),
    "ck_session_create_batch": (C.c_int, [C.c_void_p, i64p, C.c_int32, C.POINTER(AdamCfg), u64p,
                                          C.c_int32, C.POINTER(C.c_void_p)]),
    "ck_estimate_norm_batch": (C.c_int, [C.c_void_p, i64p, C.c_int32, C.POINTER(AdamCfg), u64p,
                                         C.c_uint64, C.POINTER(NormResult)]),
    "ck_dist_nccl_id": (C.c_int, [C.c_void_p]),
    "ck_dist_create": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                 C.POINTER(AdamCfg), u64p, C.c_int32, C.POINTER(C.c_void_p)]),
    "ck_dist_run": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_int32)]),
    "ck_dist_time": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_double)]),
    "ck_dist_result": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(NormResult), dp]),
    "ck_dist_part_info": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(MatrixInfo)]),
    "ck_dist_free": (C.c_int, [C.c_void_p]),
    "ck_column_norms": (C.c_int, [C.c_void_p, dp]),
    "ck_row_norms": (C.c_int, [C.c_void_p, dp]),
    "ck_column_scale": (C.c_int, [C.c_void_p, i32p, dp, dp, dp, i64p]),
    "ck_row_scale": (C.c_int, [C.c_void_p, i64p, dp, dp, dp, dp, dp, i64p]),
    "ck_unscale_solution": (C.c_int, [C.c_int64, dp, dp, dp]),
    "ck_session_create_inverse_batch": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32,
                                                  C.POINTER(AdamCfg), u64p, C.c_int32,
                                                  C.POINTER(C.c_void_p)]),
    "ck_inv_estimate_norm_batch": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(AdamCfg),
                                             u64p, C.c_uint64, C.POINTER(NormResult)]),
    "ck_generate": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.c_uint64, i64p, i64p, i64p, i32p,
                              dp]),
}

_lib = None
_lock = threading.Lock()


def load() -> C.CDLL:
    """Load the native library (raises ``NativeLibraryMissing`` if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise errors.NativeLibraryMissing(
                    f"{LIB_PATH} not built; run `python -m paper_2409_11515_b200.build`")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                f = getattr(lib, name)
                f.restype = res
                f.argtypes = args
            _lib = lib
    return _lib


def check(status: int, where: str = "") -> None:
    if status == 0:
        return
    msg = load().ck_last_error()
    msg = msg.decode() if msg else ""
    raise errors.from_status(status, f"{where}: {msg}" if where else msg)


_device_ready = False


def ensure_device() -> None:
    """Bind the calling thread to cuda:0 (or $CK_DEVICE); fails loudly without one."""
    global _device_ready
    lib = load()
    if _device_ready:
        return
    n = C.c_int32(0)
    check(lib.ck_device_count(C.byref(n)), "ck_device_count")
    if n.value == 0:
        raise errors.DeviceUnavailable("no CUDA device visible; this build has no CPU path")
    check(lib.ck_set_device(int(os.environ.get("CK_DEVICE", "0"))), "ck_set_device")
    _device_ready = True


def dptr(a: np.ndarray):
    return a.ctypes.data_as(dp)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(i64p)


def i32ptr(a: np.ndarray):
    return a.ctypes.data_as(i32p)


def as_f64(x, n: int | None = None, what: str = "vector") -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float64)
    if a.ndim != 1:
        raise errors.DimensionMismatch(f"{what} must be one-dimensional")
    if n is not None and a.size != n:
        raise errors.DimensionMismatch(f"{what}: length {a.size} != {n}")
    return a


def cfg_struct(cfg) -> AdamCfg:
    return AdamCfg(float(cfg.alpha), float(cfg.beta1), float(cfg.beta2), float(cfg.eps_stab),
                   int(cfg.max_iter), int(cfg.seed) & 0xFFFFFFFFFFFFFFFF, float(cfg.rel_tol),
                   int(cfg.patience))
