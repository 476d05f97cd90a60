"""ctypes binding of libblockct_cuda.so (include/blockct.h).

There is deliberately no fallback: if the library or a GPU is missing every
call raises NativeLibraryError.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import ConfigurationError, ExecutorError, NativeLibraryError, ScheduleError

LIB_PATH = os.environ.get("BCT_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libblockct_cuda.so")

BCT_OK, BCT_EINVAL, BCT_ECUDA, BCT_ENOMEM, BCT_ESCHEDULE = 0, -1, -2, -3, -4
BCT_F64, BCT_F32 = 0, 1
MODES = {"serial_faithful": 0, "parallel": 1}
BCT_COMMIT, BCT_METRICS, BCT_SHARDED, BCT_GUARD, BCT_GUARD_REF = 1, 2, 4, 8, 16
STRATEGY_CODES = {"importance": 0, "random": 1, "mixed": 2}
BCT_ROW_ACTION, BCT_COLUMN_ACTION = 0, 1
M_RULE_CODES = {"identity": 0, "sum_inverse": 1, "norm_inverse": 2}

_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_dbl = ctypes.c_double
_p = ctypes.c_void_p
_pp = ctypes.POINTER(ctypes.c_void_p)


class Panel(ctypes.Structure):
    _fields_ = [("n_rows", _i64), ("nnz", _i64), ("data", _p), ("cols", _p),
                ("indptr", _p), ("rbp", _p), ("l2g", _p)]


class SystemDesc(ctypes.Structure):
    _fields_ = [("m", _i32), ("n_panels", _i32), ("n_meas", _i64), ("n_vox", _i64),
                ("row_block_ptr", _p), ("row_block_rows", _p), ("col_block_ptr", _p),
                ("col_block_vox", _p), ("table_values", _p), ("table_totals", _p),
                ("panel_begin", _i32), ("panel_end", _i32), ("dtype", _i32), ("device", _i32)]


class PBDesc(ctypes.Structure):
    _fields_ = [("n", _i64), ("views", _i64), ("bins", _i64), ("m", _i32), ("nc", _i32),
                ("cos_views", _p), ("sin_views", _p), ("panel_begin", _i32),
                ("panel_end", _i32), ("dtype", _i32), ("device", _i32)]


class ScanDesc(ctypes.Structure):
    _fields_ = [("dims", _i64 * 3), ("voxel_size", _dbl * 3), ("origin", _dbl * 3),
                ("det_nu", _i64), ("det_nv", _i64), ("det_du", _dbl), ("det_dv", _dbl),
                ("n_views", _i64), ("poses", _p), ("m", _i32), ("n_panels", _i32),
                ("row_block_ptr", _p), ("row_block_rows", _p), ("box_lo", _p), ("box_hi", _p),
                ("table_values", _p), ("table_totals", _p), ("panel_begin", _i32),
                ("panel_end", _i32), ("dtype", _i32), ("device", _i32)]


class EpochResult(ctypes.Structure):
    _fields_ = [("n_tasks", _i64), ("n_visits", _i64), ("n_degenerate", _i64),
                ("resid_sq", _dbl), ("x_sq", _dbl), ("err_sq", _dbl), ("kernel_ms", _dbl)]


# name -> argtypes (all return int32 except bct_last_error / bct_version)
_SIGS = {
    "bct_create": [ctypes.POINTER(SystemDesc), ctypes.POINTER(Panel), _pp],
    "bct_create_parallel_beam": [ctypes.POINTER(PBDesc), _pp],
    "bct_create_scan": [ctypes.POINTER(ScanDesc), _pp],
    "bct_destroy": [_p],
    "bct_info": [_p, _p],
    "bct_panel_info": [_p, _i32, _p, _p, _p],
    "bct_get_panel": [_p, _i32, _p, _p, _p, _p, _p],
    "bct_get_table": [_p, _p, _p],
    "bct_get_stream": [_p, _pp],
    "bct_set_y": [_p, _p],
    "bct_set_x": [_p, _p],
    "bct_get_x": [_p, _p],
    "bct_set_r": [_p, _p],
    "bct_get_r": [_p, _p],
    "bct_set_z": [_p, _i32, _p],
    "bct_get_z": [_p, _i32, _p],
    "bct_get_xhat": [_p, _p],
    "bct_set_x_true": [_p, _p],
    "bct_reset_accumulators": [_p],
    "bct_clear_state": [_p],
    "bct_get_counts": [_p, _p],
    "bct_commit_epoch": [_p],
    "bct_reset_residual": [_p],
    "bct_begin_solve": [_p, _p, _p],
    "bct_fill_z_from_image": [_p],
    "bct_projection_sum": [_p, _p],
    "bct_forward": [_p, _p, _p],
    "bct_audit": [_p, _p],
    "bct_run_epoch": [_p, _i32, _i64, _p, _p, _p, _p, _p, _i32],
    "bct_sample_epoch": [_p, _i32, _i32, _p, _p, _i64, _p, _i32, _dbl, _i32, _dbl, _i32, _p],
    "bct_wait_epoch": [_p, ctypes.POINTER(EpochResult), _p, _p],
    "bct_set_divergence_factor": [_p, ctypes.c_double],
    "bct_exchange_buffer": [_p, _pp, ctypes.POINTER(_i64)],
    "bct_finish_sharded": [_p, _i32, _p],
    "bct_debug_timeline": [_p, _p, _i64, _p],
    "bct_baseline_init": [_p, _i32, _i32],
    "bct_baseline_epoch": [_p, _dbl, _p],
    "bct_baseline_get_x": [_p, _p],
}

EXPORTED = tuple(_SIGS) + ("bct_last_error", "bct_version")

_LIB = None


def load(path=LIB_PATH):
    """Load the library (no GPU needed to load; calls need one)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    # profiling: BCT_LIB selects a variant build (tools/build_variant.sh)
    path = os.environ.get("BCT_LIB") or path
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} is missing; build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (there is no CPU fallback)")
    L = ctypes.CDLL(path)
    for name, args in _SIGS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = _i32
    L.bct_last_error.argtypes = [_p]
    L.bct_last_error.restype = ctypes.c_char_p
    L.bct_version.argtypes = []
    L.bct_version.restype = _i32
    _LIB = L
    return L


def ptr(a):
    """Address of a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data


def check(rc, ctx=None, what="", task=None):
    """Map a status code to the reference's exception types."""
    if rc == BCT_OK:
        return
    msg = load().bct_last_error(ctx).decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == BCT_ESCHEDULE:
        raise ExecutorError(text, task=task)
    if rc == BCT_EINVAL:
        raise ConfigurationError(text)
    raise NativeLibraryError(text)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


__all__ = ["load", "ptr", "check", "Panel", "SystemDesc", "PBDesc", "EpochResult", "EXPORTED",
           "MODES", "BCT_F64", "BCT_F32", "BCT_COMMIT", "BCT_METRICS", "BCT_SHARDED",
           "BCT_GUARD", "BCT_GUARD_REF",
           "STRATEGY_CODES", "ScheduleError"]
