"""ctypes binding of ``libzks_b200.so`` (include/zipfks_b200.h).

There is no CPU implementation behind this module: if the library is missing or no sm_100
device is visible, every engine call raises.
"""
from __future__ import annotations

import ctypes
import os

from ._build import LIB

ZKS_OK, ZKS_EINVAL, ZKS_ECUDA = 0, 1, 2
STATUS_OK, STATUS_RETRIED, STATUS_FAILED = 0, 1, 2
MLE_TABLE, MLE_DIRECT = 0, 1
KERNEL_KINDS = ("row", "draw", "fit", "retry", "batch", "single", "select", "other")  # ZKS_KERNEL_*
ABI_VERSION = 3

# every symbol include/zipfks_b200.h declares
EXPORTS = (
    "zks_version",
    "zks_last_error",
    "zks_engine_create",
    "zks_engine_destroy",
    "zks_engine_set_stream",
    "zks_engine_sync",
    "zks_engine_launches",
    "zks_engine_set_timing",
    "zks_engine_kernel_times",
    "zks_table_create",
    "zks_table_destroy",
    "zks_run_replicates",
    "zks_run_cells",
    "zks_tail_mass",
    "zks_engine_set_rng",
    "zks_select_ranks",
    "zks_select_ranks_async",
    "zks_select_ranks_batch",
    "zks_select_dist_begin",
    "zks_select_dist_count",
    "zks_select_dist_pick",
    "zks_select_dist_end",
    "zks_normaliser",
    "zks_stream_uniforms",
    "zks_stream_uniforms_key",
    "zks_engine_set_chunk_bytes",
    "zks_draw",
    "zks_fit_samples",
    "zks_series_eval",
    "zks_solve_exponents",
    "zks_engine_set_mle_mode",
    "zks_fit_eval",
    "zks_engine_set_counters",
    "zks_probe_peaks",
)


FIT_EXPONENT, FIT_KS = 1, 2
SAMPLE_OK, SAMPLE_NOROOT, SAMPLE_OUTSIDE, SAMPLE_EMPTY = 0, 2, 3, 4


class ZksMleSettings(ctypes.Structure):
    _fields_ = [
        ("initial_guess", ctypes.c_double),
        ("absolute_tolerance", ctypes.c_double),
        ("max_iterations", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("bracket_lo", ctypes.c_double),
        ("bracket_hi", ctypes.c_double),
    ]


class ZksCell(ctypes.Structure):
    _fields_ = [
        ("support_k", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("gamma", ctypes.c_double),
        ("n", ctypes.c_int64),
        ("base_seed", ctypes.c_uint64),
        ("repetition", ctypes.c_uint64),
        ("first", ctypes.c_uint64),
        ("count", ctypes.c_uint64),
    ]


_lib = None


def load() -> ctypes.CDLL:
    """Load the engine library (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        raise ImportError(
            f"CUDA engine library {LIB} is missing; build it with "
            "`python -m paper_1305_6738_b200._build` (there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB)
    vp, i32, i64, u64, dp = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
    lib.zks_version.restype = ctypes.c_int
    lib.zks_last_error.restype = ctypes.c_char_p
    lib.zks_engine_create.argtypes = [ctypes.c_int, dp, i64, ctypes.POINTER(vp)]
    lib.zks_engine_destroy.argtypes = [vp]
    lib.zks_engine_destroy.restype = None
    lib.zks_engine_set_stream.argtypes = [vp, vp]
    lib.zks_engine_sync.argtypes = [vp]
    lib.zks_engine_launches.argtypes = [vp, dp]
    lib.zks_engine_set_timing.argtypes = [vp, ctypes.c_int]
    lib.zks_engine_kernel_times.argtypes = [vp, dp, dp]
    lib.zks_table_create.argtypes = [vp, dp, i64, ctypes.POINTER(vp)]
    lib.zks_table_destroy.argtypes = [vp]
    lib.zks_table_destroy.restype = None
    lib.zks_run_replicates.argtypes = [vp, vp, ctypes.POINTER(ZksCell), dp, dp, dp]
    lib.zks_run_cells.argtypes = [vp, i32, dp, dp, dp, dp, dp]
    lib.zks_tail_mass.argtypes = [vp, ctypes.c_double, dp, i64, dp]
    lib.zks_engine_set_rng.argtypes = [vp, ctypes.c_int]
    lib.zks_select_ranks.argtypes = [vp, dp, i64, dp, i32, dp]
    lib.zks_select_ranks_async.argtypes = [vp, dp, i64, dp, i32, dp]
    lib.zks_select_ranks_batch.argtypes = [vp, dp, dp, i32, dp, i32, dp, dp, dp]
    lib.zks_select_dist_begin.argtypes = [vp, dp, dp, dp, i32, dp, i32, dp, dp, dp]
    lib.zks_select_dist_count.argtypes = [vp, i32, dp]
    lib.zks_select_dist_pick.argtypes = [vp, i32, dp]
    lib.zks_select_dist_end.argtypes = [vp]
    lib.zks_normaliser.argtypes = [vp, ctypes.c_double, i32, dp]
    lib.zks_stream_uniforms.argtypes = [vp, u64, u64, u64, i64, dp]
    lib.zks_stream_uniforms_key.argtypes = [vp, u64, u64, i64, dp]
    lib.zks_engine_set_chunk_bytes.argtypes = [vp, u64]
    lib.zks_draw.argtypes = [vp, vp, dp, i64, dp]
    lib.zks_engine_set_counters.argtypes = [vp, dp]
    lib.zks_fit_samples.argtypes = [vp, i32, dp, dp, i64, i32, ctypes.POINTER(ZksMleSettings), dp, dp, dp, dp, dp, dp,
                                    dp]
    lib.zks_series_eval.argtypes = [vp, i32, dp, i64, dp]
    lib.zks_solve_exponents.argtypes = [vp, i32, dp, i64, ctypes.POINTER(ZksMleSettings), i32, dp, dp]
    lib.zks_engine_set_mle_mode.argtypes = [vp, ctypes.c_int]
    lib.zks_fit_eval.argtypes = [vp, i32, dp, i64, dp, dp, dp]
    lib.zks_probe_peaks.argtypes = [vp, dp]
    for name in EXPORTS:
        if name not in ("zks_version", "zks_last_error", "zks_engine_destroy", "zks_table_destroy"):
            getattr(lib, name).restype = ctypes.c_int
    if lib.zks_version() != ABI_VERSION:
        raise ImportError(f"{LIB}: ABI version {lib.zks_version()} != {ABI_VERSION}; rebuild")
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a C return code onto the reference's exception types."""
    if rc == ZKS_OK:
        return
    msg = (_lib.zks_last_error() or b"").decode()
    if rc == ZKS_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"zipfks_b200 CUDA error: {msg}")
