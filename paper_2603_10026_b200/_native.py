"""ctypes binding of librf_cuda (include/rf_cuda.h).

The library is built in-tree (paper_2603_10026_b200/librf_cuda.so, see
__graft_entry__.build()). There is no fallback: if the shared object is
missing or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librf_cuda.so")

# rf_status
RF_OK = 0
RF_ERR_SHAPE = 1
RF_ERR_SEGMENTATION = 2
RF_ERR_DOMAIN = 3
RF_ERR_UNSUPPORTED = 4
RF_ERR_CUDA = 5
RF_ERR_NCCL = 6
RF_ERR_ARG = 7

# rf_pattern
RF_PATTERN_SAFE_SOFTMAX = 1
RF_PATTERN_ATTENTION = 2
RF_PATTERN_QUANT_GEMM_E4M3 = 3
RF_PATTERN_RMSNORM_GEMM = 4
RF_PATTERN_MOE_ROUTING = 5
RF_PATTERN_LAYERNORM_GEMM = 6
RF_PATTERN_VARIANCE = 7
RF_PATTERN_SUM_SUM = 8
RF_PATTERN_MOMENTS = 9
RF_PATTERN_MOE_ROUTER = 10
RF_PATTERN_MLA_DECODE = 11

ABI_VERSION = 5

# rf_dtype
RF_F32 = 0
RF_BF16 = 1
RF_E4M3 = 2


class rf_desc(ctypes.Structure):
    _fields_ = [
        ("pattern", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("batch", ctypes.c_int64),
        ("heads", ctypes.c_int64),
        ("rows", ctypes.c_int64),
        ("len", ctypes.c_int64),
        ("free_len", ctypes.c_int64),
        ("segments", ctypes.c_int64),
        ("fmax", ctypes.c_double),
        ("eps", ctypes.c_double),
        ("softmax_scale", ctypes.c_double),
        ("offset", ctypes.c_double),
        ("tile_rows", ctypes.c_int32),
        ("tile_stream", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("producer_len", ctypes.c_int32),
        ("stat_len", ctypes.c_int64),
        ("fuse_level", ctypes.c_int32),
        ("tree_depth", ctypes.c_int32),
        ("tree", ctypes.c_int64 * 8),
    ]


class rf_io(ctypes.Structure):
    _fields_ = [("in_", ctypes.c_void_p * 4), ("d", ctypes.c_void_p * 4)]


class rf_partials(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_void_p),
        ("l", ctypes.c_void_p),
        ("o", ctypes.c_void_p),
        ("nslices", ctypes.c_int64),
    ]


# Every symbol include/rf_cuda.h declares, with its ctypes signature.
_P = ctypes.c_void_p
SIGNATURES = {
    "rf_abi_version": (ctypes.c_int, []),
    "rf_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "rf_last_error": (ctypes.c_char_p, []),
    "rf_plan_create": (ctypes.c_int, [ctypes.POINTER(rf_desc), ctypes.POINTER(_P)]),
    "rf_plan_destroy": (None, [_P]),
    "rf_plan_describe": (ctypes.c_int, [_P, ctypes.c_char_p, ctypes.c_size_t]),
    "rf_plan_launches_per_run": (ctypes.c_int64, [_P]),
    "rf_plan_io_bytes": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]),
    "rf_pack_weight": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "rf_pack_weight_host": (ctypes.c_int, [_P, _P, _P, ctypes.POINTER(_P)]),
    "rf_packed_bytes": (ctypes.c_size_t, [_P]),
    "rf_buffer_free": (None, [_P]),
    "rf_run": (ctypes.c_int, [_P, ctypes.POINTER(rf_io), _P]),
    "rf_run_host": (ctypes.c_int, [_P, ctypes.POINTER(rf_io)]),
    "rf_run_partials": (
        ctypes.c_int,
        [_P, ctypes.POINTER(rf_io), ctypes.c_int64, ctypes.POINTER(rf_partials), _P],
    ),
    "rf_merge_partials": (
        ctypes.c_int,
        [_P, ctypes.POINTER(rf_partials), ctypes.POINTER(rf_io), _P],
    ),
    "rf_check_domain": (ctypes.c_int, [_P, _P]),
}

_lib = None
_lock = threading.Lock()


class NativeLibraryMissing(RuntimeError):
    """librf_cuda.so is not built or cannot be loaded (there is no fallback)."""


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} not found: run __graft_entry__.build() (no CPU fallback exists)"
                )
            try:
                h = ctypes.CDLL(LIB_PATH)
            except OSError as e:  # pragma: no cover
                raise NativeLibraryMissing(f"cannot load {LIB_PATH}: {e}") from e
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            if h.rf_abi_version() != ABI_VERSION:
                raise NativeLibraryMissing("librf_cuda ABI version mismatch")
            _lib = h
        return _lib


def last_error() -> str:
    return lib().rf_last_error().decode()
