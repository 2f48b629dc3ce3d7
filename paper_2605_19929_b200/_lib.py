"""ctypes binding of the C-ABI in include/splitq.h.

This is the whole Python<->native boundary: plain pointers and sizes. The
library is built in-tree by ``_build.py``; importing this module never falls
back to anything else — a missing library raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

from . import _build

SPLITQ_OK = 0
SPLITQ_ERR_INVALID = -1
SPLITQ_ERR_UNSUPPORTED = -2
SPLITQ_ERR_CUDA = -3
SPLITQ_ERR_DATA = -4
SPLITQ_ERR_NCCL = -5

F16, F32, F64, BF16 = 0, 1, 2, 3
FWD_RAW = 1
FWD_PROFILE = 2
FWD_UNPACKED = 4

STATUS_NONFINITE = 1
STATUS_SCALE = 2
STATUS_TAG = 4
STATUS_LR_RANGE = 8

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32


class QSpec(C.Structure):
    _fields_ = [("bits", _i32), ("symmetric", _i32)]


class LayerDesc(C.Structure):
    _fields_ = [
        ("d_in", _i64), ("d_out", _i64),
        ("n_main", _i64), ("n_text", _i64), ("n_vision", _i64),
        ("c_main", _p), ("c_text", _p), ("c_vision", _p),
        ("scale_main", _p), ("scale_text", _p), ("scale_vision", _p),
        ("act", QSpec), ("weight", QSpec), ("aux_bits_floor", _i32),
        ("use_cws", _i32), ("use_mac", _i32),
        ("r_cws", _i64), ("r_mac", _i64),
        ("q_main", _p), ("s_main", _p),
        ("q_text", _p), ("s_text", _p),
        ("q_vision", _p), ("s_vision", _p),
        ("q_us", _p), ("s_us", _p),
        ("q_vs", _p), ("s_vs", _p),
        ("q_uc", _p), ("s_uc", _p),
        ("q_vc", _p), ("s_vc", _p),
    ]


class WsLayout(C.Structure):
    _fields_ = [(n, _i64) for n in (
        "total_bytes", "status", "text_idx", "text_rows", "n_text",
        "a_main", "ld_main", "s_main", "sf_main", "zp_main", "lrs_main", "rho",
        "a_text", "ld_text", "s_text", "sf_text", "zp_text",
        "a_vision", "ld_vision", "s_vision", "sf_vision", "zp_vision",
        "a_mac", "s_mac", "zp_mac", "lrs_mac",
        "lr_a", "k_lr",
    )] + [("code_centered_main", _i32), ("code_centered_aux", _i32), ("main_natural", _i32),
          ("reserved", _i32), ("acc_scratch", _i64), ("acc_scratch_bytes", _i64), ("a_main_fp4", _i64)]


class SplitqError(RuntimeError):
    """Runtime failure inside the native library (CUDA / NCCL)."""


_LIB = None


def lib_path() -> str:
    return _build.LIB_PATH


def load(build_if_missing: bool = True):
    """Load libsplitq_b200.so (building it first when it is missing or stale
    and nvcc is available). Raises OSError when the library cannot be had."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = _build.LIB_PATH
    if build_if_missing and not _build.up_to_date():
        try:
            _build.build()
        except (OSError, FileNotFoundError) as exc:  # no nvcc here
            if not os.path.exists(path):
                raise OSError(f"{path} missing and could not be built: {exc}") from exc
    lib = C.CDLL(path)
    sig = {
        "splitq_last_error": (C.c_char_p, []),
        "splitq_version": (C.c_int, []),
        "splitq_device_sm_count": (C.c_int, [C.c_int, C.POINTER(C.c_int)]),
        "splitq_layer_create": (C.c_int, [C.POINTER(LayerDesc), C.c_int, C.POINTER(_p)]),
        "splitq_layer_destroy": (C.c_int, [_p]),
        "splitq_workspace_layout": (C.c_int, [_p, _i64, C.POINTER(WsLayout)]),
        "splitq_forward": (C.c_int, [_p, _p, C.c_int, _i64, _p, _i64, _p, C.c_int, _i64,
                                     _p, C.c_size_t, _p, C.c_int]),
        "splitq_read_status": (C.c_int, [_p, _p, C.POINTER(_i32)]),
        "splitq_profile_read": (C.c_int, [_p, C.POINTER(C.c_double), C.POINTER(_i32)]),
        "splitq_quantize_rows": (C.c_int, [_p, C.c_int, _i64, _i64, _i64, QSpec, _p, _i64,
                                           _p, _p, _p, C.POINTER(_i32), _p]),
        "splitq_gemm_i8": (C.c_int, [_p, _i64, C.c_int, _p, _i64, _p, _i64, _i64, _i64,
                                     _i64, _p]),
        "splitq_mocd_absmax": (C.c_int, [_p, C.c_int, _i64, _p, _i64, _i64, _p, _p, _p, _p]),
        "splitq_mocd_rank_counts": (C.c_int, [_p, C.c_int, _i64, _p, _p, _i64, _p, _i64, _p,
                                              _p]),
        "splitq_mocd_transpose_u16": (C.c_int, [_p, _i64, _i64, _p, _i64, _p]),
        "splitq_mocd_text_score": (C.c_int, [_p, _i64, _i64, _i64, C.c_int, C.c_int, _i64, _i64,
                                             _p, _p]),
        "splitq_mocd_topk": (C.c_int, [_p, _i64, _i64, _p, _p, _p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


EXPORTED_SYMBOLS = (
    "splitq_last_error", "splitq_version", "splitq_device_sm_count",
    "splitq_layer_create", "splitq_layer_destroy", "splitq_workspace_layout",
    "splitq_forward", "splitq_read_status", "splitq_profile_read", "splitq_quantize_rows", "splitq_gemm_i8",
    "splitq_mocd_absmax", "splitq_mocd_rank_counts", "splitq_mocd_transpose_u16",
    "splitq_mocd_text_score", "splitq_mocd_topk",
)


def check(rc: int) -> None:
    """Map a C status to the reference's exception types."""
    if rc == SPLITQ_OK:
        return
    msg = load().splitq_last_error().decode(errors="replace")
    if rc in (SPLITQ_ERR_INVALID, SPLITQ_ERR_UNSUPPORTED, SPLITQ_ERR_DATA):
        raise ValueError(msg)
    raise SplitqError(msg)
