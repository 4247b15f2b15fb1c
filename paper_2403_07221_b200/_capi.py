"""ctypes binding of the C-ABI in include/lffn_gpu.h (liblffn_gpu.so).

This is the same binding a Python user of the reference would add (see
INTEGRATION.md).  The library is loaded from the package's ``csrc/``
directory; there is no fallback -- if the shared object is missing or the
device is not a B200 the calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "csrc", "liblffn_gpu.so")

LFFN_OK, LFFN_ERR_USAGE, LFFN_ERR_NUMERIC, LFFN_ERR_RUNTIME = 0, 1, 2, 3
LFFN_CLASS_SIZE, LFFN_CLASS_USAGE, LFFN_CLASS_NUMERIC, LFFN_CLASS_RUNTIME = 1, 2, 3, 4
LFFN_F32, LFFN_BF16, LFFN_F64 = 0, 1, 2
LFFN_OPT_DENSE_EXACT, LFFN_OPT_TABLE_GROUP_BYTES, LFFN_OPT_GATHER_VARIANT = 1, 2, 3
LFFN_OPT_BF16_COEFF_FMA, LFFN_OPT_BWD_ONE_PASS, LFFN_OPT_HASH_EXACT, LFFN_OPT_HOST_CHUNKS = 5, 6, 7, 8
LFFN_COMBINE_REDUCE_SCATTER, LFFN_COMBINE_ALL_REDUCE, LFFN_COMBINE_NONE = 0, 1, 2
LFFN_OPT_SMALL_MAX_TOKENS, LFFN_OPT_GATHER_SMS, LFFN_OPT_HOST_DIRECT = 10, 11, 12


class lffn_cfg(C.Structure):
    _fields_ = [("d_in", C.c_int64), ("d_out", C.c_int64), ("tables", C.c_int64),
                ("code_bits", C.c_int64), ("variant", C.c_int32), ("neighbor_count", C.c_int32)]


class lffn_proj(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("d_in", C.c_int64),
                ("d_out", C.c_int64), ("stages", C.c_int64), ("block", C.c_int64),
                ("depth", C.c_int64), ("blob", C.POINTER(C.c_double)), ("blob_len", C.c_int64)]


_VP = C.c_void_p
_I64 = C.c_int64

# name -> (restype, argtypes); every function declared in include/lffn_gpu.h
SIGNATURES = {
    "lffn_cfg_validate": (C.c_int, [C.POINTER(lffn_cfg)]),
    "lffn_proj_validate": (C.c_int, [C.POINTER(lffn_proj)]),
    "lffn_transform_width": (_I64, [C.POINTER(lffn_proj)]),
    "lffn_proj_blob_size": (_I64, [C.POINTER(lffn_proj)]),
    "lffn_proj_init": (C.c_int, [C.POINTER(lffn_proj), C.c_uint64, _VP]),
    "lffn_fill_gaussian": (C.c_int, [C.c_uint64, _VP, _I64, C.c_double]),
    "lffn_fill_gaussian_slice": (C.c_int, [C.c_uint64, _I64, _VP, _I64, C.c_double]),
    "lffn_fill_signs": (C.c_int, [C.c_uint64, _VP, _I64]),
    "lffn_tables_init": (C.c_int, [C.POINTER(lffn_cfg), C.c_uint64, _VP]),
    "lffn_convert": (C.c_int, [_VP, C.c_int, _VP, C.c_int, _I64]),
    "lffn_checkpoint_header": (C.c_int, [C.c_char_p, C.POINTER(lffn_cfg), C.POINTER(lffn_proj),
                                         C.POINTER(_I64)]),
    "lffn_checkpoint_load": (C.c_int, [C.c_char_p, _VP, _VP]),
    "lffn_checkpoint_save": (C.c_int, [C.c_char_p, C.POINTER(lffn_cfg), C.POINTER(lffn_proj), _VP]),
    "lffn_ctx_create_from_checkpoint": (C.c_int, [C.POINTER(_VP), C.c_int, _I64, C.c_char_p,
                                                  C.c_int, _I64, _I64]),
    "lffn_ctx_create": (C.c_int, [C.POINTER(_VP), C.c_int, _I64, C.POINTER(lffn_cfg),
                                  C.POINTER(lffn_proj)]),
    "lffn_ctx_create_shard": (C.c_int, [C.POINTER(_VP), C.c_int, _I64, C.POINTER(lffn_cfg),
                                        C.POINTER(lffn_proj), _I64, _I64]),
    "lffn_ctx_destroy": (C.c_int, [_VP]),
    "lffn_ctx_table_range": (C.c_int, [_VP, C.POINTER(_I64), C.POINTER(_I64)]),
    "lffn_tables_upload": (C.c_int, [_VP, _VP, C.c_int, C.c_int]),
    "lffn_tables_upload_slice": (C.c_int, [_VP, _VP, C.c_int, C.c_int]),
    "lffn_tables_attach": (C.c_int, [_VP, _VP, C.c_int]),
    "lffn_hash": (C.c_int, [_VP, _VP, _I64, _VP, _VP, _VP, _VP]),
    "lffn_lookup_accumulate": (C.c_int, [_VP, _VP, _VP, _I64, _VP, C.c_int, _VP]),
    "lffn_forward": (C.c_int, [_VP, _VP, _I64, _VP, _VP]),
    "lffn_forward_host": (C.c_int, [_VP, _VP, _I64, _VP]),
    "lffn_backward": (C.c_int, [_VP, _VP, _VP, _I64, _VP, _VP, _VP, _VP]),
    "lffn_proj_backward": (C.c_int, [_VP, _VP, _VP, _I64, _VP, _VP, _VP]),
    "lffn_sync": (C.c_int, [_VP, _VP]),
    "lffn_ctx_set_option": (C.c_int, [_VP, C.c_int, _I64]),
    "lffn_ctx_launch_count": (_I64, [_VP]),
    "lffn_ctx_set_timing": (C.c_int, [_VP, C.c_int]),
    "lffn_ctx_stage_ms": (C.c_int, [_VP, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "lffn_probe_bandwidth": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "lffn_last_error": (C.c_char_p, []),
    "lffn_last_error_class": (C.c_int, []),
    "lffn_version": (C.c_char_p, []),
    "lffn_nccl_unique_id": (C.c_int, [_VP, _I64]),
    "lffn_group_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, _I64, C.POINTER(lffn_cfg),
                                    C.POINTER(lffn_proj), _VP, C.c_int, C.c_int]),
    "lffn_group_destroy": (C.c_int, [_VP]),
    "lffn_group_shard": (_VP, [_VP]),
    "lffn_group_set_chunks": (C.c_int, [_VP, C.c_int]),
    "lffn_forward_sharded": (C.c_int, [_VP, _VP, _I64, _VP, C.c_int, _VP]),
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load liblffn_gpu.so once; raise (never fall back) when it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `make -C paper_2403_07221_b200/csrc` "
                    "or __graft_entry__.build(); there is no CPU fallback")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


class LffnError(Exception):
    """Base of the errors mapped from C-ABI status codes."""


class ValidationError(LffnError, ValueError):
    """Status 1: the reference's std::invalid_argument family (common.hpp:17-23)."""


class SizeError(ValidationError):
    """SizeError analog: shape / size checks (lffn_last_error_class() == SIZE)."""


class UsageError(ValidationError):
    """UsageError analog: unknown names, checkpoint I/O, wrong call order."""


class NumericError(LffnError, ArithmeticError):
    """NumericError analog (status 2; common.hpp:27-29): non-finite stage."""


class DeviceError(LffnError, RuntimeError):
    """CUDA runtime failure (status 3)."""


def check(rc: int) -> None:
    if rc == LFFN_OK:
        return
    msg = lib().lffn_last_error().decode(errors="replace")
    if rc == LFFN_ERR_USAGE:
        raise (SizeError if lib().lffn_last_error_class() == LFFN_CLASS_SIZE else UsageError)(msg)
    if rc == LFFN_ERR_NUMERIC:
        raise NumericError(msg)
    raise DeviceError(msg)
