"""ctypes binding of libmm_b200.so (include/mm.h).  Argument marshalling only:
every step of the product runs in the library's CUDA kernels.  The library is
required — there is no fallback path."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MM_B200_LIB") or os.path.join(_HERE, "libmm_b200.so")  # override: A/B builds

MM_F64, MM_BF16_F32, MM_S8_S32 = 0, 1, 2
MM_OK, MM_ERR_RUNTIME, MM_ERR_USAGE, MM_ERR_UNSUPPORTED, MM_ERR_WORKSPACE = 0, 1, 2, 3, 4
MM_ROW_BLOCK, MM_SUMMA_2D, MM_SUMMA_25D = 0, 1, 2
MM_BCAST_B, MM_GATHER_C, MM_GATHER_C_FUSED, MM_REPLICATE = 1, 2, 4, 8

# every symbol include/mm.h declares
EXPORTS = (
    "mm_create", "mm_destroy", "mm_gemm", "mm_gemm_host", "mm_sync_check", "mm_status_string",
    "mm_last_error", "mm_gemm_sharded", "mm_shard_range", "mm_summa_panels", "mm_launches", "mm_version",
)

_i64, _vp, _int, _uint, _sz = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_uint, ctypes.c_size_t
_lib = None


def load():
    """Load libmm_b200.so (raises if it is missing: the product has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                           "there is no non-CUDA fallback")
    lib = ctypes.CDLL(LIB_PATH)
    lib.mm_create.argtypes = [_int, _vp, _sz, ctypes.POINTER(_vp)]
    lib.mm_create.restype = _int
    lib.mm_destroy.argtypes = [_vp]
    lib.mm_destroy.restype = None
    lib.mm_gemm.argtypes = [_vp, _i64, _i64, _i64, _int, _vp, _vp, _vp, _vp]
    lib.mm_gemm.restype = _int
    lib.mm_gemm_host.argtypes = [_vp, _i64, _i64, _i64, _int, _vp, _vp, _vp, _vp]
    lib.mm_gemm_host.restype = _int
    lib.mm_sync_check.argtypes = [_vp, _vp]
    lib.mm_sync_check.restype = _int
    lib.mm_status_string.argtypes = [_int]
    lib.mm_status_string.restype = ctypes.c_char_p
    lib.mm_last_error.argtypes = [_vp]
    lib.mm_last_error.restype = ctypes.c_char_p
    lib.mm_gemm_sharded.argtypes = [_vp, _i64, _i64, _i64, _int, _int, _int, _int, _vp, _vp, _vp, _vp, _uint, _int,
                                    _vp, _vp]
    lib.mm_gemm_sharded.restype = _int
    lib.mm_shard_range.argtypes = [_i64, _int, _int, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
    lib.mm_shard_range.restype = None
    lib.mm_summa_panels.argtypes = [_i64, _int, _int, _i64, _int, _vp, _vp, _vp, _vp]
    lib.mm_summa_panels.restype = _int
    lib.mm_launches.argtypes = [_vp]
    lib.mm_launches.restype = ctypes.c_uint64
    lib.mm_version.argtypes = []
    lib.mm_version.restype = ctypes.c_char_p
    _lib = lib
    return lib
