"""ctypes binding of libmm_b200.so (include/mm.h).  Argument marshalling only:
every step of the product runs in the library's CUDA kernels.  The library is
required — there is no fallback path."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MM_B200_LIB") or os.path.join(_HERE, "libmm_b200.so")  # override: A/B builds

MM_F64, MM_BF16_F32, MM_S8_S32, MM_F64_EMU = 0, 1, 2, 3
MM_OK, MM_ERR_RUNTIME, MM_ERR_USAGE, MM_ERR_UNSUPPORTED, MM_ERR_WORKSPACE = 0, 1, 2, 3, 4
MM_ROW_BLOCK, MM_SUMMA_2D, MM_SUMMA_25D = 0, 1, 2
MM_BCAST_B, MM_GATHER_C, MM_GATHER_C_FUSED, MM_REPLICATE, MM_C_WINDOW = 1, 2, 4, 8, 16

# every symbol include/mm.h declares
EXPORTS = (
    "mm_create", "mm_destroy", "mm_gemm", "mm_gemm_host", "mm_sync_check", "mm_status_string",
    "mm_last_error", "mm_gemm_sharded", "mm_shard_range", "mm_summa_panels", "mm_launches", "mm_version",
    "mm_shard_plan", "mm_workspace_size", "mm_ipc_export", "mm_ipc_open", "mm_clock_meter",
    "mm_window_alloc", "mm_window_free", "mm_f64_emu_plan",
)

# mm_plan_op / mm_plan_buf / mm_plan_comm (include/mm.h)
OPS = {1: "GEMM", 2: "COPY2D", 3: "BCAST", 4: "SEND", 5: "RECV", 6: "GROUP_START", 7: "GROUP_END", 8: "REDUCE_SUM",
       9: "MEMSET0", 10: "BARRIER", 11: "MAP_PEER", 12: "RECORD", 13: "WAIT"}
BUFS = {0: None, 1: "A", 2: "B", 3: "C", 4: "CFULL", 5: "CPEER", 6: "S0", 7: "S1", 8: "S2", 9: "S3"}
COMMS = {0: "WORLD", 1: "ROW", 2: "COL", 3: "DEPTH"}


class PlanStep(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("stream", ctypes.c_int32), ("comm", ctypes.c_int32), ("peer", ctypes.c_int32),
                ("dst", ctypes.c_int32), ("src", ctypes.c_int32), ("src2", ctypes.c_int32), ("beta", ctypes.c_int32),
                ("dst_off", ctypes.c_int64), ("src_off", ctypes.c_int64), ("src2_off", ctypes.c_int64),
                ("dst_ld", ctypes.c_int64), ("src_ld", ctypes.c_int64), ("src2_ld", ctypes.c_int64),
                ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("p", ctypes.c_int64),
                ("event", ctypes.c_int32), ("overlap", ctypes.c_int32)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_int32), ("events", ctypes.c_int32), ("color", ctypes.c_int32 * 4),
                ("key", ctypes.c_int32 * 4), ("stage_bytes", ctypes.c_int64 * 4)]


class IpcHandle(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_ubyte * 72)]

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
    lib.mm_shard_plan.argtypes = [_i64, _i64, _i64, _int, _int, _int, _int, _uint, _int, _int, _int, _i64,
                                  ctypes.POINTER(PlanStep), _int, ctypes.POINTER(PlanInfo)]
    lib.mm_shard_plan.restype = _int
    lib.mm_workspace_size.argtypes = [_i64, _i64, _i64, _int, _int, _int]
    lib.mm_workspace_size.restype = _sz
    lib.mm_ipc_export.argtypes = [_vp, _vp, ctypes.POINTER(IpcHandle)]
    lib.mm_ipc_export.restype = _int
    lib.mm_ipc_open.argtypes = [_vp, ctypes.POINTER(IpcHandle), ctypes.POINTER(_vp)]
    lib.mm_ipc_open.restype = _int
    lib.mm_window_alloc.argtypes = [_vp, _vp, ctypes.c_size_t, ctypes.POINTER(_vp)]
    lib.mm_window_alloc.restype = _int
    lib.mm_window_free.argtypes = [_vp, _vp]
    lib.mm_window_free.restype = _int
    lib.mm_clock_meter.argtypes = [_vp, _int, ctypes.POINTER(ctypes.c_double)]
    lib.mm_clock_meter.restype = _int
    lib.mm_f64_emu_plan.argtypes = [_i64, ctypes.POINTER(_int), ctypes.POINTER(_int), ctypes.POINTER(_int)]
    lib.mm_f64_emu_plan.restype = _int
    lib.mm_version.argtypes = []
    lib.mm_version.restype = ctypes.c_char_p
    _lib = lib
    return lib
