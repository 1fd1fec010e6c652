"""GPU evaluation of the synthgen recipe (libsynthgen_cuda.so): the same matrices as
synthgen's host generator, created directly in device memory.
Returns torch tensors; bf16 matrices come back as torch.bfloat16."""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsynthgen_cuda.so")
_lib = None

F64, I8, BF16_NORMAL, EXACT_F64, EXACT_BF16 = 0, 1, 2, 3, 4


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `make`")
        lib = ctypes.CDLL(_LIB_PATH)
        lib.sgc_generate.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        lib.sgc_generate.restype = ctypes.c_int
        _lib = lib
    return _lib


def _gen(kind, seed, role, K, rows, cols, dtype, device):
    out = torch.empty(rows, cols, dtype=dtype, device=device)
    st = _load().sgc_generate(kind, seed, role, K, rows, cols, out.data_ptr(),
                              torch.cuda.current_stream(out.device).cuda_stream)
    if st != 0:
        raise RuntimeError(f"sgc_generate failed ({st})")
    return out


def uniform_f64(seed, role, rows, cols, device="cuda"):
    return _gen(F64, seed, role, 0, rows, cols, torch.float64, device)


def uniform_i8(seed, role, rows, cols, device="cuda"):
    return _gen(I8, seed, role, 0, rows, cols, torch.int8, device)


def normal_bf16(seed, role, rows, cols, device="cuda"):
    return _gen(BF16_NORMAL, seed, role, 0, rows, cols, torch.bfloat16, device)


def exact_f64(seed, role, K, rows, cols, device="cuda"):
    return _gen(EXACT_F64, seed, role, K, rows, cols, torch.float64, device)


def exact_bf16(seed, role, K, rows, cols, device="cuda"):
    return _gen(EXACT_BF16, seed, role, K, rows, cols, torch.bfloat16, device)
