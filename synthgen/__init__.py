"""Seeded synthetic inputs shared by the oracle side and the product side.

Holds none of the method's arithmetic (no products, no sums over k): it only
maps (seed, role, index) to matrix entries and hashes matrices.  The recipe is
in ``synthgen.c`` and DESIGN.md ("Input recipe"); it follows the paper's
Box-Muller generator (§IV "Experimental Dataset") for the
normal entries and BASELINE.json's configs for the uniform ones.

All matrices are dense row-major.  BF16 matrices are returned as
``numpy.uint16`` arrays holding raw bf16 bit patterns.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsynthgen.so")
_lib = None

ROLE_A, ROLE_B, ROLE_ROWS, ROLE_COLS = 1, 2, 3, 4

_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_vp = ctypes.c_void_p


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"{_LIB_PATH} missing: run `make` (or __graft_entry__.build())")
    lib = ctypes.CDLL(_LIB_PATH)
    for name in ("sg_gen_f64", "sg_gen_normal_f64"):
        getattr(lib, name).argtypes = [_u64, _u64, _i64, _i64, _vp]
    for name in ("sg_gen_i8", "sg_gen_bf16_normal"):
        getattr(lib, name).argtypes = [_u64, _u64, _i64, _i64, _vp]
    for name in ("sg_gen_exact_f64", "sg_gen_exact_bf16", "sg_gen_exact_i8"):
        getattr(lib, name).argtypes = [_u64, _u64, _u64, _i64, _i64, _vp]
    lib.sg_sample_indices.argtypes = [_u64, _u64, _i64, _i64, _vp]
    for name in ("sg_checksum_f64", "sg_checksum_f32", "sg_checksum_i32", "sg_checksum_bf16", "sg_checksum_i8"):
        getattr(lib, name).argtypes = [_vp, _i64]
        getattr(lib, name).restype = _u64
    for name in ("sg_fmix64",):
        getattr(lib, name).argtypes = [_u64]
        getattr(lib, name).restype = _u64
    lib.sg_key.argtypes = [_u64, _u64]
    lib.sg_key.restype = _u64
    lib.sg_word.argtypes = [_u64, _u64]
    lib.sg_word.restype = _u64
    lib.sg_bf16_from_double.argtypes = [ctypes.c_double]
    lib.sg_bf16_from_double.restype = ctypes.c_uint16
    for name in ("sg_checksum_f64_off", "sg_checksum_f32_off", "sg_checksum_f64_as_f32_off", "sg_checksum_i32_off"):
        getattr(lib, name).argtypes = [_vp, _i64, _i64]
        getattr(lib, name).restype = _u64
    lib.sg_box_muller.argtypes = [ctypes.c_double, ctypes.c_double, _vp, _vp]
    _lib = lib
    return lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def fmix64(z: int) -> int:
    return _load().sg_fmix64(z)


def key(seed: int, role: int) -> int:
    return _load().sg_key(seed, role)


def word(k: int, idx: int) -> int:
    return _load().sg_word(k, idx)


def bf16_from_double(x: float) -> int:
    """Single round-to-nearest-even double -> bf16 bit pattern (reading R9)."""
    return int(_load().sg_bf16_from_double(float(x)))


def box_muller(u1: float, u2: float) -> tuple[float, float]:
    """(Z0, Z1) of PAPER.md:162-167 for given uniforms in (0, 1)."""
    z0, z1 = ctypes.c_double(), ctypes.c_double()
    _load().sg_box_muller(u1, u2, ctypes.addressof(z0), ctypes.addressof(z1))
    return z0.value, z1.value


def uniform_f64(seed: int, role: int, rows: int, cols: int) -> np.ndarray:
    """FP64 entries i.i.d. uniform on [-1, 1) (BASELINE.json configs 0, 1, 4)."""
    out = np.empty((rows, cols), dtype=np.float64)
    _load().sg_gen_f64(seed, role, rows, cols, _ptr(out))
    return out


def normal_f64(seed: int, role: int, rows: int, cols: int) -> np.ndarray:
    """Unrounded Box-Muller doubles."""
    out = np.empty((rows, cols), dtype=np.float64)
    _load().sg_gen_normal_f64(seed, role, rows, cols, _ptr(out))
    return out


def normal_bf16(seed: int, role: int, rows: int, cols: int) -> np.ndarray:
    """Box-Muller normals rounded once (RNE) to bf16; raw uint16 bit patterns (config 3)."""
    out = np.empty((rows, cols), dtype=np.uint16)
    _load().sg_gen_bf16_normal(seed, role, rows, cols, _ptr(out))
    return out


def uniform_i8(seed: int, role: int, rows: int, cols: int) -> np.ndarray:
    """INT8 entries i.i.d. uniform on {-127..127} (BASELINE.json config 2)."""
    out = np.empty((rows, cols), dtype=np.int8)
    _load().sg_gen_i8(seed, role, rows, cols, _ptr(out))
    return out


def exact_f64(seed: int, role: int, K: int, rows: int, cols: int) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float64)
    _load().sg_gen_exact_f64(seed, role, K, rows, cols, _ptr(out))
    return out


def exact_bf16(seed: int, role: int, K: int, rows: int, cols: int) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.uint16)
    _load().sg_gen_exact_bf16(seed, role, K, rows, cols, _ptr(out))
    return out


def exact_i8(seed: int, role: int, K: int, rows: int, cols: int) -> np.ndarray:
    assert K <= 255
    out = np.empty((rows, cols), dtype=np.int8)
    _load().sg_gen_exact_i8(seed, role, K, rows, cols, _ptr(out))
    return out


def sample_indices(seed: int, role: int, count: int, limit: int) -> np.ndarray:
    out = np.empty(count, dtype=np.int64)
    _load().sg_sample_indices(seed, role, count, limit, _ptr(out))
    return out


def checksum(x: np.ndarray, kind: str | None = None) -> int:
    """Position-sensitive, order-free checksum."""
    x = np.ascontiguousarray(x)
    lib = _load()
    kind = kind or {np.dtype(np.float64): "f64", np.dtype(np.float32): "f32",
                    np.dtype(np.int32): "i32", np.dtype(np.uint16): "bf16",
                    np.dtype(np.int8): "i8"}[x.dtype]
    fn = {"f64": lib.sg_checksum_f64, "f32": lib.sg_checksum_f32, "i32": lib.sg_checksum_i32,
          "bf16": lib.sg_checksum_bf16, "i8": lib.sg_checksum_i8}[kind]
    return int(fn(_ptr(x), x.size))


def checksum_block(x: np.ndarray, offset: int, kind: str) -> int:
    """Checksum terms of a block whose first element has global row-major index `offset`
    (kind: "f64", "f32", or "f64_as_f32" for exactly-representable doubles stored as fp32)."""
    x = np.ascontiguousarray(x)
    lib = _load()
    fn = {"f64": lib.sg_checksum_f64_off, "f32": lib.sg_checksum_f32_off,
          "f64_as_f32": lib.sg_checksum_f64_as_f32_off, "i32": lib.sg_checksum_i32_off}[kind]
    return int(fn(_ptr(x), x.size, offset))


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    """Exact decode of bf16 bit patterns (bf16 is the top half of an fp32)."""
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
