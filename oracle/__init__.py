"""CPU oracle for the dense product C = A·B (§III).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2408_15384_b200`` (the CUDA path),
and the CUDA path never imports it.

The arithmetic lives in ``mmref.c`` (plain loops, k ascending, one
accumulator per element, built ``-O3 -fopenmp -ffp-contract=off``); this
module only marshals numpy arrays.  Every function cites the passage it
follows in ``mmref.c``'s header.

Pins (tests/test_oracle.py): hand-worked products (BASELINE.json north_star's
2×3·3×2; SPEC.md:183 2×2; SPEC.md:195 1×1), identity and zero matrices
(SPEC.md:184-185), the transpose invariant (AB)ᵀ = BᵀAᵀ, brute force against
exact Python integers / ``fractions.Fraction`` on tiny inputs, closed forms
(all-ones, rank-1), the i-j-k ≡ i-k-j bit identity, the FP error bound
γ_n·D against the exactly rounded sum (``math.fsum``), and the SURVEY.md §8
c6/c7 golden values computed by two independent implementations.
No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
_i64, _vp = ctypes.c_int64, ctypes.c_void_p


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"{_LIB_PATH} missing: run `make` (or __graft_entry__.build())")
    lib = ctypes.CDLL(_LIB_PATH)
    for name in ("mmref_f64_ijk", "mmref_f64", "mmref_f64_absden", "mmref_s8"):
        getattr(lib, name).argtypes = [_i64, _i64, _i64, _vp, _vp, _vp]
    lib.mmref_bf16.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp, _vp]
    for name in ("mmref_f64_rows", "mmref_f64_cols", "mmref_bf16_rows", "mmref_bf16_cols"):
        getattr(lib, name).argtypes = [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp]
    lib.mmref_s8_rows.argtypes = [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp]
    lib.mmref_max_threads.restype = ctypes.c_int
    _lib = lib
    return lib


def _c(a, dtype):
    a = np.ascontiguousarray(a)
    assert a.dtype == dtype, (a.dtype, dtype)
    return a


def _shapes(A, B):
    assert A.ndim == 2 and B.ndim == 2 and A.shape[1] == B.shape[0], (A.shape, B.shape)
    return A.shape[0], A.shape[1], B.shape[1]


def max_threads() -> int:
    return int(_load().mmref_max_threads())


def gemm_f64_ijk(A, B):
    """Literal i-j-k definition."""
    A, B = _c(A, np.float64), _c(B, np.float64)
    m, n, p = _shapes(A, B)
    C = np.empty((m, p), np.float64)
    _load().mmref_f64_ijk(m, n, p, A.ctypes.data, B.ctypes.data, C.ctypes.data)
    return C


def gemm_f64(A, B):
    """C = A·B in double, k ascending, unfused."""
    A, B = _c(A, np.float64), _c(B, np.float64)
    m, n, p = _shapes(A, B)
    C = np.empty((m, p), np.float64)
    _load().mmref_f64(m, n, p, A.ctypes.data, B.ctypes.data, C.ctypes.data)
    return C


def absden_f64(A, B):
    """D[i][j] = Σ_k |A[i][k]·B[k][j]| — BASELINE.json north_star's normaliser."""
    A, B = _c(A, np.float64), _c(B, np.float64)
    m, n, p = _shapes(A, B)
    D = np.empty((m, p), np.float64)
    _load().mmref_f64_absden(m, n, p, A.ctypes.data, B.ctypes.data, D.ctypes.data)
    return D


def gemm_f64_rows(A, B, rows):
    A, B = _c(A, np.float64), _c(B, np.float64)
    m, n, p = _shapes(A, B)
    rows = _c(np.asarray(rows, np.int64), np.int64)
    assert rows.size == 0 or (rows.min() >= 0 and rows.max() < m)
    C = np.empty((rows.size, p), np.float64)
    D = np.empty((rows.size, p), np.float64)
    _load().mmref_f64_rows(m, n, p, A.ctypes.data, B.ctypes.data, rows.size, rows.ctypes.data,
                           C.ctypes.data, D.ctypes.data)
    return C, D


def gemm_f64_cols(A, B, cols):
    A, B = _c(A, np.float64), _c(B, np.float64)
    m, n, p = _shapes(A, B)
    cols = _c(np.asarray(cols, np.int64), np.int64)
    assert cols.size == 0 or (cols.min() >= 0 and cols.max() < p)
    C = np.empty((m, cols.size), np.float64)
    D = np.empty((m, cols.size), np.float64)
    _load().mmref_f64_cols(m, n, p, A.ctypes.data, B.ctypes.data, cols.size, cols.ctypes.data,
                           C.ctypes.data, D.ctypes.data)
    return C, D


def gemm_bf16(A_bits, B_bits):
    """bf16 inputs (raw uint16 bits), exact decode, double accumulation. Returns (C, D)."""
    A, B = _c(A_bits, np.uint16), _c(B_bits, np.uint16)
    m, n, p = _shapes(A, B)
    C = np.empty((m, p), np.float64)
    D = np.empty((m, p), np.float64)
    _load().mmref_bf16(m, n, p, A.ctypes.data, B.ctypes.data, C.ctypes.data, D.ctypes.data)
    return C, D


def gemm_bf16_rows(A_bits, B_bits, rows):
    A, B = _c(A_bits, np.uint16), _c(B_bits, np.uint16)
    m, n, p = _shapes(A, B)
    rows = _c(np.asarray(rows, np.int64), np.int64)
    assert rows.size == 0 or (rows.min() >= 0 and rows.max() < m)
    C = np.empty((rows.size, p), np.float64)
    D = np.empty((rows.size, p), np.float64)
    _load().mmref_bf16_rows(m, n, p, A.ctypes.data, B.ctypes.data, rows.size, rows.ctypes.data,
                            C.ctypes.data, D.ctypes.data)
    return C, D


def gemm_bf16_cols(A_bits, B_bits, cols):
    A, B = _c(A_bits, np.uint16), _c(B_bits, np.uint16)
    m, n, p = _shapes(A, B)
    cols = _c(np.asarray(cols, np.int64), np.int64)
    assert cols.size == 0 or (cols.min() >= 0 and cols.max() < p)
    C = np.empty((m, cols.size), np.float64)
    D = np.empty((m, cols.size), np.float64)
    _load().mmref_bf16_cols(m, n, p, A.ctypes.data, B.ctypes.data, cols.size, cols.ctypes.data,
                            C.ctypes.data, D.ctypes.data)
    return C, D


def gemm_s8(A, B):
    """Exact integer product of int8 matrices (int64 result)."""
    A, B = _c(A, np.int8), _c(B, np.int8)
    m, n, p = _shapes(A, B)
    C = np.empty((m, p), np.int64)
    _load().mmref_s8(m, n, p, A.ctypes.data, B.ctypes.data, C.ctypes.data)
    return C


def gemm_s8_rows(A, B, rows):
    A, B = _c(A, np.int8), _c(B, np.int8)
    m, n, p = _shapes(A, B)
    rows = _c(np.asarray(rows, np.int64), np.int64)
    C = np.empty((rows.size, p), np.int64)
    _load().mmref_s8_rows(m, n, p, A.ctypes.data, B.ctypes.data, rows.size, rows.ctypes.data, C.ctypes.data)
    return C


def normalized_error(C_test, C_ref, D):
    """max_ij |C_test − C_ref| / D_ij (BASELINE.json north_star; reading R1-R3).

    D_ij = 0 ⇒ the exact result is 0, so the element must be exactly ±0 (error 0, else inf).
    Any NaN/Inf in C_test fails (returns inf)."""
    C_test = np.asarray(C_test, np.float64)
    C_ref = np.asarray(C_ref, np.float64)
    D = np.asarray(D, np.float64)
    if not np.all(np.isfinite(C_test)):
        return float("inf")
    diff = np.abs(C_test - C_ref)
    zero = D == 0
    if np.any(diff[zero] != 0):
        return float("inf")
    with np.errstate(divide="ignore", invalid="ignore"):
        err = np.where(zero, 0.0, diff / np.where(zero, 1.0, D))
    return float(err.max()) if err.size else 0.0
