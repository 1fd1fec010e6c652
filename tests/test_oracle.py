"""Pins for the CPU oracle (oracle/mmref.c) — every check is against something
other than the oracle itself: hand-worked values, closed forms, exact rational
arithmetic, the FP error bound, library integer arithmetic, or SURVEY.md's
independently computed golden values.  CPU only."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synthgen as sg

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
U = 2.0 ** -53  # unit roundoff of binary64


def to_bf16_bits(x):
    x = np.asarray(x, np.float64)
    return np.vectorize(sg.bf16_from_double, otypes=[np.uint16])(x).reshape(x.shape)


def run(dtype, A, B):
    """Oracle product in `dtype` from float64 arrays holding exactly-representable values."""
    A = np.asarray(A, np.float64)
    B = np.asarray(B, np.float64)
    if dtype == "f64":
        return oracle.gemm_f64(A, B)
    if dtype == "bf16":
        C, _ = oracle.gemm_bf16(to_bf16_bits(A), to_bf16_bits(B))
        return C
    if dtype == "s8":
        return oracle.gemm_s8(A.astype(np.int8), B.astype(np.int8)).astype(np.float64)
    raise ValueError(dtype)


# ---------------------------------------------------------------- hand-worked
with open(os.path.join(GOLDEN, "handworked.json")) as f:
    HAND = json.load(f)["cases"]


@pytest.mark.parametrize("case", HAND, ids=[c["name"] for c in HAND])
def test_handworked(case):
    for dt in case["dtypes"]:
        C = run(dt, case["A"], case["B"])
        assert np.array_equal(C, np.asarray(case["C"], np.float64)), (dt, C)


@pytest.mark.parametrize("case", HAND, ids=[c["name"] for c in HAND])
def test_handworked_ijk_literal(case):
    C = oracle.gemm_f64_ijk(np.asarray(case["A"], np.float64), np.asarray(case["B"], np.float64))
    assert np.array_equal(C, np.asarray(case["C"], np.float64))


# ------------------------------------------------------- identity / zero
@pytest.mark.parametrize("m,n", [(1, 1), (3, 5), (17, 33), (64, 48)])
def test_identity_and_zero(m, n):
    A = sg.uniform_f64(11, 1, m, n)
    I_n = np.eye(n)
    I_m = np.eye(m)
    assert np.array_equal(oracle.gemm_f64(A, I_n), A)
    assert np.array_equal(oracle.gemm_f64(I_m, A), A)
    Z = oracle.gemm_f64(A, np.zeros((n, 7)))
    assert np.array_equal(Z, np.zeros((m, 7)))
    # bf16
    Ab = sg.normal_bf16(11, 1, m, n)
    C, D = oracle.gemm_bf16(Ab, to_bf16_bits(I_n))
    assert np.array_equal(C, sg.bf16_bits_to_f64(Ab))
    assert np.array_equal(D, np.abs(sg.bf16_bits_to_f64(Ab)))
    C, _ = oracle.gemm_bf16(to_bf16_bits(I_m), Ab)
    assert np.array_equal(C, sg.bf16_bits_to_f64(Ab))
    # s8
    As = sg.uniform_i8(11, 1, m, n)
    assert np.array_equal(oracle.gemm_s8(As, np.eye(n, dtype=np.int8)), As.astype(np.int64))
    assert np.array_equal(oracle.gemm_s8(np.eye(m, dtype=np.int8), As), As.astype(np.int64))
    assert not oracle.gemm_s8(As, np.zeros((n, 5), np.int8)).any()


# ------------------------------------------------ transpose invariant (AB)^T = B^T A^T
@pytest.mark.parametrize("m,n,p", [(1, 1, 1), (2, 3, 4), (31, 17, 45), (64, 100, 33)])
def test_transpose_invariant(m, n, p):
    A = sg.uniform_f64(5, 1, m, n)
    B = sg.uniform_f64(5, 2, n, p)
    C = oracle.gemm_f64(A, B)
    Ct = oracle.gemm_f64(np.ascontiguousarray(B.T), np.ascontiguousarray(A.T))
    # same products, same k order, and IEEE multiply commutes -> bit-identical
    assert np.array_equal(C.T, Ct)
    As, Bs = sg.uniform_i8(5, 1, m, n), sg.uniform_i8(5, 2, n, p)
    assert np.array_equal(oracle.gemm_s8(As, Bs).T,
                          oracle.gemm_s8(np.ascontiguousarray(Bs.T), np.ascontiguousarray(As.T)))
    Ab, Bb = sg.normal_bf16(5, 1, m, n), sg.normal_bf16(5, 2, n, p)
    C1, D1 = oracle.gemm_bf16(Ab, Bb)
    C2, D2 = oracle.gemm_bf16(np.ascontiguousarray(Bb.T), np.ascontiguousarray(Ab.T))
    assert np.array_equal(C1.T, C2) and np.array_equal(D1.T, D2)


# --------------------------------------------------------- brute force, exact
def _exact_product(A, B):
    m, n = len(A), len(A[0])
    p = len(B[0])
    return [[sum((Fraction(A[i][k]) * Fraction(B[k][j]) for k in range(n)), Fraction(0))
             for j in range(p)] for i in range(m)]


def test_bruteforce_all_tiny_shapes_exact_ints():
    """Every (m,n,p) in {1..8}^3 with integer entries: exact."""
    rng = np.random.default_rng(1234)
    for m in range(1, 9):
        for n in range(1, 9):
            for p in range(1, 9):
                A = rng.integers(-127, 128, (m, n))
                B = rng.integers(-127, 128, (n, p))
                exact = np.array([[sum(int(A[i, k]) * int(B[k, j]) for k in range(n))
                                   for j in range(p)] for i in range(m)], dtype=np.int64)
                assert np.array_equal(oracle.gemm_s8(A.astype(np.int8), B.astype(np.int8)), exact)
                assert np.array_equal(oracle.gemm_f64(A.astype(float), B.astype(float)), exact)
                C, _ = oracle.gemm_bf16(to_bf16_bits(A), to_bf16_bits(B))
                # |entries| <= 127 are exact in bf16 only if they have <= 8 significant bits: all are
                assert np.array_equal(C, exact)


@pytest.mark.parametrize("m,n,p", [(3, 7, 5), (8, 64, 8), (4, 1000, 3)])
def test_fp64_within_error_bound_of_exact_sum(m, n, p):
    """Sequential summation error bound |C - exact| <= gamma_n * D (Higham, gamma_n = nu/(1-nu)).
    A dropped, doubled or sign-flipped term violates it by orders of magnitude."""
    A = sg.uniform_f64(7, 1, m, n)
    B = sg.uniform_f64(7, 2, n, p)
    C = oracle.gemm_f64(A, B)
    D = oracle.absden_f64(A, B)
    gamma = n * U / (1 - n * U)
    ex = _exact_product(A.tolist(), B.tolist())
    for i in range(m):
        for j in range(p):
            err = abs(Fraction(C[i, j]) - ex[i][j])
            assert err <= Fraction(gamma) * Fraction(D[i, j]), (i, j)
            # D is the exact sum of |products| up to the same bound
            exD = sum(abs(Fraction(A[i, k]) * Fraction(B[k, j])) for k in range(n))
            assert abs(Fraction(D[i, j]) - exD) <= Fraction(gamma) * exD


def test_bf16_products_exact_and_sum_bounded():
    """bf16 products are exact in double; the oracle's error vs math.fsum is within gamma_n*D."""
    m, n, p = 5, 2048, 6
    A = sg.normal_bf16(8, 1, m, n)
    B = sg.normal_bf16(8, 2, n, p)
    C, D = oracle.gemm_bf16(A, B)
    Af, Bf = sg.bf16_bits_to_f64(A), sg.bf16_bits_to_f64(B)
    gamma = n * U / (1 - n * U)
    for i in range(m):
        for j in range(p):
            terms = [Af[i, k] * Bf[k, j] for k in range(n)]
            for k in range(0, n, 97):  # products exact: reconstruct as Fractions
                assert Fraction(terms[k]) == Fraction(Af[i, k]) * Fraction(Bf[k, j])
            exact = math.fsum(terms)
            assert abs(C[i, j] - exact) <= gamma * D[i, j] + abs(exact) * U


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("m,n,p", [(1, 1, 1), (5, 300, 7), (33, 1025, 17)])
def test_all_ones_closed_form(m, n, p):
    for dt in ("f64", "bf16", "s8"):
        C = run(dt, np.ones((m, n)), np.ones((n, p)))
        assert np.all(C == n), dt


def test_rank_one_closed_form():
    m, n, p = 9, 77, 13
    x = np.arange(-4, m - 4, dtype=float)
    z = np.arange(-6, p - 6, dtype=float)
    A = np.repeat(x[:, None], n, axis=1)
    B = np.repeat(z[None, :], n, axis=0)
    for dt in ("f64", "bf16", "s8"):
        C = run(dt, A, B)
        assert np.array_equal(C, n * np.outer(x, z)), dt


# ------------------------------------------- loop-order identity (E12 / DESIGN R5)
@pytest.mark.parametrize("m,n,p", [(1, 1, 1), (17, 129, 33), (128, 256, 96)])
def test_ijk_equals_ikj_bitwise(m, n, p):
    A = sg.uniform_f64(9, 1, m, n)
    B = sg.uniform_f64(9, 2, n, p)
    assert np.array_equal(oracle.gemm_f64_ijk(A, B), oracle.gemm_f64(A, B))


def test_sampled_variants_match_full():
    m, n, p = 70, 90, 110
    A, B = sg.uniform_f64(3, 1, m, n), sg.uniform_f64(3, 2, n, p)
    C = oracle.gemm_f64(A, B)
    D = oracle.absden_f64(A, B)
    rows = np.array([0, 5, 69, 5])
    cols = np.array([109, 0, 50])
    Cr, Dr = oracle.gemm_f64_rows(A, B, rows)
    Cc, Dc = oracle.gemm_f64_cols(A, B, cols)
    assert np.array_equal(Cr, C[rows]) and np.array_equal(Dr, D[rows])
    assert np.array_equal(Cc, C[:, cols]) and np.array_equal(Dc, D[:, cols])
    Ab, Bb = sg.normal_bf16(3, 1, m, n), sg.normal_bf16(3, 2, n, p)
    Cb, Db = oracle.gemm_bf16(Ab, Bb)
    Cr, Dr = oracle.gemm_bf16_rows(Ab, Bb, rows)
    Cc, Dc = oracle.gemm_bf16_cols(Ab, Bb, cols)
    assert np.array_equal(Cr, Cb[rows]) and np.array_equal(Dr, Db[rows])
    assert np.array_equal(Cc, Cb[:, cols]) and np.array_equal(Dc, Db[:, cols])
    As, Bs = sg.uniform_i8(3, 1, m, n), sg.uniform_i8(3, 2, n, p)
    assert np.array_equal(oracle.gemm_s8_rows(As, Bs, rows), oracle.gemm_s8(As, Bs)[rows])


def test_s8_matches_numpy_integer_matmul():
    """numpy's int64 matmul is exact integer arithmetic (independent implementation)."""
    A, B = sg.uniform_i8(2, 1, 300, 500), sg.uniform_i8(2, 2, 500, 200)
    assert np.array_equal(oracle.gemm_s8(A, B), A.astype(np.int64) @ B.astype(np.int64))


def test_bf16_oracle_agrees_with_f64_oracle_on_decoded_inputs():
    A, B = sg.normal_bf16(4, 1, 40, 300), sg.normal_bf16(4, 2, 300, 50)
    C, D = oracle.gemm_bf16(A, B)
    Af, Bf = sg.bf16_bits_to_f64(A), sg.bf16_bits_to_f64(B)
    assert np.array_equal(C, oracle.gemm_f64(Af, Bf))
    assert np.array_equal(D, oracle.absden_f64(Af, Bf))


# -------------------------------------------------------- normalized error metric
def test_normalized_error_rules():
    C_ref = np.array([[1.0, 0.0]])
    D = np.array([[2.0, 0.0]])
    assert oracle.normalized_error(np.array([[1.5, 0.0]]), C_ref, D) == 0.25
    assert oracle.normalized_error(np.array([[1.0, -0.0]]), C_ref, D) == 0.0
    assert oracle.normalized_error(np.array([[1.0, 1e-300]]), C_ref, D) == math.inf
    assert oracle.normalized_error(np.array([[np.nan, 0.0]]), C_ref, D) == math.inf


# ----------------------------------------------------- SURVEY.md §8 c6 goldens
with open(os.path.join(GOLDEN, "survey_c6.json")) as f:
    C6 = json.load(f)


def _h(s):
    return int(s, 16)


def test_golden_C1_full():
    g = C6["C1"]
    A = sg.uniform_f64(g["seed"], 1, 256, 256)
    B = sg.uniform_f64(g["seed"], 2, 256, 256)
    C = oracle.gemm_f64(A, B)
    assert sg.checksum(C) == _h(g["csC"])
    assert C[0, 0] == g["C00"] and C[-1, -1] == g["Clast"]


def test_golden_C2_full():
    g = C6["C2"]
    A = sg.uniform_f64(g["seed"], 1, g["m"], g["n"])
    B = sg.uniform_f64(g["seed"], 2, g["n"], g["p"])
    C = oracle.gemm_f64(A, B)
    assert sg.checksum(C) == _h(g["csC"])
    assert C[0, 0] == g["C00"] and C[-1, -1] == g["Clast"]


def test_golden_C3_full():
    g = C6["C3"]
    A = sg.uniform_i8(g["seed"], 1, 4096, 4096)
    B = sg.uniform_i8(g["seed"], 2, 4096, 4096)
    C = oracle.gemm_s8(A, B)
    assert np.abs(C).max() == g["maxabsC"]
    C32 = C.astype(np.int32)
    assert sg.checksum(C32) == _h(g["csC_i32"])
    assert C[0, 0] == g["C00"] and C[-1, -1] == g["Clast"]


def test_golden_C4_corners():
    g = C6["C4"]
    N = 16384
    A = sg.normal_bf16(g["seed"], 1, N, N)
    B = sg.normal_bf16(g["seed"], 2, N, N)
    C, D = oracle.gemm_bf16_rows(A, B, [0, N - 1])
    assert C[0, 0] == g["C00"] and abs(D[0, 0] - g["D00"]) < 0.05
    assert C[0, -1] == g["C0_last"] and C[1, 0] == g["Clast_0"] and C[1, -1] == g["Clast_last"]
