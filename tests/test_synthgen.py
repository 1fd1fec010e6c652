"""Pins for the shared input generator (synthgen/): recipe goldens (SURVEY.md
§8 c6), ranges, determinism, the Box-Muller formulas (SPEC.md:
126-128) and the single-rounding bf16 conversion.  CPU only."""
import json
import math
import os
import struct

import numpy as np
import pytest

import synthgen as sg

with open(os.path.join(os.path.dirname(__file__), "golden", "survey_c6.json")) as f:
    C6 = json.load(f)


def test_sanity_words():
    assert sg.key(0, 1) == int(C6["sanity"]["key_seed0_roleA"], 16)
    assert sg.word(sg.key(0, 1), 0) == int(C6["sanity"]["w_seed0_roleA_idx0"], 16)


def _splitmix_py(seed_key, idx):
    M = (1 << 64) - 1

    def fmix(z):
        z ^= z >> 30
        z = (z * 0xBF58476D1CE4E5B9) & M
        z ^= z >> 27
        z = (z * 0x94D049BB133111EB) & M
        z ^= z >> 31
        return z
    return fmix((seed_key + (idx + 1) * 0x9E3779B97F4A7C15) & M)


def test_word_matches_python_reimplementation():
    k = sg.key(3, 2)
    for idx in (0, 1, 2, 1000, 2 ** 40 + 7):
        assert sg.word(k, idx) == _splitmix_py(k, idx)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_f64_golden(cfg):
    g = C6[cfg]
    A = sg.uniform_f64(g["seed"], 1, g["m"], g["n"])
    B = sg.uniform_f64(g["seed"], 2, g["n"], g["p"])
    assert sg.checksum(A) == int(g["csA"], 16)
    assert sg.checksum(B) == int(g["csB"], 16)
    if "A00_03" in g:
        assert A[0, :4].tolist() == g["A00_03"]
    else:
        assert A[0, 0] == g["A00"]


def test_i8_golden():
    g = C6["C3"]
    A = sg.uniform_i8(g["seed"], 1, 4096, 4096)
    B = sg.uniform_i8(g["seed"], 2, 4096, 4096)
    assert A[0, :4].tolist() == g["A00_03"]
    assert sg.checksum(A) == int(g["csA"], 16) and sg.checksum(B) == int(g["csB"], 16)
    assert A.min() >= -127 and A.max() <= 127  # -128 never generated (DESIGN R7)
    assert A.min() == -127 and A.max() == 127


def test_bf16_golden():
    g = C6["C4"]
    A = sg.normal_bf16(g["seed"], 1, 16384, 16384)
    assert sg.bf16_bits_to_f64(A[0, :4]).tolist() == g["A00_03"]
    assert sg.checksum(A) == int(g["csA"], 16)


def test_f64_range_and_grid():
    A = sg.uniform_f64(0, 1, 1000, 1000)
    assert A.min() >= -1.0 and A.max() < 1.0
    # grid 2^-52: (x + 1) * 2^52 is an integer
    assert np.all(np.floor((A + 1) * 2.0 ** 52) == (A + 1) * 2.0 ** 52)
    assert abs(A.mean()) < 5e-3 and abs(A.var() - 1 / 3) < 5e-3


def test_determinism_and_seed_sensitivity():
    assert np.array_equal(sg.uniform_f64(5, 1, 10, 10), sg.uniform_f64(5, 1, 10, 10))
    assert not np.array_equal(sg.uniform_f64(5, 1, 10, 10), sg.uniform_f64(6, 1, 10, 10))
    assert not np.array_equal(sg.uniform_f64(5, 1, 10, 10), sg.uniform_f64(5, 2, 10, 10))
    # counter-based: a sub-block equals the prefix of a bigger matrix with the same cols
    assert np.array_equal(sg.uniform_f64(5, 1, 3, 10), sg.uniform_f64(5, 1, 10, 10)[:3])


def test_box_muller_formulas():
    # SPEC.md:126-128 worked examples of PAPER.md:162-167
    z0, z1 = sg.box_muller(0.5, 0.25)
    assert abs(z0) < 1e-15 and abs(z1 - math.sqrt(2 * math.log(2))) < 1e-15
    assert abs(z1 - 1.1774) < 1e-4
    z0, z1 = sg.box_muller(0.3, 0.7)
    assert abs(z0 * z0 + z1 * z1 - (-2 * math.log(0.3))) < 1e-12
    z0, z1 = sg.box_muller(1 - 2 ** -53, 0.3)
    assert abs(z0) < 1e-7 and abs(z1) < 1e-7


def test_normals_moments():
    Z = sg.normal_f64(3, 1, 1000, 1000)
    assert abs(Z.mean()) < 5e-3 and abs(Z.var() - 1.0) < 1e-2
    assert np.all(np.isfinite(Z))


def _bf16_rne_reference(x: float) -> int:
    """Independent RNE double->bf16 via integer bit manipulation of the double."""
    b = struct.unpack("<Q", struct.pack("<d", x))[0]
    sign = b >> 63
    exp = (b >> 52) & 0x7FF
    mant = b & ((1 << 52) - 1)
    if exp == 0 and mant == 0:
        return sign << 15
    full = (1 << 52) | mant          # 53-bit significand
    keep = full >> 45                # 8 significant bits
    rem = full & ((1 << 45) - 1)
    half = 1 << 44
    if rem > half or (rem == half and (keep & 1)):
        keep += 1
    e = exp - 1023
    if keep == 1 << 8:
        keep >>= 1
        e += 1
    f32 = struct.unpack("<f", struct.pack("<I", (sign << 31) | ((e + 127) << 23) | ((keep & 0x7F) << 16)))[0]
    return struct.unpack("<I", struct.pack("<f", f32))[0] >> 16


def test_bf16_single_rounding():
    # ties to even: 1+2^-8 -> 1.0, 1+3*2^-8 -> 1.015625
    assert sg.bf16_from_double(1 + 2 ** -8) == 0x3F80
    assert sg.bf16_from_double(1 + 3 * 2 ** -8) == 0x3F82
    assert sg.bf16_from_double(-0.0) == 0x8000
    Z = sg.normal_f64(3, 1, 1, 20000).ravel()
    bits = sg.normal_bf16(3, 1, 1, 20000).ravel()
    for z, b in zip(Z[:5000], bits[:5000]):
        assert b == _bf16_rne_reference(float(z))
    # the rounded value is the nearest bf16 (error <= half an ulp of 8 significant bits)
    back = sg.bf16_bits_to_f64(bits)
    rel = np.abs(back - Z) / np.maximum(np.abs(Z), 1e-300)
    assert rel.max() <= 2.0 ** -8


def test_exact_int_ranges():
    for K in (3, 9, 2049):
        X = sg.exact_f64(4, 1, K, 200, 200)
        h = (K - 1) // 2
        assert X.min() == -h and X.max() == h and np.all(X == np.round(X))
    Xb = sg.bf16_bits_to_f64(sg.exact_bf16(4, 1, 9, 100, 100))
    assert set(np.unique(Xb).tolist()) == set(range(-4, 5))
    Xi = sg.exact_i8(4, 1, 3, 100, 100)
    assert set(np.unique(Xi).tolist()) == {-1, 0, 1}


def test_checksum_properties():
    x = np.arange(10, dtype=np.float64)
    y = x.copy()
    y[[2, 3]] = y[[3, 2]]
    assert sg.checksum(x) != sg.checksum(y)  # position-sensitive
    z = np.zeros(5)
    assert sg.checksum(z) == sg.checksum(-z)  # -0 canonicalised
    assert sg.checksum(np.zeros(5, np.float32)) == sg.checksum(-np.zeros(5, np.float32))
