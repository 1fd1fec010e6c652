"""Seeded fuzz of the CUDA path against the CPU oracle: random shapes (biased toward tile
seams: multiples of 16/32/64/128/256 and one off), dtypes and schedule knobs (tail split
modes, tile widths, K atoms per stage, CTA pairs, cluster multicast, FP64 tile and split),
exact-integer inputs so every comparison is bit-exact in any summation order
(SURVEY 8(c) c4).  Each case also runs with a guard-banded output (no store outside C).
MM_F64_EMU is fuzzed the same way (its INT8 products under random knobs).
"""
import os
import random

import numpy as np
import pytest
import torch

import oracle
import synthgen as sg

pytestmark = pytest.mark.gpu

N_CASES = 160
KNOBS_TC = {
    "MM_STREAMK": [None, "0", "1", "2", "3", "4"],
    "MM_NT": [None, "1", "2"],
    "MM_KA": [None, "1"],
    "MM_FORCE_CG": [None, "1", "2"],
    "MM_MC": [None, None, "2"],
    "MM_L2_HINT": [None, None, None, "1", "3"],
    "MM_WAVE_SYNC": [None, None, None, "2"],
}
KNOBS_F64 = {
    "MM_F64_TILE": [None, "32", "64", "128"],
    "MM_F64_STREAMK": [None, "0", "1"],
    "MM_F64_W8": [None, None, None, "1"],
    "MM_F64_CK": [None, None, "1"],
    "MM_F64_KS": [None, None, None, "2", "4", "8", "44"],
    "MM_F64_KB": [None, None, "1"],
}


@pytest.fixture(scope="module")
def mm(cuda_device):
    import paper_2408_15384_b200 as mm_
    return mm_


def _dim(rng):
    r = rng.random()
    if r < 0.5:
        base = rng.choice([16, 32, 64, 128, 256, 512])
        return max(1, base * rng.randint(1, 6) + rng.choice([-1, 0, 0, 1]))
    if r < 0.8:
        return rng.randint(1, 1400)
    return rng.randint(1, 40)


def _cases():
    rng = random.Random(20261019)
    out = []
    for i in range(N_CASES):
        dt = rng.choice(["i8", "bf16", "f64"])
        m, n, p = _dim(rng), _dim(rng), _dim(rng)
        knobs = KNOBS_F64 if dt == "f64" else KNOBS_TC
        env = {k: rng.choice(v) for k, v in knobs.items()}
        out.append((i, dt, m, n, p, {k: v for k, v in env.items() if v is not None}))
    return out


def _gen(dt, seed, m, n, p):
    if dt == "f64":
        return sg.exact_f64(seed, 1, 2049, m, n), sg.exact_f64(seed, 2, 2049, n, p)
    if dt == "bf16":
        return sg.exact_bf16(seed, 1, 9, m, n), sg.exact_bf16(seed, 2, 9, n, p)
    return sg.exact_i8(seed, 1, 255, m, n), sg.exact_i8(seed, 2, 255, n, p)


def _ref(dt, A, B):
    if dt == "f64":
        return np.asarray(oracle.gemm_f64(A, B), np.float64)
    if dt == "bf16":
        return np.asarray(oracle.gemm_bf16(A, B)[0], np.float64)
    return np.asarray(oracle.gemm_s8(A, B), np.float64)


def _dev(x, dt):
    if dt == "bf16":
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c[0]}-{c[1]}-{c[2]}x{c[3]}x{c[4]}")
def test_fuzz_exact(mm, case):
    i, dt, m, n, p, env = case
    A, B = _gen(dt, 700 + i, m, n, p)
    Cref = _ref(dt, A, B)
    out = {"f64": torch.float64, "bf16": torch.float32, "i8": torch.int32}[dt]
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        guard = 4096
        buf = torch.full((guard + m * p + guard,), -7, dtype=out, device="cuda")
        C = buf[guard:guard + m * p].view(m, p)
        C.fill_(5)  # stale contents must be overwritten everywhere
        mm.gemm(_dev(A, dt), _dev(B, dt), out=C)
        mm.sync_check()
        h = buf.cpu().numpy()
        assert np.all(h[:guard] == -7) and np.all(h[guard + m * p:] == -7), ("store outside C", env)
        got = C.cpu().numpy().astype(np.float64)
        bad = int((got != Cref).sum())
        assert bad == 0, (f"{bad} mismatches", env)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _cases_random():
    rng = random.Random(20261020)
    out = []
    for i in range(24):
        dt = rng.choice(["bf16", "f64"])
        m, n, p = _dim(rng), _dim(rng), _dim(rng)
        knobs = KNOBS_F64 if dt == "f64" else KNOBS_TC
        env = {k: rng.choice(v) for k, v in knobs.items()}
        out.append((i, dt, m, n, p, {k: v for k, v in env.items() if v is not None}))
    return out


@pytest.mark.parametrize("case", _cases_random(), ids=lambda c: f"r{c[0]}-{c[1]}-{c[2]}x{c[3]}x{c[4]}")
def test_fuzz_random_values(mm, case):
    """Random-valued inputs (U[-1,1) FP64, N(0,1) BF16) under random knobs: normalised error
    within the contract (1e-12 FP64, 2e-2 BF16) and the BF16 diagnostic bound (1e-4)."""
    i, dt, m, n, p, env = case
    if dt == "f64":
        A, B = sg.uniform_f64(800 + i, 1, m, n), sg.uniform_f64(800 + i, 2, n, p)
        Cref, D = oracle.gemm_f64(A, B), oracle.absden_f64(A, B)
        tol = 1e-12
    else:
        A, B = sg.normal_bf16(800 + i, 1, m, n), sg.normal_bf16(800 + i, 2, n, p)
        Cref, D = oracle.gemm_bf16(A, B)
        tol = 1e-4
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        C = mm.gemm(_dev(A, dt), _dev(B, dt))
        mm.sync_check()
        err = oracle.normalized_error(C.cpu().numpy(), Cref, D)
        assert err <= tol, (err, env)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _cases_emu():
    rng = random.Random(20261021)
    out = []
    for i in range(32):
        m, n, p = _dim(rng), _dim(rng), _dim(rng)
        if i % 8 == 7:
            n = rng.randint(20000, 70000)  # long K: INT32 sums of residue products near their bound
            m, p = rng.randint(1, 64), rng.randint(1, 64)
        env = {k: rng.choice(v) for k, v in KNOBS_TC.items()}
        out.append((i, m, n, p, {k: v for k, v in env.items() if v is not None}))
    return out


@pytest.mark.parametrize("case", _cases_emu(), ids=lambda c: f"e{c[0]}-{c[1]}x{c[2]}x{c[3]}")
def test_fuzz_f64_emulation(mm, case):
    """MM_F64_EMU under random shapes and random schedule knobs of its INT8 products (their
    epilogue writes residue bytes; a forced reduce-add tail must fall back): exact-integer inputs
    bit-exact against the oracle with a guard-banded output, then U[-1,1) inputs with rows and
    columns scaled by random powers of two within the FP64 tolerance and DMMA's ~1e-16 class."""
    i, m, n, p, env = case
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        A, B = _gen("f64", 900 + i, m, n, p)
        Cref = _ref("f64", A, B)
        guard = 4096
        buf = torch.full((guard + m * p + guard,), -7.0, dtype=torch.float64, device="cuda")
        C = buf[guard:guard + m * p].view(m, p)
        C.fill_(5.0)
        mm.gemm(_dev(A, "f64"), _dev(B, "f64"), out=C, f64_emulation=True)
        mm.sync_check()
        h = buf.cpu().numpy()
        assert np.all(h[:guard] == -7) and np.all(h[guard + m * p:] == -7), ("store outside C", env)
        bad = int((C.cpu().numpy() != Cref).sum())
        assert bad == 0, (f"{bad} mismatches", env)
        rng = np.random.default_rng(900 + i)
        A = sg.uniform_f64(950 + i, 1, m, n) * np.ldexp(1.0, rng.integers(-60, 60, m))[:, None]
        B = sg.uniform_f64(950 + i, 2, n, p) * np.ldexp(1.0, rng.integers(-60, 60, p))[None, :]
        Cref, D = oracle.gemm_f64(A, B), oracle.absden_f64(A, B)
        C = mm.gemm(_dev(A, "f64"), _dev(B, "f64"), f64_emulation=True)
        mm.sync_check()
        err = oracle.normalized_error(C.cpu().numpy(), Cref, D)
        assert err <= 1e-12 and err <= 1e-15, (err, env)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
