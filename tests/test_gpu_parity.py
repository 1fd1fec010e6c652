"""GPU parity: the CUDA path (through the C-ABI, via the ctypes binding) against
the CPU oracle, element by element, on seeded inputs (synthgen/).

Bars (BASELINE.json north_star):
  INT8 -> INT32 : bit-exact.
  exact-integer FP inputs (any dtype): bit-exact (every partial sum is an
                  exactly representable integer, so any summation order is exact).
  FP64 random   : max_ij |C - C_ref| / D_ij <= 1e-12,  D_ij = Σ_k |A_ik B_kj|.
  BF16 random   : <= 2e-2 (contract) and <= 1e-4 (diagnostic; FP32 accumulation
                  error is ~1e-7).
Full config sizes (BASELINE.json configs 0-4) run in the launch configuration
bench.py times; where the oracle is too slow for the full product, seeded rows
and columns (plus shard/tile seams) are checked one by one, and the exact-integer
pins compare the full-output checksum with tests/golden/oracle_fullsize.json
(written by tools/make_golden.py from the oracle only).
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synthgen as sg

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TOL = {"f64": 1e-12, "bf16": 2e-2}
DIAG_BF16 = 1e-4


@pytest.fixture(scope="module")
def mm(cuda_device):
    import paper_2408_15384_b200 as mm_
    return mm_


@pytest.fixture(autouse=True)
def _clear_cg_env():
    os.environ.pop("MM_FORCE_CG", None)
    yield
    os.environ.pop("MM_FORCE_CG", None)


def to_dev(x: np.ndarray, dt: str) -> torch.Tensor:
    if dt == "bf16":
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def run_gpu(mm, A, B, dt, cg=None) -> np.ndarray:
    if cg:
        os.environ["MM_FORCE_CG"] = str(cg)
    C = mm.gemm(to_dev(A, dt), to_dev(B, dt))
    mm.sync_check()
    return C.cpu().numpy()


def gen(dt, kind, seed, m, n, p, K=None):
    if kind == "exact":
        if dt == "f64":
            return sg.exact_f64(seed, 1, K, m, n), sg.exact_f64(seed, 2, K, n, p)
        if dt == "bf16":
            return sg.exact_bf16(seed, 1, K, m, n), sg.exact_bf16(seed, 2, K, n, p)
        return sg.exact_i8(seed, 1, K, m, n), sg.exact_i8(seed, 2, K, n, p)
    if dt == "f64":
        return sg.uniform_f64(seed, 1, m, n), sg.uniform_f64(seed, 2, n, p)
    if dt == "bf16":
        return sg.normal_bf16(seed, 1, m, n), sg.normal_bf16(seed, 2, n, p)
    return sg.uniform_i8(seed, 1, m, n), sg.uniform_i8(seed, 2, n, p)


def ref(dt, A, B):
    """(C_ref, D) from the oracle."""
    if dt == "f64":
        return oracle.gemm_f64(A, B), oracle.absden_f64(A, B)
    if dt == "bf16":
        return oracle.gemm_bf16(A, B)
    C = oracle.gemm_s8(A, B)
    return C, None


def check(dt, C, Cref, D, exact):
    if dt == "i8" or exact:
        assert np.array_equal(np.asarray(C, np.float64), np.asarray(Cref, np.float64)), \
            f"mismatches: {(np.asarray(C, np.float64) != Cref).sum()}"
        return 0.0
    err = oracle.normalized_error(C, Cref, D)
    assert err <= TOL[dt], err
    if dt == "bf16":
        assert err <= DIAG_BF16, f"diagnostic bf16 bound exceeded: {err}"
    return err


# ------------------------------------------------------------------ fixtures (hand-worked)
with open(os.path.join(GOLDEN, "handworked.json")) as f:
    HAND = json.load(f)["cases"]


@pytest.mark.parametrize("case", HAND, ids=[c["name"] for c in HAND])
def test_handworked(mm, case):
    A = np.asarray(case["A"], np.float64)
    B = np.asarray(case["B"], np.float64)
    for dt in case["dtypes"]:
        dtk = {"s8": "i8"}.get(dt, dt)
        if dtk == "f64":
            Ag, Bg = A, B
        elif dtk == "bf16":
            Ag = np.vectorize(sg.bf16_from_double, otypes=[np.uint16])(A)
            Bg = np.vectorize(sg.bf16_from_double, otypes=[np.uint16])(B)
        else:
            Ag, Bg = A.astype(np.int8), B.astype(np.int8)
        for cg in ((1, 2) if dtk != "f64" else (None,)):
            C = run_gpu(mm, Ag, Bg, dtk, cg)
            assert np.array_equal(np.asarray(C, np.float64), np.asarray(case["C"], np.float64)), (dtk, cg, C)


# ------------------------------------------------------------------ brute force, tiny shapes
@pytest.mark.parametrize("dt", ["i8", "bf16", "f64"])
def test_all_tiny_shapes_exact(mm, dt):
    """Every (m,n,p) in {1..8}^3: exact-integer inputs, bit-exact."""
    K = {"i8": 255, "bf16": 9, "f64": 2049}[dt]
    for m in range(1, 9):
        for n in range(1, 9):
            for p in range(1, 9):
                seed = 1000 + m * 100 + n * 10 + p
                A, B = gen(dt, "exact", seed, m, n, p, K)
                Cref, D = ref(dt, A, B)
                C = run_gpu(mm, A, B, dt)
                check(dt, C, Cref, D, exact=True)


SEAMS = [1, 15, 16, 17, 63, 64, 65, 127, 128, 129, 255, 256, 257]


def _seam_shapes(count, seed):
    rng = np.random.default_rng(seed)
    return [tuple(int(x) for x in rng.choice(SEAMS, 3)) for _ in range(count)]


@pytest.mark.parametrize("dt", ["i8", "bf16"])
@pytest.mark.parametrize("cg", [1, 2])
def test_tile_seams_tc(mm, dt, cg):
    for (m, n, p) in _seam_shapes(24, 7 + cg) + [(257, 257, 257), (129, 63, 513), (384, 320, 272)]:
        A, B = gen(dt, "exact", 77, m, n, p, 255 if dt == "i8" else 9)
        Cref, D = ref(dt, A, B)
        C = run_gpu(mm, A, B, dt, cg)
        check(dt, C, Cref, D, exact=True)


def test_tile_seams_f64(mm):
    for (m, n, p) in _seam_shapes(24, 3) + [(257, 257, 257), (129, 17, 131), (384, 320, 272)]:
        A, B = gen("f64", "exact", 78, m, n, p, 2049)
        Cref, D = ref("f64", A, B)
        check("f64", run_gpu(mm, A, B, "f64"), Cref, D, exact=True)


@pytest.mark.parametrize("dt", ["i8", "bf16", "f64"])
@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("streamk", ["default", "1", "2", "3"])
def test_stream_k_split_tiles(mm, dt, cg, streamk):
    """Few tiles, long K: tiles split over several CTAs/clusters (stream-K partials +
    finisher) — default policy, the general split (1), the exact-halves split with
    landing in the operand ring (2) and the exact halves added into C by TMA reduce-add (3)
    — and a ragged split tail after full waves."""
    if dt == "f64" and (cg == 2 or streamk != "default"):
        pytest.skip("FP64: no CTA pair; its stream-K is always on")
    if streamk != "default":
        os.environ["MM_STREAMK"] = streamk
    try:
        for (m, n, p) in [(512, 4096, 512), (130, 3000, 260), (2048, 2048, 2304), (1300, 1024, 2600),
                          (2304, 1024, 2048), (2560, 768, 2560)]:
            A, B = gen(dt, "exact", 41, m, n, p, {"i8": 255, "bf16": 9, "f64": 2049}[dt])
            Cref, D = ref(dt, A, B)
            check(dt, run_gpu(mm, A, B, dt, cg if dt != "f64" else None), Cref, D, exact=True)
            A, B = gen(dt, "random", 42, m, n, p)
            Cref, D = ref(dt, A, B)
            check(dt, run_gpu(mm, A, B, dt, cg if dt != "f64" else None), Cref, D, exact=False)
    finally:
        os.environ.pop("MM_STREAMK", None)


@pytest.mark.parametrize("dt", ["i8", "bf16"])
@pytest.mark.parametrize("streamk", ["0", "1", "3"])
def test_wide_tiles_nt2(mm, dt, streamk):
    """512-wide CTA-pair tiles (two TMEM accumulators), forced on small/ragged shapes,
    with and without the stream-K split tail."""
    os.environ["MM_NT"] = "2"
    os.environ["MM_STREAMK"] = streamk
    try:
        for (m, n, p) in [(300, 200, 520), (512, 4096, 1024), (1100, 768, 1700), (256, 64, 2048), (2048, 1024, 4608)]:
            A, B = gen(dt, "exact", 43, m, n, p, 255 if dt == "i8" else 9)
            Cref, D = ref(dt, A, B)
            check(dt, run_gpu(mm, A, B, dt, 2), Cref, D, exact=True)
    finally:
        os.environ.pop("MM_NT", None)
        os.environ.pop("MM_STREAMK", None)


@pytest.mark.parametrize("dt,mode", [("f64", "1"), ("bf16", "1"), ("i8", "1"), ("bf16", "3"), ("i8", "3")])
def test_split_tile_fixup_repeated(mm, dt, mode):
    """Race check of the split-tile fix-up (contributors publish partials, the finisher waits on
    a counter and adds them; mode 3: one half zeroes C and publishes, both reduce-add into C):
    many back-to-back launches of split-heavy shapes, every output compared bit-exactly
    (exact-integer inputs).  A premature release of the finisher's named barrier (bar.sync by a
    divergent warp) showed up here as a few wrong rows in one tile."""
    env = {"f64": {"MM_F64_TILE": "128", "MM_F64_STREAMK": "1"}, "bf16": {"MM_STREAMK": mode},
           "i8": {"MM_STREAMK": mode}}[dt]
    os.environ.update(env)
    try:
        for (m, n, p) in [(1100, 768, 1700), (513, 2048, 700), (2560, 768, 2560)]:
            A, B = gen(dt, "exact", 49, m, n, p, {"i8": 255, "bf16": 9, "f64": 2049}[dt])
            Cref, _ = ref(dt, A, B)
            Ad, Bd = to_dev(A, dt), to_dev(B, dt)
            outs = [mm.gemm(Ad, Bd) for _ in range(12)]
            mm.sync_check()
            for C in outs:
                assert np.array_equal(C.cpu().numpy().astype(np.float64), np.asarray(Cref, np.float64)), (m, n, p)
    finally:
        for k in env:
            os.environ.pop(k, None)


@pytest.mark.parametrize("dt", ["bf16", "i8"])
def test_reduce_add_tail(mm, dt):
    """Tail tiles split in exact K halves, both added into C by TMA reduce-add (the half holding
    k-block 0 zeroes C first): C3-like 256-tile shapes whose last wave has <= 37 tiles.  Random
    inputs: within tolerance of the oracle and bit-identical over repeated launches (two addends
    into +0 commute exactly); a guard-banded C (no store outside it); int8 wrap-around sums."""
    os.environ["MM_STREAMK"] = "3"
    try:
        for (m, n, p) in [(4096, 512, 4096), (2560, 768, 2560), (2400, 1000, 2700)]:
            A, B = gen(dt, "random", 51, m, n, p)
            Cref, D = ref(dt, A, B)
            Ad, Bd = to_dev(A, dt), to_dev(B, dt)
            outs = [mm.gemm(Ad, Bd) for _ in range(8)]
            mm.sync_check()
            check(dt, outs[0].cpu().numpy(), Cref, D, exact=False)
            for C in outs[1:]:
                assert torch.equal(C, outs[0]), (m, n, p)
        out = torch.float32 if dt == "bf16" else torch.int32
        m, n, p = 2560, 768, 2560
        A, B = gen(dt, "exact", 52, m, n, p, 255 if dt == "i8" else 9)
        Cref, _ = ref(dt, A, B)
        guard = 8192
        buf = torch.full((guard + m * p + guard,), -7, dtype=out, device="cuda")
        C = buf[guard:guard + m * p].view(m, p)
        C.fill_(123)  # stale contents: the zeroing half must overwrite them
        mm.gemm(to_dev(A, dt), to_dev(B, dt), out=C)
        mm.sync_check()
        h = buf.cpu().numpy()
        assert np.all(h[:guard] == -7) and np.all(h[guard + m * p:] == -7)
        assert np.array_equal(C.cpu().numpy().astype(np.float64), np.asarray(Cref, np.float64))
    finally:
        os.environ.pop("MM_STREAMK", None)


@pytest.mark.parametrize("dt", ["bf16", "i8"])
def test_reduce_add_tail_same_output_back_to_back(mm, dt):
    """The reduce-add tail zeroes C before its MMAs finish; with programmatic dependent launch the
    next product in the stream starts while the previous one still stores.  Back-to-back products
    into the SAME output, alternating inputs, on shapes whose split tile is a CTA's first item
    (no full wave): each result must be exactly its own product."""
    os.environ["MM_STREAMK"] = "3"
    try:
        for (m, n, p) in [(1024, 2048, 1024), (512, 4096, 768)]:
            out = torch.float32 if dt == "bf16" else torch.int32
            pairs = [gen(dt, "exact", 60 + s, m, n, p, 255 if dt == "i8" else 9) for s in range(2)]
            refs = [np.asarray(ref(dt, A, B)[0], np.float64) for A, B in pairs]
            dev = [(to_dev(A, dt), to_dev(B, dt)) for A, B in pairs]
            C = torch.empty(m, p, dtype=out, device="cuda")
            snaps = []
            for it in range(16):
                Ad, Bd = dev[it % 2]
                mm.gemm(Ad, Bd, out=C)
                if it >= 14:
                    snaps.append(C.clone())
            mm.sync_check()
            for it, S in zip((14, 15), snaps):
                assert np.array_equal(S.cpu().numpy().astype(np.float64), refs[it % 2]), (m, n, p, it)
    finally:
        os.environ.pop("MM_STREAMK", None)


@pytest.mark.parametrize("tile", ["32ks4", "32ks2", "32ks1", "64", "96", "128"])
@pytest.mark.parametrize("streamk", ["0", "1"])
def test_f64_tiles_and_schedules(mm, tile, streamk):
    """FP64 kernel at every CTA tile (32x32 with 4 k-block groups of one warp, 2 of 4 warps, or one
    group of 4; 64x64 /
    96x128 and 128x128 with 16 warps), with whole-tile waves only or with the split last wave, on ragged
    and multi-wave shapes; the exact-integer inputs make every tile, seam, k-group and
    partial-tile sum bit-exact."""
    os.environ["MM_F64_TILE"] = tile[:2] if tile.startswith("32") else tile
    os.environ["MM_F64_KS"] = tile[4:] if tile.startswith("32") else "1"
    os.environ["MM_F64_STREAMK"] = streamk
    try:
        for (m, n, p) in [(256, 256, 256), (300, 200, 520), (129, 1000, 77), (1100, 768, 1700), (2100, 300, 2050),
                          (300, 208, 528), (100, 1024, 160), (33, 16, 48), (250, 80, 240)]:
            # (16-multiple n and p: the 32x32 whole-tile path loads 4 k-blocks per 3-D TMA box,
            # incl. a partial last group when n/16 is not a multiple of 4)
            A, B = gen("f64", "exact", 47, m, n, p, 2049)
            Cref, D = ref("f64", A, B)
            check("f64", run_gpu(mm, A, B, "f64"), Cref, D, exact=True)
        A, B = gen("f64", "random", 48, 1100, 768, 1700)
        Cref, D = ref("f64", A, B)
        check("f64", run_gpu(mm, A, B, "f64"), Cref, D, exact=False)
    finally:
        os.environ.pop("MM_F64_TILE", None)
        os.environ.pop("MM_F64_KS", None)
        os.environ.pop("MM_F64_STREAMK", None)


@pytest.mark.parametrize("dt", ["i8", "bf16"])
@pytest.mark.parametrize("nt,ka", [("1", None), ("1", "1"), ("2", None)])
def test_cluster_multicast_mc2(mm, dt, nt, ka):
    """Clusters of two CTA pairs (512-row tiles) sharing every B slab by TMA multicast, each
    pair loading half of its K rows: ragged m (partial second pair), ragged n and p, and a
    guard-banded C (no store outside C).  256-wide tiles with one or (default for n >= 8 atoms)
    two K atoms per stage."""
    os.environ["MM_MC"] = "2"
    os.environ["MM_NT"] = nt
    if ka:
        os.environ["MM_KA"] = ka
    try:
        for (m, n, p) in [(300, 200, 520), (513, 1024, 1100), (1100, 768, 1700), (2048, 2048, 2048), (777, 64, 300)]:
            A, B = gen(dt, "exact", 44, m, n, p, 255 if dt == "i8" else 9)
            Cref, D = ref(dt, A, B)
            check(dt, run_gpu(mm, A, B, dt, 2), Cref, D, exact=True)
        A, B = gen(dt, "random", 45, 1100, 768, 1700)
        Cref, D = ref(dt, A, B)
        check(dt, run_gpu(mm, A, B, dt, 2), Cref, D, exact=False)
        out = torch.float32 if dt == "bf16" else torch.int32
        m, n, p = 900, 512, 700
        A, B = gen(dt, "exact", 46, m, n, p, 255 if dt == "i8" else 9)
        Cref, _ = ref(dt, A, B)
        guard = 4096
        buf = torch.full((guard + m * p + guard,), -7, dtype=out, device="cuda")
        C = buf[guard:guard + m * p].view(m, p)
        mm.gemm(to_dev(A, dt), to_dev(B, dt), out=C)
        mm.sync_check()
        h = buf.cpu().numpy()
        assert np.all(h[:guard] == -7) and np.all(h[guard + m * p:] == -7)
        assert np.array_equal(C.cpu().numpy().astype(np.float64), np.asarray(Cref, np.float64))
    finally:
        os.environ.pop("MM_MC", None)
        os.environ.pop("MM_NT", None)
        os.environ.pop("MM_KA", None)


@pytest.mark.parametrize("dt", ["i8", "bf16", "f64"])
def test_random_values_ragged(mm, dt):
    for cg in ((1, 2) if dt != "f64" else (None,)):
        for (m, n, p) in [(300, 200, 520), (129, 1000, 77), (1024, 768, 1280), (5, 4096, 9)]:
            A, B = gen(dt, "random", 11, m, n, p)
            Cref, D = ref(dt, A, B)
            check(dt, run_gpu(mm, A, B, dt, cg), Cref, D, exact=False)


# ------------------------------------------------------------------ special cases
@pytest.mark.parametrize("dt", ["i8", "bf16", "f64"])
def test_identity_zero_transpose(mm, dt):
    m, n, p = 200, 136, 264
    A, B = gen(dt, "random", 5, m, n, p)
    if dt == "bf16":
        one = sg.bf16_from_double(1.0)
        I = np.zeros((n, n), np.uint16)
        np.fill_diagonal(I, one)
        Z = np.zeros((n, p), np.uint16)
        Af = sg.bf16_bits_to_f64(A)
    elif dt == "i8":
        I = np.eye(n, dtype=np.int8)
        Z = np.zeros((n, p), np.int8)
        Af = A.astype(np.float64)
    else:
        I = np.eye(n)
        Z = np.zeros((n, p))
        Af = A
    assert np.array_equal(np.asarray(run_gpu(mm, A, I, dt), np.float64), Af)  # A·I = A
    assert not np.asarray(run_gpu(mm, A, Z, dt), np.float64).any()             # A·0 = 0
    # (AB)^T = B^T A^T through the library: exact for int8 and exact-int FP
    Ae, Be = gen(dt, "exact", 6, m, n, p, 255 if dt == "i8" else 9)
    C1 = run_gpu(mm, Ae, Be, dt)
    C2 = run_gpu(mm, np.ascontiguousarray(Be.T), np.ascontiguousarray(Ae.T), dt)
    assert np.array_equal(C1.T, C2)


@pytest.mark.parametrize("dt", ["i8", "bf16", "f64"])
def test_misaligned_operands_use_pack_path(mm, dt):
    """Base pointers off 16-B alignment and odd pitches: padded copy path."""
    m, n, p = 97, 61, 83  # odd pitches
    A, B = gen(dt, "exact", 9, m, n, p, 255 if dt == "i8" else 9)
    Cref, D = ref(dt, A, B)
    check(dt, run_gpu(mm, A, B, dt), Cref, D, exact=True)
    # aligned pitch but misaligned base: view into a larger buffer at offset 1 element
    m, n, p = 64, 64, 64
    A, B = gen(dt, "exact", 10, m, n, p, 255 if dt == "i8" else 9)
    Cref, D = ref(dt, A, B)
    Ad = to_dev(np.concatenate([A.ravel()[:1], A.ravel()]), dt)[1:].view(m, n)
    Bd = to_dev(np.concatenate([B.ravel()[:1], B.ravel()]), dt)[1:].view(n, p)
    assert Ad.data_ptr() % 16 != 0
    C = mm.gemm(Ad, Bd)
    mm.sync_check()
    check(dt, C.cpu().numpy(), Cref, D, exact=True)


@pytest.mark.parametrize("dt", ["i8", "bf16", "f64"])
def test_no_writes_outside_c(mm, dt):
    """Bounds check of every store path (compute-sanitizer is closed on this pool): C lives
    inside a larger buffer filled with a sentinel; the product must leave the guard bands,
    and the row tails beyond p inside a wider pitch, untouched."""
    out = {"f64": torch.float64, "bf16": torch.float32, "i8": torch.int32}[dt]
    sentinel = -7
    for (m, n, p, cg, nt) in [(300, 200, 520, 1, 1), (300, 200, 520, 2, 1), (513, 1024, 1100, 2, 2),
                              (129, 64, 33, None, None), (1000, 2000, 260, None, None)]:
        if dt == "f64" and cg == 2:
            continue
        A, B = gen(dt, "exact", 51, m, n, p, 255 if dt == "i8" else 9)
        Cref, _ = ref(dt, A, B)
        guard = 4096
        buf = torch.full((guard + m * p + guard,), sentinel, dtype=out, device="cuda")
        C = buf[guard:guard + m * p].view(m, p)
        if cg:
            os.environ["MM_FORCE_CG"] = str(cg)
        if nt:
            os.environ["MM_NT"] = str(nt)
        try:
            mm.gemm(to_dev(A, dt), to_dev(B, dt), out=C)
            mm.sync_check()
        finally:
            os.environ.pop("MM_FORCE_CG", None)
            os.environ.pop("MM_NT", None)
        h = buf.cpu().numpy()
        assert np.all(h[:guard] == sentinel) and np.all(h[guard + m * p:] == sentinel), (m, n, p, cg, nt)
        assert np.array_equal(C.cpu().numpy().astype(np.float64), np.asarray(Cref, np.float64))


@pytest.mark.parametrize("G", [2, 4, 8])
def test_row_blocks_bit_identical_to_full_product(mm, G):
    """G-invariance (SURVEY 8(b) determinism): the row blocks mm_shard_range gives
    G ranks, each multiplied on its own, reproduce the single-product C bit for bit — also for
    random BF16 inputs, whose FP32 sums would differ under any change of summation order —
    because no K-split is used at these shapes (tile choices differ between the full problem
    and the blocks: 512- vs 256-wide tiles, one vs several waves)."""
    m, n, p = 4100, 1024, 4096  # ragged last block
    A, B = gen("bf16", "random", 60 + G, m, n, p)
    Ad, Bd = to_dev(A, "bf16"), to_dev(B, "bf16")
    os.environ["MM_STREAMK"] = "0"  # the contract holds without K-split (a 1025-row block would split)
    try:
        full = mm.gemm(Ad, Bd)
        mm.sync_check()
        for r in range(G):
            r0, rows = mm.shard_range(m, G, r)
            if rows == 0:
                continue
            blk = mm.gemm(Ad[r0:r0 + rows].contiguous(), Bd)
            mm.sync_check()
            assert torch.equal(blk, full[r0:r0 + rows]), (G, r)
    finally:
        os.environ.pop("MM_STREAMK", None)


@pytest.mark.parametrize("dt", ["i8", "bf16"])
def test_epilogue_guard_bands_both_tile_widths(mm, dt):
    """The eight-warp epilogue (two warps per TMEM lane quarter, one per column half / NT=2
    region) with TMA stores, on ragged shapes with both tile widths, inside guard bands
    (bit-exact, nothing written outside C)."""
    out = torch.float32 if dt == "bf16" else torch.int32
    try:
        for (m, n, p, nt) in [(300, 200, 520, "1"), (513, 1024, 1100, "2"), (1100, 768, 1700, "2"), (777, 64, 300, "1")]:
            os.environ["MM_NT"] = nt
            A, B = gen(dt, "exact", 52, m, n, p, 255 if dt == "i8" else 9)
            Cref, _ = ref(dt, A, B)
            guard = 4096
            buf = torch.full((guard + m * p + guard,), -7, dtype=out, device="cuda")
            C = buf[guard:guard + m * p].view(m, p)
            mm.gemm(to_dev(A, dt), to_dev(B, dt), out=C)
            mm.sync_check()
            h = buf.cpu().numpy()
            assert np.all(h[:guard] == -7) and np.all(h[guard + m * p:] == -7), (m, n, p, nt)
            assert np.array_equal(C.cpu().numpy().astype(np.float64), np.asarray(Cref, np.float64)), (m, n, p, nt)
    finally:
        os.environ.pop("MM_NT", None)


def test_determinism(mm):
    for dt in ("bf16", "f64", "i8"):
        A, B = gen(dt, "random", 12, 700, 900, 650)
        C1 = run_gpu(mm, A, B, dt)
        C2 = run_gpu(mm, A, B, dt)
        assert np.array_equal(C1, C2)


def test_usage_errors(mm):
    A = torch.zeros(4, 4, dtype=torch.float64, device="cuda")
    lib = mm._lib.load()
    ctx = mm.context(0)
    assert lib.mm_gemm(ctx.handle, 0, 4, 4, 0, A.data_ptr(), A.data_ptr(), A.data_ptr(), None) == mm._lib.MM_ERR_USAGE
    assert b"dimensions" in lib.mm_last_error(ctx.handle)
    assert lib.mm_gemm(ctx.handle, 4, 4, 4, 7, A.data_ptr(), A.data_ptr(), A.data_ptr(), None) == mm._lib.MM_ERR_USAGE
    assert lib.mm_gemm(ctx.handle, 4, 4, 4, 0, None, A.data_ptr(), A.data_ptr(), None) == mm._lib.MM_ERR_USAGE
    # C overlapping A
    assert lib.mm_gemm(ctx.handle, 4, 4, 4, 0, A.data_ptr(), A.data_ptr(), A.data_ptr(), None) == mm._lib.MM_ERR_USAGE
    assert b"overlaps" in lib.mm_last_error(ctx.handle)
    with pytest.raises(ValueError):
        mm.gemm(torch.zeros(3, 4, device="cuda", dtype=torch.float64), torch.zeros(5, 4, device="cuda", dtype=torch.float64))
    with pytest.raises(TypeError):
        mm.gemm(torch.zeros(3, 4, device="cuda"), torch.zeros(4, 4, device="cuda"))


def test_int32_accumulate_large_k(mm):
    """INT32 accumulation exact up to n·128² < 2^31: worst-case signs at n = 65536."""
    m, n, p = 128, 65536, 256
    A = np.full((m, n), -127, np.int8)
    B = np.full((n, p), -127, np.int8)
    A[1] = 127
    C = run_gpu(mm, A, B, "i8")
    assert np.all(C[0] == n * 127 * 127) and np.all(C[1] == -n * 127 * 127)


@pytest.mark.parametrize("cg", [1, 2])
def test_int32_overflow_wraps(mm, cg):
    """Beyond BASELINE.json's range (R10): with n*128^2 > 2^31 - 1
    the INT32 accumulators wrap modulo 2^32 (measured on the B200: all -128 inputs, n = 131088,
    exact 2,147,745,792 -> -2,147,221,504), i.e. C equals the oracle's exact int64 sum reduced
    to int32 two's complement."""
    m, n, p = 256, 131088, 256
    os.environ["MM_FORCE_CG"] = str(cg)
    A = torch.full((m, n), -128, dtype=torch.int8, device="cuda")
    B = torch.full((n, p), -128, dtype=torch.int8, device="cuda")
    C = mm.gemm(A, B)
    mm.sync_check()
    exact = oracle.gemm_s8(np.full((1, n), -128, np.int8), np.full((n, 1), -128, np.int8))[0, 0]
    assert exact == n * 128 * 128
    wrapped = ((int(exact) + 2**31) % 2**32) - 2**31
    assert torch.all(C == wrapped), np.unique(C.cpu().numpy())


def test_bf16_subnormals_not_flushed(mm):
    """the configs never produce subnormals, so the hardware's handling is
    measured here: subnormal bf16 inputs (exponent 0) times 1.0, and normal inputs whose product
    (2^-70 * 2^-70 = 2^-140) and sums are FP32 subnormals — the tcgen05 BF16 path keeps both
    exactly (no flush to zero), equal to the oracle's exact double result."""
    n = 128
    sub = (np.arange(1, n + 1, dtype=np.uint16) & 0x7F)
    sub[sub == 0] = 1
    A = np.zeros((256, n), np.uint16)
    A[0] = sub
    A[0, :2] = 0  # keep row 0 away from the columns 200-201 products (below FP32's range)
    A[1, 0], A[1, 1] = 0x1C80, 0x1C80  # 2^-70
    B = np.zeros((n, 256), np.uint16)
    B[np.arange(n), np.arange(n)] = 0x3F80  # 1.0 on the diagonal
    B[0, 200], B[1, 200] = 0x1C80, 0x9C80  # +2^-70, -2^-70 -> row 1 col 200: 2^-140 - 2^-140 = 0
    B[0, 201] = 0x1C80                      # row 1 col 201: 2^-140
    Cref, _ = oracle.gemm_bf16(A, B)
    C = run_gpu(mm, A, B, "bf16")
    assert np.array_equal(C.astype(np.float64), Cref)
    assert C[1, 201] == np.float32(2.0 ** -140) and C[0, 5] != 0


def test_host_operand_path(mm):
    """mm_gemm_host (H2D, product, D2H in overlapped row blocks) equals the oracle."""
    for dt in ("f64", "bf16", "i8"):
        m, n, p = 1100, 520, 784
        A, B = gen(dt, "exact", 13, m, n, p, 255 if dt == "i8" else 9)
        Cref, D = ref(dt, A, B)
        if dt == "bf16":
            At = torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).pin_memory()
            Bt = torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).pin_memory()
        else:
            At, Bt = torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory()
        C = mm.gemm_host(At, Bt)
        check(dt, C.numpy(), Cref, D, exact=True)


def test_host_operand_path_f64_emulated(mm):
    """mm_gemm_host with MM_F64_EMU at a size the host path splits into 4 x 4 blocks (operands above
    64 MB): every block is its own emulated product (ragged last blocks); exact-integer inputs
    bit-exact against the oracle."""
    m, n, p = 2600, 1900, 2300
    A, B = gen("f64", "exact", 14, m, n, p, 2049)
    C = mm.gemm_host(torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory(), f64_emulation=True)
    assert np.array_equal(C.numpy(), oracle.gemm_f64(A, B))


# ------------------------------------------------------------------ BASELINE.json configs, full size
with open(os.path.join(GOLDEN, "oracle_fullsize.json")) as f:
    FULL = json.load(f)


def _gpu_checksum(C: torch.Tensor, kind: str) -> int:
    return sg.checksum(C.cpu().numpy(), kind)


def test_config0_fp64_256(mm):
    A, B = gen("f64", "random", 0, 256, 256, 256)
    Cref, D = ref("f64", A, B)
    check("f64", run_gpu(mm, A, B, "f64"), Cref, D, exact=False)
    A, B = gen("f64", "exact", 0, 256, 256, 256, 2049)
    C = run_gpu(mm, A, B, "f64")
    assert sg.checksum(C) == int(FULL["C1x"]["checksum"], 16)


def test_config1_fp64_ragged(mm):
    m, n, p = 2000, 1500, 1750
    A, B = gen("f64", "random", 1, m, n, p)
    Cref, D = ref("f64", A, B)
    check("f64", run_gpu(mm, A, B, "f64"), Cref, D, exact=False)
    A, B = gen("f64", "exact", 1, m, n, p, 2049)
    assert sg.checksum(run_gpu(mm, A, B, "f64")) == int(FULL["C2x"]["checksum"], 16)


@pytest.mark.parametrize("cg", [1, 2])
def test_config2_int8_4096(mm, cg):
    A, B = gen("i8", "random", 2, 4096, 4096, 4096)
    C = run_gpu(mm, A, B, "i8", cg)
    assert C.dtype == np.int32
    assert sg.checksum(C) == int(FULL["C3"]["checksum"], 16)
    Cref = oracle.gemm_s8(A, B)
    assert np.array_equal(C.astype(np.int64), Cref)


def _sample(n_total, count, role, seed, seams):
    idx = set(sg.sample_indices(seed, role, count, n_total).tolist())
    idx |= {i for i in seams if 0 <= i < n_total}
    return np.array(sorted(idx), np.int64)


def test_config3_bf16_16384(mm):
    N = 16384
    A, B = gen("bf16", "random", 3, N, N, N)
    C = run_gpu(mm, A, B, "bf16")
    seams = [0, N - 1] + [s + d for s in range(0, N, 2048) for d in (-1, 0)] + [255, 256, 257, 8191, 8192]
    rows = _sample(N, 48, 3, 3, seams)
    cols = _sample(N, 48, 4, 3, seams)
    Cr, Dr = oracle.gemm_bf16_rows(A, B, rows)
    Cc, Dc = oracle.gemm_bf16_cols(A, B, cols)
    e1 = check("bf16", C[rows], Cr, Dr, exact=False)
    e2 = check("bf16", C[:, cols], Cc, Dc, exact=False)
    print(f"C4 bf16 sampled max normalized error: rows {e1:.3e} cols {e2:.3e}")


def test_config3_row_blocks_bit_identical(mm):
    """C4 at full size on the config's own Box-Muller bf16 inputs (on-GPU generator,
    bit-identical to synthgen): the row blocks of the 2-, 4- and 8-GPU row-block sharding
    (mm_shard_range), each multiplied on its own as a rank would.  Without K-split
    (MM_STREAMK=0) every block equals the single-GPU product bit for bit ("ROW_BLOCK
    result is bit-identical to G=1 when no K-split is used"; the full C4 product has a 50-tile
    last wave, too many to split).  In the default configuration bench.py times, the G=8 block
    (3.46 waves of 512-wide tiles) splits its 34 tail tiles in K halves added by TMA reduce-add:
    those blocks are run-to-run identical and within the BF16 tolerance of the full product."""
    from synthgen import gpu as sgg
    N = 16384
    A = sgg.normal_bf16(3, sg.ROLE_A, N, N)
    B = sgg.normal_bf16(3, sg.ROLE_B, N, N)
    full = mm.gemm(A, B)
    mm.sync_check()
    absA, absB = A.float().abs(), B.float().abs()
    for G in (2, 4, 8):
        for r in range(G):
            r0, rows = mm.shard_range(N, G, r)
            Ab = A[r0:r0 + rows].contiguous()
            os.environ["MM_STREAMK"] = "0"
            try:
                blk = mm.gemm(Ab, B)
                mm.sync_check()
            finally:
                os.environ.pop("MM_STREAMK", None)
            assert torch.equal(blk, full[r0:r0 + rows]), (G, r)
            b1, b2 = mm.gemm(Ab, B), mm.gemm(Ab, B)
            mm.sync_check()
            assert torch.equal(b1, b2), (G, r)
            if not torch.equal(b1, full[r0:r0 + rows]):
                # normalised error vs the full product on a row sample (D = sum |a||b|)
                idx = torch.arange(0, rows, max(1, rows // 64), device="cuda")
                D = absA[r0 + idx] @ absB
                err = ((b1[idx] - full[r0 + idx]).abs() / D.clamp_min(1e-30)).max().item()
                assert err <= TOL["bf16"] and err <= DIAG_BF16, (G, r, err)
            del blk, b1, b2
    del full
    torch.cuda.empty_cache()


@pytest.mark.parametrize("K", [3, 9])
def test_config3_bf16_16384_exact_pins(mm, K):
    key = f"C4x{K}"
    if key not in FULL:
        pytest.skip(f"{key} golden not generated yet (tools/make_golden.py)")
    N = 16384
    A, B = gen("bf16", "exact", 3, N, N, N, K)
    Ct = mm.gemm(to_dev(A, "bf16"), to_dev(B, "bf16"))
    mm.sync_check()
    C = Ct.cpu().numpy()
    assert sg.checksum(C) == int(FULL[key]["checksum"], 16)
    rows = _sample(N, 16, 3, 30 + K, [0, N - 1, 8191, 8192])
    Cr, _ = oracle.gemm_bf16_rows(A, B, rows)
    assert np.array_equal(C[rows].astype(np.float64), Cr)


def test_config4_fp64_32768_exact_pin(mm):
    """configs[4]'s shape (FP64 32768^3, seed 4) on exact-integer inputs
    from [-1024, 1024] (every partial sum an integer < 2^53, so exact in any order): the
    full output's checksum equals the oracle's (tests/golden/oracle_fullsize.json, written by
    tools/make_golden.py from oracle/ only), bit for bit, as do its corners."""
    key = "C5x"
    if key not in FULL:
        pytest.skip(f"{key} golden not generated yet (tools/make_golden.py --only C5x)")
    from synthgen import gpu as sgg
    N = 32768
    A = sgg.exact_f64(4, sg.ROLE_A, 2049, N, N)
    B = sgg.exact_f64(4, sg.ROLE_B, 2049, N, N)
    C = mm.gemm(A, B)
    mm.sync_check()
    del A, B
    torch.cuda.empty_cache()
    Ch = C.cpu().numpy()
    del C
    g = FULL[key]
    assert Ch[0, 0] == g["C00"] and Ch[0, -1] == g["C0_last"]
    assert Ch[-1, 0] == g["Clast_0"] and Ch[-1, -1] == g["Clast_last"]
    assert sg.checksum(Ch) == int(g["checksum"], 16)


def test_config4_fp64_32768_sampled(mm):
    """configs[4] at full size on one GPU (the SUMMA G=1 reference), oracle on sampled rows/cols
    (>= 64 seeded rows and >= 64 seeded columns, plus the SUMMA grid's block
    boundaries — rows of the 2-row-block grids, columns of the 2- and 4-column-block grids of
    configs[4] at G = 2/4/8 — and the first/last row and column)."""
    N = 32768
    A, B = gen("f64", "random", 4, N, N, N)
    Ad, Bd = to_dev(A, "f64"), to_dev(B, "f64")
    C = mm.gemm(Ad, Bd)
    mm.sync_check()
    row_seams = [0, N - 1, 16383, 16384]
    col_seams = [0, N - 1] + [b + d for b in (8192, 16384, 24576) for d in (-1, 0)]
    rows = _sample(N, 64, 3, 4, row_seams)
    cols = _sample(N, 64, 4, 4, col_seams)
    assert rows.size >= 64 + len(row_seams) - 2 and cols.size >= 64 + len(col_seams) - 2
    Crow = C[torch.from_numpy(rows).cuda()].cpu().numpy()
    Ccol = C[:, torch.from_numpy(cols).cuda()].cpu().numpy()
    del C, Ad, Bd
    torch.cuda.empty_cache()
    Cr, Dr = oracle.gemm_f64_rows(A, B, rows)
    check("f64", Crow, Cr, Dr, exact=False)
    Cc, Dc = oracle.gemm_f64_cols(A, B, cols)
    check("f64", Ccol, Cc, Dc, exact=False)
    g = json.load(open(os.path.join(GOLDEN, "survey_c6.json")))["C5"]
    assert Crow[0, 0] == pytest.approx(g["C00"], abs=1e-12 * g["D00"])


@pytest.mark.parametrize("dt", ["i8", "bf16"])
def test_n_half_tail(mm, dt):
    """Tail mode 4: the partial last round's 256-wide pair tiles run as two N-halves on two
    clusters (pair MMA N = 128, whole K; int8 B through a SWIZZLE_64B map), no partial sums:
    bit-exact on exact-integer inputs, incl. ragged edges where a half lies outside C, and
    nothing written outside C (guard bands)."""
    os.environ["MM_STREAMK"] = "4"
    try:
        K = 255 if dt == "i8" else 9
        out = torch.float32 if dt == "bf16" else torch.int32
        for (m, n, p) in [(4096, 4096, 4096), (2560, 768, 2560), (2400, 1000, 2700), (4096, 512, 4096),
                          (1100, 2048, 1700), (2048, 4096, 2176)]:
            A, B = gen(dt, "exact", 53, m, n, p, K)
            Cref, _ = ref(dt, A, B)
            guard = 4096
            buf = torch.full((guard + m * p + guard,), -7, dtype=out, device="cuda")
            C = buf[guard:guard + m * p].view(m, p)
            Ad, Bd = to_dev(A, dt), to_dev(B, dt)
            for _ in range(3):
                mm.gemm(Ad, Bd, out=C)
            mm.sync_check()
            h = buf.cpu().numpy()
            assert np.all(h[:guard] == -7) and np.all(h[guard + m * p:] == -7), (m, n, p)
            assert np.array_equal(C.cpu().numpy().astype(np.float64), np.asarray(Cref, np.float64)), (m, n, p)
    finally:
        os.environ.pop("MM_STREAMK", None)


@pytest.mark.parametrize("dt", ["i8", "bf16"])
def test_n_half_tail_same_bits_as_whole_tiles(mm, dt):
    """N halves keep each element's K summation exactly as in a whole tile (only N is split), so
    random-valued results equal the whole-tile schedule bit for bit (R17: no K split)."""
    m, n, p = 4096, 2048, 4096
    A, B = gen(dt, "random", 54, m, n, p)
    Ad, Bd = to_dev(A, dt), to_dev(B, dt)
    outs = {}
    for mode in ("0", "4"):
        os.environ["MM_STREAMK"] = mode
        try:
            outs[mode] = mm.gemm(Ad, Bd)
            mm.sync_check()
        finally:
            os.environ.pop("MM_STREAMK", None)
    assert torch.equal(outs["0"], outs["4"])
    Cref, D = ref(dt, A[:64], B)
    check(dt, outs["4"][:64].cpu().numpy(), Cref, D, exact=False)


@pytest.mark.parametrize("shape", [(256, 256, 256), (2000, 1500, 1750), (1000, 333, 517), (37, 4100, 29), (1, 1, 1),
                                   (3300, 700, 3100)])
def test_f64_emulation(mm, shape):
    """MM_F64_EMU (f64_emu.cu): the binary64 product on the INT8 tensor cores (integer scaling,
    residues modulo 14-16 coprime moduli, one exact INT8 product per modulus, Chinese remaindering).
    Exact-integer inputs (|x| <= 1024, K = 2049 pins) bit-exact — the scaling leaves integers
    unrounded and the remaindering is exact; U[-1,1) inputs within the FP64 tolerance of the oracle
    and, diagnostically, of DMMA's ~1e-16; ragged n (K padding) and p % 16 != 0 (padded planes).
    Below two waves of tiles the N products run as one batched launch; 3300x700x3100 (169 tiles)
    takes the N-launch path."""
    m, n, p = shape
    A, B = gen("f64", "exact", 71, m, n, p, 2049)
    Cref, _ = ref("f64", A, B)
    C = mm.gemm(to_dev(A, "f64"), to_dev(B, "f64"), f64_emulation=True)
    mm.sync_check()
    assert np.array_equal(C.cpu().numpy(), Cref)
    A, B = gen("f64", "random", 72, m, n, p)
    Cref, D = ref("f64", A, B)
    C = mm.gemm(to_dev(A, "f64"), to_dev(B, "f64"), f64_emulation=True)
    mm.sync_check()
    err = oracle.normalized_error(C.cpu().numpy(), Cref, D)
    assert err <= TOL["f64"], err
    assert err <= 1e-15, f"diagnostic: emulation error {err} well above DMMA's"


def test_f64_emulation_dynamic_range(mm):
    """MM_F64_EMU scales each row of A / column of B by its own power of two: rows spanning 2^-450 ..
    2^450, columns 2^-450 .. 2^450 (products stay finite), one row decaying over 2^-60 inside itself, an all-zero row and
    column, subnormal entries; the result matches the oracle within the FP64 tolerance (normalised by
    Σ|a·b| per element) and within DMMA's ~1e-16 class diagnostically.  Zero rows / columns give
    exact zeros."""
    m, n, p = 300, 1000, 260
    A, B = gen("f64", "random", 73, m, n, p)
    rng = np.random.default_rng(73)
    A = A * np.ldexp(1.0, rng.integers(-450, 450, m))[:, None]
    B = B * np.ldexp(1.0, rng.integers(-450, 450, p))[None, :]
    A[5] = A[5] * np.ldexp(1.0, -(np.arange(n) * 60 // n))  # within-row range of 2^60
    A[7] = 0.0
    B[:, 11] = 0.0
    A[9] = np.ldexp(A[9], -1070)  # subnormal row (products underflow; the oracle's do too)
    A[9, :3] = [4.9e-324, -4.9e-324, 0.0]
    Cref, D = ref("f64", A, B)
    C = mm.gemm(to_dev(A, "f64"), to_dev(B, "f64"), f64_emulation=True)
    mm.sync_check()
    C = C.cpu().numpy()
    assert np.all(C[7] == 0.0) and np.all(C[:, 11] == 0.0)
    keep = np.ones(m, bool)
    keep[9] = False  # subnormal row: compared in absolute terms below
    err = oracle.normalized_error(C[keep], Cref[keep], D[keep])
    assert err <= TOL["f64"], err
    keep[5] = False
    err = oracle.normalized_error(C[keep], Cref[keep], D[keep])
    assert err <= 1e-15, f"diagnostic: emulation error {err} well above DMMA's"
    # row 5 (its elements fall to 2^-60 of its maximum): each a_5k carries a scaling error up to
    # 2^-54 of the row maximum, while D counts |a_5k| itself — the a-priori bound is
    # 2^-53 · max|a_5·| · Σ|b| / D ≈ 2^-53 · 60/ln 2 / 2 ≈ 5e-15 of D
    err5 = oracle.normalized_error(C[5], Cref[5], D[5])
    assert err5 <= 1e-14, err5
    assert np.max(np.abs(C[9] - Cref[9])) <= 1e-300


def test_f64_emulation_long_k(mm):
    """n beyond what 7-bit digit slicing allowed (33280): n = 70001 (ragged), exact-integer inputs
    bit-exact against the oracle and random inputs within tolerance; n = 131072 (INT32 sums of
    residue products could overflow) is refused with MM_ERR_UNSUPPORTED, not computed wrongly."""
    m, n, p = 40, 70001, 36
    A, B = gen("f64", "exact", 74, m, n, p, 2049)
    Cref, _ = ref("f64", A, B)
    C = mm.gemm(to_dev(A, "f64"), to_dev(B, "f64"), f64_emulation=True)
    mm.sync_check()
    assert np.array_equal(C.cpu().numpy(), Cref)
    A, B = gen("f64", "random", 75, m, n, p)
    Cref, D = ref("f64", A, B)
    C = mm.gemm(to_dev(A, "f64"), to_dev(B, "f64"), f64_emulation=True)
    mm.sync_check()
    err = oracle.normalized_error(C.cpu().numpy(), Cref, D)
    assert err <= TOL["f64"] and err <= 1e-15, err
    Ad = torch.zeros(2, 131072, dtype=torch.float64, device="cuda")
    Bd = torch.zeros(131072, 2, dtype=torch.float64, device="cuda")
    with pytest.raises(RuntimeError, match="131071|exact-INT32"):
        mm.gemm(Ad, Bd, f64_emulation=True)


def test_f64_emulation_non_finite_reported(mm):
    """MM_F64_EMU cannot propagate Inf / NaN through integer arithmetic: an Inf in A or a NaN in B is
    detected by the scale kernels and reported by mm_sync_check (MM_ERR_RUNTIME naming the cause);
    the context stays usable (the next finite product is exact)."""
    m, n, p = 64, 96, 80
    A, B = gen("f64", "exact", 76, m, n, p, 2049)
    for where in ("A", "B"):
        Ab, Bb = A.copy(), B.copy()
        if where == "A":
            Ab[3, 5] = np.inf
        else:
            Bb[7, 2] = np.nan
        mm.gemm(to_dev(Ab, "f64"), to_dev(Bb, "f64"), f64_emulation=True)
        with pytest.raises(RuntimeError, match="Inf or NaN"):
            mm.sync_check()
    C = mm.gemm(to_dev(A, "f64"), to_dev(B, "f64"), f64_emulation=True)
    mm.sync_check()
    assert np.array_equal(C.cpu().numpy(), oracle.gemm_f64(A, B))


def test_f64_emulation_config1_golden(mm):
    """C2x (configs[1] shape, K=2049 exact pin): the emulated product's full-output checksum equals
    SURVEY c7's golden, like DMMA's."""
    m, n, p = 2000, 1500, 1750
    A, B = gen("f64", "exact", 1, m, n, p, 2049)
    C = mm.gemm(to_dev(A, "f64"), to_dev(B, "f64"), f64_emulation=True)
    mm.sync_check()
    assert sg.checksum(C.cpu().numpy()) == int(FULL["C2x"]["checksum"], 16)


def test_config4_fp64_32768_emulated(mm):
    """configs[4] at full size through MM_F64_EMU: the C5x exact pin (K=2049 integers; scaling,
    residue products and remaindering exact) hashes to the oracle's golden bit for bit; random U[-1,1)
    inputs match the oracle on >= 64 seeded rows and >= 64 seeded columns (+ seams) within 1e-12,
    and diagnostically within 1e-15."""
    from synthgen import gpu as sgg
    N = 32768
    A = sgg.exact_f64(4, sg.ROLE_A, 2049, N, N)
    B = sgg.exact_f64(4, sg.ROLE_B, 2049, N, N)
    C = mm.gemm(A, B, f64_emulation=True)
    mm.sync_check()
    del A, B
    Ch = C.cpu().numpy()
    del C
    torch.cuda.empty_cache()
    assert sg.checksum(Ch) == int(FULL["C5x"]["checksum"], 16)
    del Ch
    A, B = gen("f64", "random", 4, N, N, N)
    C = mm.gemm(to_dev(A, "f64"), to_dev(B, "f64"), f64_emulation=True)
    mm.sync_check()
    rows = _sample(N, 64, 3, 4, [0, N - 1, 16383, 16384])
    cols = _sample(N, 64, 4, 4, [0, N - 1, 8191, 8192])
    Crow = C[torch.from_numpy(rows).cuda()].cpu().numpy()
    Ccol = C[:, torch.from_numpy(cols).cuda()].cpu().numpy()
    del C
    torch.cuda.empty_cache()
    Cr, Dr = oracle.gemm_f64_rows(A, B, rows)
    Cc, Dc = oracle.gemm_f64_cols(A, B, cols)
    for got, want, D in ((Crow, Cr, Dr), (Ccol, Cc, Dc)):
        err = oracle.normalized_error(got, want, D)
        assert err <= TOL["f64"], err
        assert err <= 1e-15, f"diagnostic: {err}"
