"""Products that must stay correct — and must not stall — when the GPU is shared.

1. Residency: the persistent grid is sized for an idle GPU.  Here a test kernel holds most SMs
   (tests/csrc/hog.cu, one 200-KB block per SM, like a long NCCL collective or another product),
   so only a few of the product's CTAs are resident at first.  The product must finish correctly
   long before the hog does: the wave barrier is soft (abandoned after 0.5 ms) and a split tile's
   parts only ever wait for parts that already took a ticket (running CTAs) — no CTA waits for one
   that has not started.
2. Streams: one context used on two streams with overlapping launches; its scratch (wave counters,
   split-tile tickets, partial slabs) is ordered across streams by an event.
3. Release build: diagnostic knobs are refused.
"""
import ctypes
import os
import time

import numpy as np
import pytest
import torch

import oracle
import synthgen as sg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mm(cuda_device):
    import paper_2408_15384_b200 as m
    return m


@pytest.fixture(scope="module")
def hog():
    lib = ctypes.CDLL(os.path.join(ROOT, "tests", "libhog.so"))
    lib.hog_launch.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p]
    lib.hog_launch.restype = ctypes.c_int
    lib.hog_started.restype = ctypes.c_uint
    return lib


def _exact(dt, seed, m, n, p):
    if dt == "bf16":
        A, B = sg.exact_bf16(seed, 1, 9, m, n), sg.exact_bf16(seed, 2, 9, n, p)
        tA = torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).cuda()
        tB = torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).cuda()
    elif dt == "i8":
        A, B = sg.exact_i8(seed, 1, 255, m, n), sg.exact_i8(seed, 2, 255, n, p)
        tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    else:
        A, B = sg.exact_f64(seed, 1, 2049, m, n), sg.exact_f64(seed, 2, 2049, n, p)
        tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    return tA, tB


def _exact_ref(tA, tB):
    # exact-integer operands: every partial sum is an integer < 2^53, so an FP64 product is exact
    return torch.mm(tA.to(torch.float64), tB.to(torch.float64))


# (dtype, m, n, p, what it exercises)
SHARED_CASES = [
    ("bf16", 8192, 8192, 8192, "wave barrier (operands > 96 MB), 512-wide pair tiles"),
    ("bf16", 2560, 2560, 2560, "N-half split tail (mode 4)"),
    ("bf16", 4096, 4096, 4096, "reduce-add split tail (mode 3 tickets: the first ticket zeroes C)"),
    ("i8", 4096, 4096, 4096, "configs[2] shape, 256-wide pair tiles"),
    ("f64", 2000, 1500, 1750, "configs[1] shape, FP64 split tail (tickets + publish counts)"),
    ("f64", 4096, 4096, 4096, "FP64 96x128 tiles (12 warps), split tail"),
]


@pytest.mark.parametrize("dt,m,n,p,what", SHARED_CASES)
def test_product_while_sms_are_held(mm, hog, dt, m, n, p, what):
    """A product launched while a kernel holds all but 16 SMs for 6 s completes correctly in well
    under that time (it does not wait for the SMs to be released), and latches no error."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks = sms - 16
    tA, tB = _exact(dt, 71, m, n, p)
    ref = _exact_ref(tA, tB)
    C = mm.gemm(tA, tB)  # warm-up: plans, tensor maps, scratch allocations
    mm.sync_check()
    C.zero_()
    s_hog = torch.cuda.Stream()
    hold_ns = 6_000_000_000
    assert hog.hog_launch(blocks, hold_ns, ctypes.c_void_p(s_hog.cuda_stream)) == 0
    t0 = time.time()
    while hog.hog_started() < blocks:
        assert time.time() - t0 < 5, f"hog did not start ({hog.hog_started()} of {blocks} blocks)"
        time.sleep(0.001)
    t_launch = time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mm.gemm(tA, tB, out=C)
    e1.record()
    e1.synchronize()
    waited = time.time() - t_launch
    still_held = hog.hog_started() == blocks and waited < hold_ns * 1e-9 - 0.5
    s_hog.synchronize()
    mm.sync_check()  # no pipeline time-out latched
    assert still_held and waited < 3.0, (what, waited)
    assert torch.equal(C.to(torch.float64), ref), what


def test_one_context_two_streams(mm):
    """Overlapping launches of one context on two streams (split-tail, wave-barrier and FP64
    split shapes, alternating streams, no host synchronisation in between): every output exact."""
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cases = [("bf16", 2560, 2560, 2560), ("bf16", 8192, 4096, 8192), ("f64", 2000, 1500, 1750), ("i8", 2400, 5000, 2700)]
    ops = [(*c, _exact(c[0], 80 + i, *c[1:])) for i, c in enumerate(cases)]
    refs = [_exact_ref(tA, tB) for (_, _, _, _, (tA, tB)) in ops]
    torch.cuda.synchronize()
    outs = []
    for rep in range(3):
        for i, (dt, m, n, p, (tA, tB)) in enumerate(ops):
            s = s1 if (rep + i) % 2 == 0 else s2
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                outs.append((i, mm.gemm(tA, tB)))
    torch.cuda.synchronize()
    mm.sync_check()
    for i, C in outs:
        assert torch.equal(C.to(torch.float64), refs[i]), cases[i]


@pytest.mark.parametrize("knob", ["MM_DEBUG", "MM_TRACE", "MM_HOST_TRACE"])
def test_release_library_refuses_diag_knobs(mm, knob):
    A = torch.ones(64, 64, dtype=torch.bfloat16, device="cuda")
    os.environ[knob] = "1"
    try:
        with pytest.raises(mm.MMError, match="diagnostic"):
            mm.gemm(A, A)
    finally:
        os.environ.pop(knob)
    C = mm.gemm(A, A)
    mm.sync_check()
    assert torch.all(C == 64)


def test_workspace_size_bounds_allocation(mm):
    """mm_workspace_size is an upper bound of what a fresh context allocates for the call."""
    for dt, m, n, p in [("bf16", 4096, 3000, 4096), ("f64", 2000, 1500, 1750), ("i8", 4096, 4096, 4096)]:
        tA, tB = _exact(dt, 90, m, n, p)
        torch.cuda.synchronize()
        ctx = mm.Context(0)
        free0 = torch.cuda.mem_get_info()[0]
        out = torch.empty(m, p, dtype={"bf16": torch.float32, "i8": torch.int32, "f64": torch.float64}[dt],
                          device="cuda")
        free1 = torch.cuda.mem_get_info()[0]
        from paper_2408_15384_b200 import _lib
        st = _lib.load().mm_gemm(ctx.handle, m, n, p, mm.IN_DTYPE[tA.dtype], tA.data_ptr(), tB.data_ptr(),
                                 out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        ctx.check(st)
        ctx.check(_lib.load().mm_sync_check(ctx.handle, torch.cuda.current_stream().cuda_stream))
        used = free1 - torch.cuda.mem_get_info()[0]
        bound = mm.workspace_size(m, n, p, tA.dtype)
        ctx.close()
        # allocation granularity of the driver: 2 MiB pages
        assert used <= bound + (8 << 20), (dt, used, bound)
        assert torch.equal(out.to(torch.float64), _exact_ref(tA, tB))


def test_workspace_size_bounds_allocation_f64_emulated(mm):
    """The same bound for MM_F64_EMU: residue planes, INT32 product and the INT8 product's scratch."""
    m, n, p = 2000, 1500, 1750
    g = torch.Generator(device="cuda").manual_seed(92)
    A = torch.randint(-1000, 1000, (m, n), generator=g, device="cuda").double()
    B = torch.randint(-1000, 1000, (n, p), generator=g, device="cuda").double()
    torch.cuda.synchronize()
    ctx = mm.Context(0)
    out = torch.empty(m, p, dtype=torch.float64, device="cuda")
    free1 = torch.cuda.mem_get_info()[0]
    from paper_2408_15384_b200 import _lib
    s = torch.cuda.current_stream().cuda_stream
    ctx.check(_lib.load().mm_gemm(ctx.handle, m, n, p, mm.MM_F64_EMU, A.data_ptr(), B.data_ptr(), out.data_ptr(), s))
    ctx.check(_lib.load().mm_sync_check(ctx.handle, s))
    used = free1 - torch.cuda.mem_get_info()[0]
    bound = mm.workspace_size(m, n, p, torch.float64, f64_emulation=True)
    ctx.close()
    assert used <= bound + (8 << 20), (used, bound)
    assert torch.equal(out, A @ B)  # exact integers: cuBLAS's DGEMM is exact here too


def test_clock_meter(mm):
    """mm_clock_meter: records the effective SM clock of a product kernel without changing it."""
    for dt, m, n, p in [("bf16", 4096, 4096, 4096), ("f64", 1024, 1024, 1024), ("i8", 2048, 2048, 2048)]:
        tA, tB = _exact(dt, 91, m, n, p)
        ref = _exact_ref(tA, tB)
        assert mm.clock_meter(True) == 0.0
        C = mm.gemm(tA, tB)
        mhz = mm.clock_meter(False)
        mm.sync_check()
        assert 300.0 < mhz < 2300.0, (dt, mhz)
        assert torch.equal(C.to(torch.float64), ref)
