"""mm_gemm_sharded through NCCL on the one GPU this round has (world size 1):
the row-block path with MM_BCAST_B | MM_GATHER_C and the SUMMA 1×1 path run the
real NCCL calls (broadcast, grouped send/recv, comm split) and must equal the
oracle bit-exactly on exact-integer inputs.  Multi-rank schedules are covered on
CPU by tests/test_dist_gloo.py."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synthgen as sg

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def pg(cuda_device):
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_row_block_world1(pg):
    import paper_2408_15384_b200 as mm
    m, n, p = 1000, 768, 520
    for dt, gen in (("bf16", sg.exact_bf16), ("i8", sg.exact_i8), ("f64", sg.exact_f64)):
        K = {"bf16": 9, "i8": 255, "f64": 2049}[dt]
        A, B = gen(31, 1, K, m, n), gen(31, 2, K, n, p)
        if dt == "bf16":
            tA = torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).cuda()
            tB = torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).cuda()
            Cref, _ = oracle.gemm_bf16(A, B)
            tdt, odt = torch.bfloat16, torch.float32
        elif dt == "i8":
            tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
            Cref = oracle.gemm_s8(A, B)
            tdt, odt = torch.int8, torch.int32
        else:
            tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
            Cref = oracle.gemm_f64(A, B)
            tdt, odt = torch.float64, torch.float64
        C_loc = torch.empty(m, p, dtype=odt, device="cuda")
        C_full = torch.zeros(m, p, dtype=odt, device="cuda")
        mm.gemm_sharded(m, n, p, tdt, tA, tB, C_loc, layout=mm.MM_ROW_BLOCK,
                        flags=mm.MM_BCAST_B | mm.MM_GATHER_C, root=0, C_full=C_full)
        mm.sync_check()
        assert np.array_equal(C_loc.cpu().numpy().astype(np.float64), np.asarray(Cref, np.float64)), dt
        assert np.array_equal(C_full.cpu().numpy().astype(np.float64), np.asarray(Cref, np.float64)), dt


def test_row_block_fused_gather_world1(pg):
    """MM_GATHER_C_FUSED: the product kernel stores straight into the root's C_full
    (at world size 1 the root maps its own buffer; the IPC open path needs >= 2 GPUs)."""
    import paper_2408_15384_b200 as mm
    m, n, p = 1000, 512, 776
    for dt in ("bf16", "i8", "f64"):
        if dt == "bf16":
            A, B = sg.exact_bf16(34, 1, 9, m, n), sg.exact_bf16(34, 2, 9, n, p)
            tA = torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).cuda()
            tB = torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).cuda()
            Cref, _ = oracle.gemm_bf16(A, B)
            tdt, odt = torch.bfloat16, torch.float32
        elif dt == "i8":
            A, B = sg.exact_i8(34, 1, 255, m, n), sg.exact_i8(34, 2, 255, n, p)
            tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
            Cref = oracle.gemm_s8(A, B)
            tdt, odt = torch.int8, torch.int32
        else:
            A, B = sg.exact_f64(34, 1, 2049, m, n), sg.exact_f64(34, 2, 2049, n, p)
            tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
            Cref = oracle.gemm_f64(A, B)
            tdt, odt = torch.float64, torch.float64
        big = torch.zeros(m + 7, p, dtype=odt, device="cuda")  # C_full inside a larger allocation
        C_full = big[3:3 + m]
        flags = mm.MM_GATHER_C_FUSED | (mm.MM_BCAST_B if dt != "f64" else 0)  # + panel-chunked broadcast
        mm.gemm_sharded(m, n, p, tdt, tA, tB, None, layout=mm.MM_ROW_BLOCK, flags=flags, root=0,
                        C_full=C_full)
        mm.sync_check()
        assert np.array_equal(C_full.cpu().numpy().astype(np.float64), np.asarray(Cref, np.float64)), dt
        assert not big[:3].any() and not big[3 + m:].any()


@pytest.mark.parametrize("panel", ["64", "2048"])
def test_summa_world1_fp64(pg, panel):
    import paper_2408_15384_b200 as mm
    os.environ["MM_SUMMA_PANEL"] = panel
    try:
        m, n, p = 700, 1000, 900
        A, B = sg.exact_f64(32, 1, 2049, m, n), sg.exact_f64(32, 2, 2049, n, p)
        C = torch.empty(m, p, dtype=torch.float64, device="cuda")
        mm.gemm_sharded(m, n, p, torch.float64, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), C,
                        layout=mm.MM_SUMMA_2D, grid=(1, 1))
        mm.sync_check()
        assert np.array_equal(C.cpu().numpy(), oracle.gemm_f64(A, B))
        # random values: panels accumulate with beta=1, within the FP64 tolerance
        A, B = sg.uniform_f64(33, 1, m, n), sg.uniform_f64(33, 2, n, p)
        mm.gemm_sharded(m, n, p, torch.float64, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), C,
                        layout=mm.MM_SUMMA_2D, grid=(1, 1))
        mm.sync_check()
        err = oracle.normalized_error(C.cpu().numpy(), oracle.gemm_f64(A, B), oracle.absden_f64(A, B))
        assert err <= 1e-12, err
    finally:
        os.environ.pop("MM_SUMMA_PANEL", None)


@pytest.mark.parametrize("layout", ["summa", "row_block"])
def test_sharded_world1_fp64_emulated(pg, layout):
    """MM_F64_EMU through mm_gemm_sharded (real NCCL calls at world size 1): SUMMA k-panels of 256
    accumulate into C (β = 1: each panel's emulated product is rounded once, then added) and the
    row block with B broadcast + gather; exact-integer inputs bit-exact, random inputs within the
    FP64 tolerance and the DMMA-class diagnostic."""
    import paper_2408_15384_b200 as mm
    m, n, p = 700, 1000, 900
    kw = dict(layout=mm.MM_SUMMA_2D, grid=(1, 1)) if layout == "summa" else \
        dict(flags=mm.MM_BCAST_B | mm.MM_GATHER_C)
    os.environ["MM_SUMMA_PANEL"] = "256"
    try:
        for kind in ("exact", "random"):
            A, B = (sg.exact_f64(36, 1, 2049, m, n), sg.exact_f64(36, 2, 2049, n, p)) if kind == "exact" else \
                (sg.uniform_f64(37, 1, m, n), sg.uniform_f64(37, 2, n, p))
            C = torch.empty(m, p, dtype=torch.float64, device="cuda")
            Cf = torch.empty(m, p, dtype=torch.float64, device="cuda") if layout == "row_block" else None
            mm.gemm_sharded(m, n, p, torch.float64, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), C,
                            C_full=Cf, f64_emulation=True, **kw)
            mm.sync_check()
            got = (Cf if Cf is not None else C).cpu().numpy()
            if kind == "exact":
                assert np.array_equal(got, oracle.gemm_f64(A, B))
            else:
                err = oracle.normalized_error(got, oracle.gemm_f64(A, B), oracle.absden_f64(A, B))
                assert err <= 1e-12 and err <= 1e-15, err
    finally:
        os.environ.pop("MM_SUMMA_PANEL", None)


def test_sharded_usage_errors(pg):
    import paper_2408_15384_b200 as mm
    t = torch.zeros(4, 4, dtype=torch.float64, device="cuda")
    with pytest.raises(mm.MMError, match="grid"):
        mm.gemm_sharded(4, 4, 4, torch.float64, t, t.clone(), t.clone(), layout=mm.MM_SUMMA_2D, grid=(2, 1))
    with pytest.raises(mm.MMError, match="root"):
        mm.gemm_sharded(4, 4, 4, torch.float64, t, t.clone(), t.clone(), layout=mm.MM_ROW_BLOCK, root=3)


def test_summa25d_world1_fp64(pg):
    """MM_SUMMA_25D at world size 1 (one layer of a 1x1 grid): the layer/panel/reduce code
    path with the real NCCL calls; the multi-layer schedule is checked over gloo."""
    import paper_2408_15384_b200 as mm
    m, n, p = 500, 3000, 700
    A, B = sg.exact_f64(35, 1, 2049, m, n), sg.exact_f64(35, 2, 2049, n, p)
    C = torch.empty(m, p, dtype=torch.float64, device="cuda")
    mm.gemm_sharded(m, n, p, torch.float64, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), C,
                    layout=mm.MM_SUMMA_25D, grid=(1, 1), flags=mm.MM_REPLICATE)
    mm.sync_check()
    assert np.array_equal(C.cpu().numpy(), oracle.gemm_f64(A, B))


def test_collective_argument_check(pg):
    """MM_CHECK_COLLECTIVE=1: the hash all-reduce runs (world size 1: always consistent) and the
    product is unchanged."""
    import paper_2408_15384_b200 as mm
    m, n, p = 300, 200, 260
    A, B = sg.exact_f64(36, 1, 2049, m, n), sg.exact_f64(36, 2, 2049, n, p)
    C = torch.empty(m, p, dtype=torch.float64, device="cuda")
    os.environ["MM_CHECK_COLLECTIVE"] = "1"
    try:
        mm.gemm_sharded(m, n, p, torch.float64, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), C,
                        layout=mm.MM_ROW_BLOCK)
        mm.sync_check()
    finally:
        os.environ.pop("MM_CHECK_COLLECTIVE", None)
    assert np.array_equal(C.cpu().numpy(), oracle.gemm_f64(A, B))


def test_row_block_fused_gather_window_world1(pg):
    """MM_GATHER_C_FUSED | MM_C_WINDOW: C_full is NCCL symmetric memory
    (mm_window_alloc: ncclMemAlloc + ncclCommWindowRegister) and the root's address comes from the
    window (ncclGetPeerPointer) instead of a CUDA-IPC handle exchange.  At world size 1 the root
    is this rank; the window, its device-side descriptor and the products' TMA stores through the
    resolved address all run for real.  C_full sits at an offset inside the window (symmetric)."""
    import paper_2408_15384_b200 as mm
    m, n, p = 1000, 512, 776
    for dt in ("bf16", "i8", "f64"):
        if dt == "bf16":
            A, B = sg.exact_bf16(37, 1, 9, m, n), sg.exact_bf16(37, 2, 9, n, p)
            tA = torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).cuda()
            tB = torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).cuda()
            Cref, _ = oracle.gemm_bf16(A, B)
            tdt, odt = torch.bfloat16, torch.float32
        elif dt == "i8":
            A, B = sg.exact_i8(37, 1, 255, m, n), sg.exact_i8(37, 2, 255, n, p)
            tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
            Cref = oracle.gemm_s8(A, B)
            tdt, odt = torch.int8, torch.int32
        else:
            A, B = sg.exact_f64(37, 1, 2049, m, n), sg.exact_f64(37, 2, 2049, n, p)
            tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
            Cref = oracle.gemm_f64(A, B)
            tdt, odt = torch.float64, torch.float64
        win = mm.window_alloc((m + 7, p), odt)
        try:
            win.zero_()
            C_full = win[3:3 + m]
            flags = mm.MM_GATHER_C_FUSED | mm.MM_C_WINDOW | (mm.MM_BCAST_B if dt != "f64" else 0)
            mm.gemm_sharded(m, n, p, tdt, tA, tB, None, layout=mm.MM_ROW_BLOCK, flags=flags, root=0,
                            C_full=C_full)
            mm.sync_check()
            assert np.array_equal(C_full.cpu().numpy().astype(np.float64), np.asarray(Cref, np.float64)), dt
            assert not win[:3].any() and not win[3 + m:].any()
        finally:
            mm.window_free(win)


def test_window_usage_errors(pg):
    import paper_2408_15384_b200 as mm
    t = torch.zeros(64, 64, dtype=torch.float64, device="cuda")
    with pytest.raises(mm.MMError, match="MM_C_WINDOW applies"):
        mm.gemm_sharded(64, 64, 64, torch.float64, t, t.clone(), t.clone(), layout=mm.MM_ROW_BLOCK,
                        flags=mm.MM_C_WINDOW, C_full=t.clone())
    with pytest.raises(mm.MMError, match="not in a buffer from mm_window_alloc"):
        mm.gemm_sharded(64, 64, 64, torch.float64, t, t.clone(), None, layout=mm.MM_ROW_BLOCK,
                        flags=mm.MM_GATHER_C_FUSED | mm.MM_C_WINDOW, C_full=t.clone())
    with pytest.raises(mm.MMError, match="was not returned by mm_window_alloc"):
        mm.window_free(t)
