"""The library's real sharded executor and kernels at world sizes 2-4 on ONE GPU.

NCCL refuses two ranks on one device, so this test loads a test-only stand-in for the NCCL entry
points the library resolves (tests/csrc/fake_nccl.cu, selected with MM_NCCL_LIB): several processes
share the GPU, each collective synchronises its stream and moves data on the host's command
through CUDA IPC and cudaMemcpy, ranks meet at shared-memory barriers.  No kernel waits for another
rank and nothing is timed — it is a correctness harness for csrc/shard.cu at G > 1: the plan
execution (stream events, staging copies, pitched panels), the sub-communicator splits of SUMMA and
2.5D, the gather's send/receive, the fused gather's IPC handle exchange, peer mapping and the
product kernels' stores into the root's C, and the collective argument check — every assembled C
bit-exact against the oracle on exact-integer inputs.  (tests/test_dist_nccl.py runs the same
library over real NCCL when a box has >= 2 GPUs.)"""
import ctypes
import os
import uuid

import numpy as np
import pytest
import torch
import torch.multiprocessing as tmp

import plan_exec as px  # tests/plan_exec.py: the result dtypes and oracle product helper
import synthgen as sg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAKE = os.path.join(ROOT, "tests", "libfakenccl.so")
DT_CODE = {"f64": 0, "bf16": 1, "i8": 2, "emu": 3}  # emu: MM_F64_EMU (float64 operands)
TIN = {"f64": torch.float64, "bf16": torch.bfloat16, "i8": torch.int8, "emu": torch.float64}
TOUT = {"f64": torch.float64, "bf16": torch.float32, "i8": torch.int32, "emu": torch.float64}
KEXACT = {"f64": 2049, "bf16": 9, "i8": 255, "emu": 2049}


def _inputs(kind, m, n, p, seed=77):
    gen = {"f64": sg.exact_f64, "bf16": sg.exact_bf16, "i8": sg.exact_i8, "emu": sg.exact_f64}[kind]
    return gen(seed, 1, KEXACT[kind], m, n), gen(seed, 2, KEXACT[kind], n, p)


def _dev(x, kind):
    if kind == "bf16":
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _worker(rank, world, shm, cases, q):
    os.environ["MM_NCCL_LIB"] = FAKE
    import paper_2408_15384_b200 as mm
    torch.cuda.set_device(0)
    fake = ctypes.CDLL(FAKE)
    fake.fake_comm_init.restype = ctypes.c_void_p
    fake.fake_comm_init.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
    comm = fake.fake_comm_init(rank, world, shm.encode())
    assert comm, "fake_comm_init failed"
    lib = mm._lib.load()
    ctx = mm.context(0)
    stream = torch.cuda.current_stream().cuda_stream
    for i, (layout, kind, m, n, p, flags, root, grid, check_env) in enumerate(cases):
        try:
            if check_env:
                os.environ["MM_CHECK_COLLECTIVE"] = "1"
            A, B = _inputs(kind, m, n, p)
            if layout == mm.MM_ROW_BLOCK:
                if check_env == "mismatch":
                    m += rank  # rank-dependent argument: must be refused on every rank
                    A, B = _inputs(kind, m, n, p)
                s, c = mm.shard_range(m, world, rank)
                Ad = _dev(A[s:s + c], kind)
                have_b = rank == root or not (flags & mm.MM_BCAST_B)
                Bd = _dev(B, kind) if have_b else torch.zeros(n, p, dtype=TIN[kind], device="cuda")
                Cl = torch.full((max(c, 1), p), -9, dtype=TOUT[kind], device="cuda")
                Cf = torch.full((m, p), -9, dtype=TOUT[kind], device="cuda") if rank == root else None
                fused = bool(flags & mm.MM_GATHER_C_FUSED)
                st = lib.mm_gemm_sharded(ctx.handle, m, n, p, DT_CODE[kind], layout, 0, 0, Ad.data_ptr() if c else None,
                                         Bd.data_ptr(), None if (fused or not c) else Cl.data_ptr(),
                                         Cf.data_ptr() if Cf is not None else None, flags, root, comm, stream)
                if check_env == "mismatch":
                    q.put((i, rank, {"status": st, "error": lib.mm_last_error(ctx.handle).decode()}))
                    continue
                ctx.check(st)
                mm.sync_check()
                res = {"C": Cl[:c].cpu().numpy(), "rows": (s, c), "B": Bd.cpu().numpy() if kind != "bf16" else
                       Bd.view(torch.int16).cpu().numpy().view(np.uint16)}
                if rank == root:
                    res["CFULL"] = Cf.cpu().numpy()
            else:
                pr, pc = grid
                g2 = pr * pc
                l, r2 = rank // g2, rank % g2
                gi, gj = r2 // pc, r2 % pc
                am, ak = mm.shard_range(m, pr, gi), mm.shard_range(n, pc, gj)
                bk, bn = mm.shard_range(n, pr, gi), mm.shard_range(p, pc, gj)
                Ab = A[am[0]:am[0] + am[1], ak[0]:ak[0] + ak[1]]
                Bb = B[bk[0]:bk[0] + bk[1], bn[0]:bn[0] + bn[1]]
                if layout == mm.MM_SUMMA_25D and l > 0:
                    Ab, Bb = np.zeros_like(Ab), np.zeros_like(Bb)
                Ad, Bd = _dev(Ab, kind), _dev(Bb, kind)
                Cb = torch.full((am[1], bn[1]), -5.0, dtype=torch.float64, device="cuda")
                os.environ["MM_SUMMA_PANEL"] = "96"
                try:
                    st = lib.mm_gemm_sharded(ctx.handle, m, n, p, DT_CODE[kind], layout, pr, pc, Ad.data_ptr(),
                                             Bd.data_ptr(), Cb.data_ptr(), None, flags, root, comm, stream)
                finally:
                    os.environ.pop("MM_SUMMA_PANEL", None)
                ctx.check(st)
                mm.sync_check()
                res = {"C": Cb.cpu().numpy(), "layer": l, "rows": am, "cols": bn}
            q.put((i, rank, res))
        except Exception as e:  # noqa: BLE001
            q.put((i, rank, {"exc": f"{type(e).__name__}: {e}"}))
            raise
        finally:
            os.environ.pop("MM_CHECK_COLLECTIVE", None)


def _run(world, cases):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    shm = f"/mm_fake_nccl_{uuid.uuid4().hex[:12]}"
    procs = [ctx.Process(target=_worker, args=(r, world, shm, cases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = {}
    try:
        for _ in range(world * len(cases)):
            i, r, res = q.get(timeout=600)
            assert "exc" not in res, (cases[i], r, res["exc"])
            out[(i, r)] = res
    finally:
        for pr in procs:
            pr.join(timeout=120)
        try:
            os.unlink("/dev/shm" + shm)
        except OSError:
            pass
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    return out


def _check(world, cases, out):
    import paper_2408_15384_b200 as mm
    for i, (layout, kind, m, n, p, flags, root, grid, check_env) in enumerate(cases):
        if check_env == "mismatch":
            for r in range(world):
                assert out[(i, r)]["status"] == 2 and "differ across" in out[(i, r)]["error"], out[(i, r)]
            continue
        A, B = _inputs(kind, m, n, p)
        Cref = px._local_product("f64" if kind == "emu" else kind, A, B).astype(np.float64)
        if layout == mm.MM_ROW_BLOCK:
            if flags & (mm.MM_GATHER_C | mm.MM_GATHER_C_FUSED):
                assert np.array_equal(out[(i, root)]["CFULL"].astype(np.float64), Cref), case_name(cases[i])
            if not flags & mm.MM_GATHER_C_FUSED:
                for r in range(world):
                    s, c = out[(i, r)]["rows"]
                    assert np.array_equal(out[(i, r)]["C"].astype(np.float64), Cref[s:s + c]), (case_name(cases[i]), r)
            if flags & mm.MM_BCAST_B:
                for r in range(world):
                    assert np.array_equal(out[(i, r)]["B"], B), (case_name(cases[i]), r)
        else:
            C = np.full_like(Cref, np.nan)
            for r in range(world):
                res = out[(i, r)]
                if res["layer"]:
                    continue
                (r0, rc), (c0, cc) = res["rows"], res["cols"]
                C[r0:r0 + rc, c0:c0 + cc] = res["C"]
            assert np.array_equal(C, Cref), case_name(cases[i])


def case_name(c):
    return f"layout={c[0]} {c[1]} {c[2]}x{c[3]}x{c[4]} flags={c[5]} root={c[6]} grid={c[7]}"


@pytest.fixture(scope="module")
def mmod(cuda_device):
    assert os.path.exists(FAKE), "tests/libfakenccl.so missing: run make"
    import paper_2408_15384_b200 as mm
    return mm


@pytest.mark.parametrize("world", [2, 3, 4])
def test_row_block_real_executor(mmod, world):
    mm = mmod
    flags_all = [0, mm.MM_BCAST_B, mm.MM_GATHER_C, mm.MM_BCAST_B | mm.MM_GATHER_C, mm.MM_GATHER_C_FUSED,
                 mm.MM_BCAST_B | mm.MM_GATHER_C_FUSED]
    cases = []
    for j, flags in enumerate(flags_all):
        kind = ("bf16", "i8", "f64")[j % 3]
        cases.append((mm.MM_ROW_BLOCK, kind, 600 + 37 * world, 512, 776, flags, (j + 1) % world, (0, 0),
                      "1" if j == 0 else None))
    # the emulated FP64 product through the same executor (B broadcast + fused gather)
    cases.append((mm.MM_ROW_BLOCK, "emu", 520 + 11 * world, 700, 333, mm.MM_BCAST_B | mm.MM_GATHER_C_FUSED,
                  world - 1, (0, 0), None))
    cases.append((mm.MM_ROW_BLOCK, "f64", 64, 32, 48, 0, 0, (0, 0), "mismatch"))
    _check(world, cases, _run(world, cases))


@pytest.mark.parametrize("world,grids", [(2, [(1, 2), (2, 1)]), (4, [(2, 2), (1, 4)])])
def test_summa_real_executor(mmod, world, grids):
    mm = mmod
    cases = [(mm.MM_SUMMA_2D, "f64", 331, 357 + 16 * world, 313, 0, 0, g, None) for g in grids]
    cases.append((mm.MM_SUMMA_2D, "emu", 301, 389, 277, 0, 0, grids[0], None))  # k-panels accumulate (β = 1)
    if world == 4:
        cases.append((mm.MM_SUMMA_25D, "f64", 297, 450, 283, mm.MM_REPLICATE, 0, (1, 2), None))
        cases.append((mm.MM_SUMMA_25D, "f64", 297, 450, 283, mm.MM_REPLICATE, 0, (2, 1), None))
        cases.append((mm.MM_SUMMA_25D, "emu", 297, 450, 283, mm.MM_REPLICATE, 0, (1, 2), None))
    if world == 2:
        cases.append((mm.MM_SUMMA_25D, "f64", 297, 450, 283, mm.MM_REPLICATE, 0, (1, 1), None))
    _check(world, cases, _run(world, cases))


def _full_worker(rank, world, shm, q):
    """configs[3] (BF16 16384^3, exact K=3) row-block in the two gather modes and configs[4] (FP64
    32768^3, exact K=2049) SUMMA 1x2 at G = 2 through the real executor: checksums of the assembled
    outputs vs SURVEY c7's goldens (offsets beyond 2^32 bytes: C5's blocks are 4 GiB)."""
    import json
    os.environ["MM_NCCL_LIB"] = FAKE
    import paper_2408_15384_b200 as mm
    from synthgen import gpu as sgg
    torch.cuda.set_device(0)
    fake = ctypes.CDLL(FAKE)
    fake.fake_comm_init.restype = ctypes.c_void_p
    fake.fake_comm_init.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
    comm = fake.fake_comm_init(rank, world, shm.encode())
    lib = mm._lib.load()
    ctx = mm.context(0)
    stream = torch.cuda.current_stream().cuda_stream
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_fullsize.json")))
    res = {}
    try:
        N = 16384
        s, c = mm.shard_range(N, world, rank)
        A = sgg.exact_bf16(3, sg.ROLE_A, 3, N, N)[s:s + c].contiguous()
        B = sgg.exact_bf16(3, sg.ROLE_B, 3, N, N)
        for flags in (mm.MM_BCAST_B | mm.MM_GATHER_C, mm.MM_BCAST_B | mm.MM_GATHER_C_FUSED):
            Bd = B.clone() if rank == 0 else torch.zeros_like(B)
            Cl = torch.empty(c, N, dtype=torch.float32, device="cuda")
            Cf = torch.empty(N, N, dtype=torch.float32, device="cuda") if rank == 0 else None
            fused = bool(flags & mm.MM_GATHER_C_FUSED)
            ctx.check(lib.mm_gemm_sharded(ctx.handle, N, N, N, 1, mm.MM_ROW_BLOCK, 0, 0, A.data_ptr(), Bd.data_ptr(),
                                          None if fused else Cl.data_ptr(), Cf.data_ptr() if Cf is not None else None,
                                          flags, 0, comm, stream))
            mm.sync_check()
            if rank == 0:
                res[f"C4x3 flags={flags}"] = sg.checksum(Cf.cpu().numpy()) == int(gold["C4x3"]["checksum"], 16)
            del Bd, Cl, Cf
        del A, B
        torch.cuda.empty_cache()
        N = 32768
        A5 = sgg.exact_f64(4, sg.ROLE_A, 2049, N, N)
        B5 = sgg.exact_f64(4, sg.ROLE_B, 2049, N, N)
        bn = mm.shard_range(N, 2, rank)  # grid 1x2: A column block, B column block
        Ab = A5[:, bn[0]:bn[0] + bn[1]].contiguous()
        Bb = B5[:, bn[0]:bn[0] + bn[1]].contiguous()
        del A5, B5
        torch.cuda.empty_cache()
        Cb = torch.empty(N, bn[1], dtype=torch.float64, device="cuda")
        ctx.check(lib.mm_gemm_sharded(ctx.handle, N, N, N, 0, mm.MM_SUMMA_2D, 1, 2, Ab.data_ptr(), Bb.data_ptr(),
                                      Cb.data_ptr(), None, 0, 0, comm, stream))
        mm.sync_check()
        Ch = Cb.cpu().numpy()
        cs = 0
        for i in range(N):
            cs = (cs + sg.checksum_block(np.ascontiguousarray(Ch[i]), i * N + bn[0], "f64")) % (1 << 64)
        res["C5x part"] = cs
        q.put((rank, res))
    except Exception as e:  # noqa: BLE001
        q.put((rank, {"exc": f"{type(e).__name__}: {e}"}))
        raise


def test_full_size_g2_real_executor(mmod):
    import json
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    shm = f"/mm_fake_nccl_{uuid.uuid4().hex[:12]}"
    procs = [ctx.Process(target=_full_worker, args=(r, 2, shm, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    try:
        res = dict(q.get(timeout=1500) for _ in range(2))
    finally:
        for pr in procs:
            pr.join(timeout=300)
        try:
            os.unlink("/dev/shm" + shm)
        except OSError:
            pass
    for r in (0, 1):
        assert "exc" not in res[r], res[r]
    for k, v in res[0].items():
        if k.startswith("C4x3"):
            assert v, k
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_fullsize.json")))
    assert (res[0]["C5x part"] + res[1]["C5x part"]) % (1 << 64) == int(gold["C5x"]["checksum"], 16)
