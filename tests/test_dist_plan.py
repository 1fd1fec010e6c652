"""The library's own sharded plans, executed over gloo at world sizes 2, 3, 4 and 8 on CPU.

mm_gemm_sharded runs a per-rank plan that mm_shard_plan computes (include/mm.h).  Here every rank
asks the library for its plan and runs it with tests/plan_exec.py (gloo collectives, the CPU oracle
as the local product).  The assembled C must equal the single-process oracle product bit for bit
(exact-integer inputs, so any summation order is exact): that pins the library's shard offsets,
panel pitches, broadcast roots, sub-communicator colours/keys, gather order, 2.5D layer reduction
and the fused gather's peer offsets at world sizes the one-GPU box cannot run (PAPER.md:119 row
partition; PAPER.md:135 SUMMA / 2.5D; SPEC.md:210 ⌈m/G⌉ rule and G-invariance).  Every plan is also
checked for stream races (plan_exec.check_stream_order)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import oracle
import paper_2408_15384_b200 as mm
import synthgen as sg
import plan_exec as px  # tests/plan_exec.py (pytest puts tests/ on sys.path)

TORCH = {"f64": torch.float64, "bf16": torch.bfloat16, "i8": torch.int8}
KEXACT = {"f64": 2049, "bf16": 9, "i8": 255}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(kind, m, n, p, seed=41):
    gen = {"f64": sg.exact_f64, "bf16": sg.exact_bf16, "i8": sg.exact_i8}[kind]
    return gen(seed, 1, KEXACT[kind], m, n), gen(seed, 2, KEXACT[kind], n, p)


def _full_product(kind, A, B):
    return px._local_product(kind, A, B)


def _bytes(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a).reshape(-1).view(np.uint8).copy()


def _run_case(rank, world, case):
    layout, kind, m, n, p, flags, root, grid, panel = case
    A, B = _inputs(kind, m, n, p)
    eo = np.dtype(px.OUT_NP[kind]).itemsize

    def plan_of(r):
        return mm.shard_plan(m, n, p, TORCH[kind], layout=layout, grid=grid, flags=flags, root=root, world=world,
                             rank=r, panel=panel)
    groups = px.comm_groups(plan_of, world)
    steps, info = plan_of(rank)
    px.check_stream_order(steps, kind)
    if layout == mm.MM_ROW_BLOCK:
        s, c = mm.shard_range(m, world, rank)
        have_b = rank == root or not (flags & mm.MM_BCAST_B)
        bufs = {"A": _bytes(A[s:s + c]), "B": _bytes(B if have_b else np.zeros_like(B)),
                "C": np.zeros(c * p * eo, np.uint8)}
        if rank == root:
            bufs["CFULL"] = np.zeros(m * p * eo, np.uint8)
        out = px.execute(steps, info, kind, bufs, groups, m * p * eo)
        res = {"C": out["C"].view(px.OUT_NP[kind]).reshape(c, p).copy(), "rows": (s, c),
               "B": out["B"].view(px.IN_NP[kind]).reshape(n, p).copy()}
        if rank == root:
            res["CFULL"] = out["CFULL"].view(px.OUT_NP[kind]).reshape(m, p).copy()
        return res
    pr, pc = grid
    layers = world // (pr * pc)
    l, r2 = rank // (pr * pc), rank % (pr * pc)
    gi, gj = r2 // pc, r2 % pc
    am, ak = mm.shard_range(m, pr, gi), mm.shard_range(n, pc, gj)
    bk, bn = mm.shard_range(n, pr, gi), mm.shard_range(p, pc, gj)
    Ab = A[am[0]:am[0] + am[1], ak[0]:ak[0] + ak[1]]
    Bb = B[bk[0]:bk[0] + bk[1], bn[0]:bn[0] + bn[1]]
    if layers > 1 and (flags & mm.MM_REPLICATE) and l > 0:
        Ab, Bb = np.zeros_like(Ab), np.zeros_like(Bb)  # only layer 0 holds the blocks
    bufs = {"A": _bytes(Ab), "B": _bytes(Bb), "C": np.full(am[1] * bn[1] * eo, 0x5A, np.uint8)}
    out = px.execute(steps, info, kind, bufs, groups, 0)
    return {"C": out["C"].view(px.OUT_NP[kind]).reshape(am[1], bn[1]).copy(), "layer": l, "gi": gi, "gj": gj,
            "rows": am, "cols": bn}


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for i, case in enumerate(cases):
            try:
                q.put((i, rank, _run_case(rank, world, case)))
            except Exception as e:  # noqa: BLE001 — report, keep the collective schedule aligned
                q.put((i, rank, {"error": f"{type(e).__name__}: {e}"}))
                raise
    finally:
        dist.destroy_process_group()


def _spawn(world, cases):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = {}
    try:
        for _ in range(world * len(cases)):
            i, r, res = q.get(timeout=600)
            assert "error" not in res, (cases[i], r, res["error"])
            results[(i, r)] = res
    finally:
        for pr in procs:
            pr.join(timeout=120)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    return results


def _check(world, cases, results):
    for i, case in enumerate(cases):
        layout, kind, m, n, p, flags, root, grid, panel = case
        A, B = _inputs(kind, m, n, p)
        Cref = _full_product(kind, A, B)
        if layout == mm.MM_ROW_BLOCK:
            gathered = bool(flags & (mm.MM_GATHER_C | mm.MM_GATHER_C_FUSED))
            if gathered:
                assert np.array_equal(results[(i, root)]["CFULL"], Cref), case
            if not (flags & mm.MM_GATHER_C_FUSED):
                for r in range(world):
                    s, c = results[(i, r)]["rows"]
                    assert np.array_equal(results[(i, r)]["C"], Cref[s:s + c]), (case, r)
            if flags & mm.MM_BCAST_B:
                for r in range(world):
                    assert np.array_equal(results[(i, r)]["B"], B), (case, r)  # B_local holds B afterwards
        else:
            C = np.zeros_like(Cref)
            seen = np.zeros(Cref.shape, bool)
            for r in range(world):
                res = results[(i, r)]
                if res["layer"] != 0:
                    continue
                (r0, rc), (c0, cc) = res["rows"], res["cols"]
                C[r0:r0 + rc, c0:c0 + cc] = res["C"]
                seen[r0:r0 + rc, c0:c0 + cc] = True
            assert seen.all(), case
            assert np.array_equal(C, Cref), case


ROW_FLAGS = [0, mm.MM_BCAST_B, mm.MM_GATHER_C, mm.MM_BCAST_B | mm.MM_GATHER_C, mm.MM_GATHER_C_FUSED,
             mm.MM_BCAST_B | mm.MM_GATHER_C_FUSED]


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_row_block_plans(world):
    """C4's layout (row blocks of A and C, B broadcast, C gathered or fused-gathered) at G = 2..8,
    ragged row counts (m not a multiple of G; G = 8 with m < 8·⌈m/8⌉ leaves a short last block)."""
    cases = []
    for j, flags in enumerate(ROW_FLAGS):
        kind = ("bf16", "i8", "f64")[j % 3]
        root = (j + 1) % world
        cases.append((mm.MM_ROW_BLOCK, kind, 203 + 7 * world, 96, 176, flags, root, (0, 0), 64 if j % 2 else 0))
    results = _spawn(world, cases)
    _check(world, cases, results)


def test_row_block_more_ranks_than_rows():
    """G = 8 ranks over m = 5 rows: surplus ranks own empty blocks."""
    cases = [(mm.MM_ROW_BLOCK, "f64", 5, 40, 48, mm.MM_BCAST_B | mm.MM_GATHER_C, 0, (0, 0), 16),
             (mm.MM_ROW_BLOCK, "i8", 5, 64, 48, mm.MM_GATHER_C_FUSED, 7, (0, 0), 0)]
    results = _spawn(8, cases)
    _check(8, cases, results)


@pytest.mark.parametrize("world,grid", [(2, (1, 2)), (2, (2, 1)), (4, (2, 2)), (8, (2, 4)), (8, (4, 2))])
def test_summa_plans(world, grid):
    """C5's layout: SUMMA over the grids of BASELINE configs[4] (1x2, 2x2, 2x4), ragged blocks,
    k-panels narrower than a block (several panels per owner) and wider (one per block)."""
    cases = [(mm.MM_SUMMA_2D, "f64", 131, 157, 113, 0, 0, grid, 24),
             (mm.MM_SUMMA_2D, "f64", 64, 200, 72, 0, 0, grid, 0)]
    results = _spawn(world, cases)
    _check(world, cases, results)


@pytest.mark.parametrize("world,grid", [(8, (2, 2)), (4, (1, 2)), (4, (2, 1))])
def test_summa25d_plans(world, grid):
    """2.5D: c = world / (pr·pc) layers, blocks replicated from layer 0, panels
    t ≡ l (mod c) per layer, layer C blocks reduced onto layer 0 — 2x2x2 is the 8-GPU layout."""
    cases = [(mm.MM_SUMMA_25D, "f64", 97, 150, 83, mm.MM_REPLICATE, 0, grid, 16)]
    results = _spawn(world, cases)
    _check(world, cases, results)


def test_plan_race_free_and_shapes():
    """Every plan of a grid of arguments is race-free on its two streams, its products cover C
    exactly once per k-panel, and staging sizes fit the panels (no process group needed)."""
    for world in (1, 2, 3, 8):
        for r in range(world):
            for flags in ROW_FLAGS:
                for kind in ("bf16", "f64"):
                    steps, info = mm.shard_plan(1000, 300, 777, TORCH[kind], flags=flags, root=world - 1, world=world,
                                                rank=r)
                    px.check_stream_order(steps, kind)
                    s, c = mm.shard_range(1000, world, r)
                    cols = sum(st["p"] for st in steps if st["op"] == "GEMM")
                    assert cols == (777 if c else 0), (world, r, flags)
                    for st in steps:
                        if st["op"] == "GEMM" and st["src2"].startswith("S"):
                            eb = np.dtype(px.IN_NP[kind]).itemsize
                            assert st["n"] * st["p"] * eb <= info["stage_bytes"][int(st["src2"][1])]
    for world, grid, layout, flags in ((4, (2, 2), mm.MM_SUMMA_2D, 0), (8, (2, 4), mm.MM_SUMMA_2D, 0),
                                       (8, (2, 2), mm.MM_SUMMA_25D, mm.MM_REPLICATE)):
        for r in range(world):
            steps, info = mm.shard_plan(5000, 4100, 3000, torch.float64, layout=layout, grid=grid, flags=flags,
                                        world=world, rank=r, panel=512)
            px.check_stream_order(steps, "f64")
            ks = sum(st["n"] for st in steps if st["op"] == "GEMM")
            layers = world // (grid[0] * grid[1])
            l = r // (grid[0] * grid[1])
            panels = mm.summa_panels(4100, grid[0], grid[1], 512)
            assert ks == sum(kw for t, (_, kw, _, _) in enumerate(panels) if t % layers == l)


def test_emulated_fp64_plans_equal_fp64_plans():
    """MM_F64_EMU shards like MM_F64 (same element sizes, same β = 1 panel accumulation): for every
    layout, rank and flag set the plans with the same panel width are step-for-step identical, so
    the gloo executions of the FP64 plans above cover the emulated ones; by default the emulation
    takes wider panels (its per-product fixed costs); the workspace bound adds its scratch."""
    cases = [(mm.MM_ROW_BLOCK, (0, 0), f, w) for f in ROW_FLAGS for w in (1, 2, 3, 8)]
    cases += [(mm.MM_SUMMA_2D, g, 0, g[0] * g[1]) for g in ((1, 2), (2, 2), (2, 4))]
    cases += [(mm.MM_SUMMA_25D, (2, 2), mm.MM_REPLICATE, 8), (mm.MM_SUMMA_25D, (1, 2), mm.MM_REPLICATE, 4)]
    for layout, grid, flags, world in cases:
        for r in range(world):
            a = mm.shard_plan(1000, 3000, 777, torch.float64, layout=layout, grid=grid, flags=flags, world=world,
                              rank=r, panel=256)
            b = mm.shard_plan(1000, 3000, 777, torch.float64, layout=layout, grid=grid, flags=flags, world=world,
                              rank=r, f64_emulation=True, panel=256)
            assert a == b, (layout, grid, flags, world, r)
            gemms = [sum(st["op"] == "GEMM" for st in mm.shard_plan(20000, 30000, 7770, torch.float64, layout=layout,
                                                                     grid=grid, flags=flags, world=world, rank=r,
                                                                     f64_emulation=e)[0]) for e in (False, True)]
            assert gemms[1] <= gemms[0], (layout, grid, flags, world, r, gemms)
        for lay in (layout,):
            plain = mm.workspace_size(1000, 3000, 777, torch.float64, lay, world)
            emu = mm.workspace_size(1000, 3000, 777, torch.float64, lay, world, f64_emulation=True)
            assert emu > plain > 0, (lay, world)
    with pytest.raises(ValueError):
        mm.shard_plan(10, 10, 10, torch.bfloat16, f64_emulation=True)


def test_plan_usage_errors():
    with pytest.raises(mm.MMError):
        mm.shard_plan(10, 10, 10, torch.float64, flags=mm.MM_GATHER_C | mm.MM_GATHER_C_FUSED, world=2)
    with pytest.raises(mm.MMError):
        mm.shard_plan(10, 10, 10, torch.float64, root=2, world=2)
    with pytest.raises(mm.MMError):
        mm.shard_plan(10, 10, 10, torch.float64, layout=mm.MM_SUMMA_2D, grid=(2, 2), world=2)
    with pytest.raises(mm.MMError):
        mm.shard_plan(10, 10, 10, torch.bfloat16, layout=mm.MM_SUMMA_2D, grid=(1, 2), world=2)
    with pytest.raises(mm.MMError):
        mm.shard_plan(0, 10, 10, torch.float64, world=1)
    with pytest.raises(mm.MMError):
        mm.shard_plan(10, 10, 10, torch.float64, world=2, rank=2)
