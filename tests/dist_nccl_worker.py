"""torchrun worker for tests/test_dist_nccl.py: mm_gemm_sharded over NCCL, one process per GPU.

    torchrun --nproc-per-node G --master-addr 127.0.0.1 tests/dist_nccl_worker.py [--full]

Every rank runs the same list of collective products (include/mm.h) and checks its part; rank 0
prints one JSON line {"ok": bool, "checks": [...]} at the end.  Checks (PAPER.md:119 row
partition, PAPER.md:135 SUMMA / 2.5D; BASELINE.json configs[3] at G = 1/2/4/8, configs[4] over the
1x2 / 2x2 / 2x4 grids):
  * row-block products of ragged exact-integer shapes with every flag combination
    (resident, MM_BCAST_B, MM_GATHER_C, both, MM_GATHER_C_FUSED, MM_BCAST_B | MM_GATHER_C_FUSED, the same with
    MM_C_WINDOW: NCCL symmetric memory instead of a CUDA-IPC mapping),
    every dtype: C_local per rank, C_full on the root and B_local afterwards, bit-exact vs the oracle;
  * SUMMA over every grid G factors into, and 2.5D over every (grid, layers) — FP64, exact;
  * --full: configs[3] (BF16 16384^3) on exact-integer inputs K=3 in the three gather modes: the
    checksum of the gathered C equals SURVEY c7's C4x golden; random inputs: >= 64 seeded rows and
    >= 64 seeded columns of the gathered C against the oracle at the BF16 tolerance; configs[4]
    (FP64 32768^3) exact K=2049 over the SUMMA grids and 2.5D: the checksum of the assembled blocks
    equals C5x's golden.
Test infrastructure: calls oracle/.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2408_15384_b200 as mm  # noqa: E402
import synthgen as sg  # noqa: E402
from synthgen import gpu as sgg  # noqa: E402

TORCH_IN = {"f64": torch.float64, "bf16": torch.bfloat16, "i8": torch.int8}
TORCH_OUT = {"f64": torch.float64, "bf16": torch.float32, "i8": torch.int32}
KEXACT = {"f64": 2049, "bf16": 9, "i8": 255}
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_fullsize.json")))


def exact_host(dt, seed, K, rows, cols, role):
    return {"f64": sg.exact_f64, "bf16": sg.exact_bf16, "i8": sg.exact_i8}[dt](seed, role, K, rows, cols)


def to_dev(x, dt):
    if dt == "bf16":
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def oracle_full(dt, A, B):
    if dt == "f64":
        return oracle.gemm_f64(A, B)
    if dt == "bf16":
        return oracle.gemm_bf16(A, B)[0]
    return oracle.gemm_s8(A, B)


def allreduce_ok(ok: bool) -> bool:
    t = torch.tensor([0 if ok else 1], dtype=torch.int32, device="cuda")
    dist.all_reduce(t)
    return int(t.item()) == 0


def block_checksum(C: np.ndarray, r0: int, c0: int, p: int, kind: str) -> int:
    cs = 0
    for i in range(C.shape[0]):
        cs = (cs + sg.checksum_block(np.ascontiguousarray(C[i]), (r0 + i) * p + c0, kind)) % (1 << 64)
    return cs


def row_block_small(G, r, checks):
    flags_list = [0, mm.MM_BCAST_B, mm.MM_GATHER_C, mm.MM_BCAST_B | mm.MM_GATHER_C, mm.MM_GATHER_C_FUSED,
                  mm.MM_BCAST_B | mm.MM_GATHER_C_FUSED, mm.MM_BCAST_B | mm.MM_GATHER_C_FUSED | mm.MM_C_WINDOW]
    for dt in ("bf16", "i8", "f64"):
        m, n, p = 1000 + 13 * G, 768, 1100
        A = exact_host(dt, 61, KEXACT[dt], m, n, 1)
        B = exact_host(dt, 61, KEXACT[dt], n, p, 2)
        Cref = np.asarray(oracle_full(dt, A, B), np.float64)
        s, c = mm.shard_range(m, G, r)
        for j, flags in enumerate(flags_list):
            root = j % G
            Ad = to_dev(A[s:s + c], dt)
            Bd = to_dev(B, dt) if (r == root or not flags & mm.MM_BCAST_B) else torch.zeros(n, p, dtype=TORCH_IN[dt],
                                                                                          device="cuda")
            Cl = torch.full((c, p), -9, dtype=TORCH_OUT[dt], device="cuda")
            win = None
            if flags & mm.MM_C_WINDOW:  # NCCL symmetric memory on every rank, C_full at the same offset
                win = mm.window_alloc((m + 2, p), TORCH_OUT[dt])
                win.fill_(-9)
                Cf = win[1:1 + m]
            else:
                Cf = torch.full((m, p), -9, dtype=TORCH_OUT[dt], device="cuda") if r == root else None
            fused = bool(flags & mm.MM_GATHER_C_FUSED)
            mm.gemm_sharded(m, n, p, TORCH_IN[dt], Ad, Bd, None if fused else Cl, layout=mm.MM_ROW_BLOCK,
                            flags=flags, root=root, C_full=Cf)
            mm.sync_check()
            torch.cuda.synchronize()
            dist.barrier()
            ok = True
            if not fused:
                ok &= np.array_equal(Cl.cpu().numpy().astype(np.float64), Cref[s:s + c])
            if (flags & (mm.MM_GATHER_C | mm.MM_GATHER_C_FUSED)) and r == root:
                ok &= np.array_equal(Cf.cpu().numpy().astype(np.float64), Cref)
            if flags & mm.MM_BCAST_B:
                ok &= torch.equal(Bd.cpu(), to_dev(B, dt).cpu())
            if win is not None:
                ok &= bool((win[0] == -9).all() and (win[m + 1] == -9).all())
                if r != root:  # peers stored into the root's window only
                    ok &= bool((Cf == -9).all())
                dist.barrier()
                mm.window_free(win)
            checks.append({"what": f"row-block {dt} {m}x{n}x{p} flags={flags} root={root}", "ok": allreduce_ok(ok)})


def collective_check(G, r, checks):
    """MM_CHECK_COLLECTIVE=1: matching arguments pass; a rank-dependent m is MM_ERR_USAGE on every rank."""
    os.environ["MM_CHECK_COLLECTIVE"] = "1"
    try:
        m, n, p = 64 + (r if G > 1 else 0), 32, 48
        A = torch.ones(m, n, dtype=torch.float64, device="cuda")
        B = torch.ones(n, p, dtype=torch.float64, device="cuda")
        C = torch.empty(m, p, dtype=torch.float64, device="cuda")
        raised = False
        try:
            mm.gemm_sharded(m, n, p, torch.float64, A, B, C, layout=mm.MM_ROW_BLOCK)
            mm.sync_check()
        except mm.MMError as e:
            raised = "differ across" in str(e)
        checks.append({"what": f"collective argument check (mismatch expected: {G > 1})",
                       "ok": allreduce_ok(raised == (G > 1))})
    finally:
        os.environ.pop("MM_CHECK_COLLECTIVE", None)


def grids_of(G):
    return [(pr, G // pr) for pr in range(1, G + 1) if G % pr == 0]


def summa_small(G, r, checks):
    m, n, p = 700, 1000 + 16 * G, 900
    A = exact_host("f64", 62, 2049, m, n, 1)
    B = exact_host("f64", 62, 2049, n, p, 2)
    Cref = oracle.gemm_f64(A, B)
    cases = [(mm.MM_SUMMA_2D, g, 0) for g in grids_of(G)]
    for layers in (2, 4, 8):
        if G % layers == 0 and layers > 1:
            cases += [(mm.MM_SUMMA_25D, g, mm.MM_REPLICATE) for g in grids_of(G // layers)]
    # the same layouts with every local product emulated on the INT8 tensor cores (MM_F64_EMU)
    cases += [(layout, g, flags, True) for layout, g, flags in cases[:2]]
    for layout, (pr, pc), flags, *emu in cases:
        emu = bool(emu)
        g2 = pr * pc
        l, r2 = r // g2, r % g2
        gi, gj = r2 // pc, r2 % pc
        am, ak = mm.shard_range(m, pr, gi), mm.shard_range(n, pc, gj)
        bk, bn = mm.shard_range(n, pr, gi), mm.shard_range(p, pc, gj)
        Ab = A[am[0]:am[0] + am[1], ak[0]:ak[0] + ak[1]]
        Bb = B[bk[0]:bk[0] + bk[1], bn[0]:bn[0] + bn[1]]
        if layout == mm.MM_SUMMA_25D and l > 0:
            Ab, Bb = np.zeros_like(Ab), np.zeros_like(Bb)
        Cb = torch.full((am[1], bn[1]), -5.0, dtype=torch.float64, device="cuda")
        os.environ["MM_SUMMA_PANEL"] = "128"
        try:
            mm.gemm_sharded(m, n, p, torch.float64, to_dev(Ab, "f64"), to_dev(Bb, "f64"), Cb, layout=layout,
                            grid=(pr, pc), flags=flags, f64_emulation=emu)
        finally:
            os.environ.pop("MM_SUMMA_PANEL", None)
        mm.sync_check()
        torch.cuda.synchronize()
        ok = True
        if l == 0:
            ok = np.array_equal(Cb.cpu().numpy(), Cref[am[0]:am[0] + am[1], bn[0]:bn[0] + bn[1]])
        checks.append({"what": f"{'SUMMA' if layout == mm.MM_SUMMA_2D else '2.5D'} {pr}x{pc}x{G // g2} "
                               f"{'f64 emulated' if emu else 'f64'} "
                               f"{m}x{n}x{p}", "ok": allreduce_ok(ok)})


def c4_full(G, r, checks):
    """configs[3] at full size, row-block over G ranks, in the three gather modes."""
    N = 16384
    s, c = mm.shard_range(N, G, r)
    A = sgg.exact_bf16(3, sg.ROLE_A, 3, N, N)[s:s + c].contiguous()
    B = sgg.exact_bf16(3, sg.ROLE_B, 3, N, N)
    gold = int(GOLD["C4x3"]["checksum"], 16) if "C4x3" in GOLD else None
    for flags in (0, mm.MM_BCAST_B | mm.MM_GATHER_C, mm.MM_BCAST_B | mm.MM_GATHER_C_FUSED):
        Bd = B.clone() if (r == 0 or not flags & mm.MM_BCAST_B) else torch.zeros_like(B)
        Cl = torch.empty(c, N, dtype=torch.float32, device="cuda")
        Cf = torch.empty(N, N, dtype=torch.float32, device="cuda") if (r == 0 and flags) else None
        mm.gemm_sharded(N, N, N, torch.bfloat16, A, Bd, None if flags & mm.MM_GATHER_C_FUSED else Cl,
                        layout=mm.MM_ROW_BLOCK, flags=flags, root=0, C_full=Cf)
        mm.sync_check()
        torch.cuda.synchronize()
        if flags == 0:
            cs = block_checksum(Cl.cpu().numpy(), s, 0, N, "f32")
            t = torch.tensor([cs & 0xFFFFFFFF, cs >> 32], dtype=torch.int64, device="cuda")
            parts = [torch.zeros_like(t) for _ in range(G)]
            dist.all_gather(parts, t)
            total = sum((int(x[0]) | (int(x[1]) << 32)) for x in parts) % (1 << 64)
            ok = gold is None or total == gold
        else:
            ok = True
            if r == 0:
                ok = gold is None or sg.checksum(Cf.cpu().numpy()) == gold
        checks.append({"what": f"C4x K=3 16384^3 G={G} flags={flags} checksum vs golden", "ok": allreduce_ok(ok)})
        del Bd, Cl, Cf
    # random values: sampled rows and columns of the gathered C against the oracle
    A_host_full = sg.normal_bf16(3, sg.ROLE_A, N, N)
    B_host = sg.normal_bf16(3, sg.ROLE_B, N, N)
    A = to_dev(A_host_full[s:s + c], "bf16")
    Bd = to_dev(B_host, "bf16")
    Cl = torch.empty(c, N, dtype=torch.float32, device="cuda")
    Cf = torch.empty(N, N, dtype=torch.float32, device="cuda") if r == 0 else None
    mm.gemm_sharded(N, N, N, torch.bfloat16, A, Bd, Cl, layout=mm.MM_ROW_BLOCK, flags=mm.MM_GATHER_C, root=0,
                    C_full=Cf)
    mm.sync_check()
    torch.cuda.synchronize()
    ok = True
    if r == 0:
        seams = sorted({x for q in range(G) for x in (mm.shard_range(N, G, q)[0] - 1, mm.shard_range(N, G, q)[0])
                        if 0 <= x < N} | {0, N - 1})
        rows = np.array(sorted(set(sg.sample_indices(3, 3, 64, N).tolist()) | set(seams)), np.int64)
        cols = np.array(sorted(set(sg.sample_indices(3, 4, 64, N).tolist()) | {0, N - 1, 8191, 8192}), np.int64)
        Cr, Dr = oracle.gemm_bf16_rows(A_host_full, B_host, rows)
        Cc, Dc = oracle.gemm_bf16_cols(A_host_full, B_host, cols)
        got_r = Cf[torch.from_numpy(rows).cuda()].cpu().numpy()
        got_c = Cf[:, torch.from_numpy(cols).cuda()].cpu().numpy()
        err = max(oracle.normalized_error(got_r, Cr, Dr), oracle.normalized_error(got_c, Cc, Dc))
        ok = err <= 2e-2
        checks.append({"what": f"C4 random G={G} {rows.size} rows + {cols.size} cols vs oracle", "err": float(err)})
    checks.append({"what": f"C4 random G={G} sampled", "ok": allreduce_ok(ok)})


def c5_full(G, r, checks):
    """configs[4] exact K=2049 over every SUMMA grid of G (and 2.5D with 2 layers when G >= 4)."""
    N = 32768
    gold = int(GOLD["C5x"]["checksum"], 16) if "C5x" in GOLD else None
    A = sgg.exact_f64(4, sg.ROLE_A, 2049, N, N)
    B = sgg.exact_f64(4, sg.ROLE_B, 2049, N, N)
    cases = [(mm.MM_SUMMA_2D, g, 0) for g in grids_of(G) if g[0] <= 2 and g[1] <= 4]
    if G >= 4:
        cases.append((mm.MM_SUMMA_25D, (2, G // 4), mm.MM_REPLICATE))
    for layout, (pr, pc), flags in cases:
        g2 = pr * pc
        l, r2 = r // g2, r % g2
        gi, gj = r2 // pc, r2 % pc
        am, ak = mm.shard_range(N, pr, gi), mm.shard_range(N, pc, gj)
        bk, bn = mm.shard_range(N, pr, gi), mm.shard_range(N, pc, gj)
        Ab = A[am[0]:am[0] + am[1], ak[0]:ak[0] + ak[1]].contiguous()
        Bb = B[bk[0]:bk[0] + bk[1], bn[0]:bn[0] + bn[1]].contiguous()
        if layout == mm.MM_SUMMA_25D and l > 0:
            Ab.zero_()
            Bb.zero_()
        Cb = torch.empty(am[1], bn[1], dtype=torch.float64, device="cuda")
        mm.gemm_sharded(N, N, N, torch.float64, Ab, Bb, Cb, layout=layout, grid=(pr, pc), flags=flags)
        mm.sync_check()
        torch.cuda.synchronize()
        cs = block_checksum(Cb.cpu().numpy(), am[0], bn[0], N, "f64") if l == 0 else 0
        t = torch.tensor([cs & 0xFFFFFFFF, cs >> 32], dtype=torch.int64, device="cuda")
        parts = [torch.zeros_like(t) for _ in range(G)]
        dist.all_gather(parts, t)
        total = sum((int(x[0]) | (int(x[1]) << 32)) for x in parts) % (1 << 64)
        checks.append({"what": f"C5x FP64 32768^3 K=2049 {'SUMMA' if flags == 0 else '2.5D'} {pr}x{pc}x{G // g2}",
                       "ok": allreduce_ok(gold is None or total == gold)})
        del Ab, Bb, Cb
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    args = ap.parse_args()
    G = int(os.environ.get("WORLD_SIZE", "1"))
    r = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    checks = []
    try:
        row_block_small(G, r, checks)
        summa_small(G, r, checks)
        collective_check(G, r, checks)
        if args.full:
            c4_full(G, r, checks)
            c5_full(G, r, checks)
    except Exception as e:  # noqa: BLE001
        checks.append({"what": "exception", "ok": False, "error": f"{type(e).__name__}: {e}"})
    ok = all(c.get("ok", True) for c in checks)
    if r == 0:
        print(json.dumps({"ok": ok, "world": G, "checks": checks}), flush=True)
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
