"""Kernel timing sweep (CUDA events, L2 flushed between reps) with cuBLAS beside it.
    python tools/timeit_gpu.py [--reps 10] [--only bf16,i8,f64]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402

FLUSH = None


def flush():
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    FLUSH.zero_()


def bench(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2], ts[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="bf16,i8,f64")
    ap.add_argument("--cg", default="1,2")
    args = ap.parse_args()
    only = args.only.split(",")
    cases = []
    if "bf16" in only:
        cases += [("bf16", 16384, 16384, 16384), ("bf16", 8192, 8192, 8192), ("bf16", 4096, 4096, 4096)]
    if "i8" in only:
        cases += [("i8", 4096, 4096, 4096), ("i8", 8192, 8192, 8192)]
    if "f64" in only:
        cases += [("f64", 256, 256, 256), ("f64", 2000, 1500, 1750), ("f64", 8192, 8192, 8192)]
    for dt, m, n, p in cases:
        if dt == "bf16":
            A = torch.randn(m, n, device="cuda").to(torch.bfloat16)
            B = torch.randn(n, p, device="cuda").to(torch.bfloat16)
            ref = lambda: torch.matmul(A, B)  # noqa: E731
        elif dt == "i8":
            A = torch.randint(-127, 128, (m, n), device="cuda", dtype=torch.int8)
            B = torch.randint(-127, 128, (n, p), device="cuda", dtype=torch.int8)
            ref = lambda: torch._int_mm(A, B)  # noqa: E731
        else:
            A = torch.rand(m, n, device="cuda", dtype=torch.float64)
            B = torch.rand(n, p, device="cuda", dtype=torch.float64)
            ref = lambda: torch.matmul(A, B)  # noqa: E731
        C = torch.empty(m, p, device="cuda", dtype=mm.OUT_DTYPE[mm.IN_DTYPE[A.dtype]])
        flops = 2.0 * m * n * p
        cgs = [int(c) for c in args.cg.split(",")] if dt != "f64" else [0]
        for cg in cgs:
            if cg:
                os.environ["MM_FORCE_CG"] = str(cg)
            med, best = bench(lambda: mm.gemm(A, B, out=C), args.reps)
            mm.sync_check()
            print(f"{dt:5s} {m}x{n}x{p} cg{cg}: median {med*1e3:9.1f} us  {flops/med/1e9:8.1f} TFLOPS "
                  f"(best {flops/best/1e9:8.1f})", flush=True)
        os.environ.pop("MM_FORCE_CG", None)
        try:
            med, best = bench(ref, args.reps)
            print(f"{dt:5s} {m}x{n}x{p} torch : median {med*1e3:9.1f} us  {flops/med/1e9:8.1f} TFLOPS "
                  f"(best {flops/best/1e9:8.1f})", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{dt} torch ref failed: {e}")
        del A, B, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
