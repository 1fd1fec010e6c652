"""Raster/group sweep for the BF16 C4 kernel: sustained throughput with clocks.
    python tools/sweep_raster.py [--secs 2] [--groups 4,8,16,32]
"""
import argparse
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402
from bench import ClockSampler  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--secs", type=float, default=2.0)
    ap.add_argument("--groups", default="4,8,16,32")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--dtype", default="bf16")
    args = ap.parse_args()
    N = args.n
    if args.dtype == "bf16":
        A = torch.randn(N, N, device="cuda").to(torch.bfloat16)
        B = torch.randn(N, N, device="cuda").to(torch.bfloat16)
        C = torch.empty(N, N, device="cuda", dtype=torch.float32)
    else:
        A = torch.randint(-127, 128, (N, N), device="cuda", dtype=torch.int8)
        B = torch.randint(-127, 128, (N, N), device="cuda", dtype=torch.int8)
        C = torch.empty(N, N, device="cuda", dtype=torch.int32)
    flops = 2.0 * N ** 3
    for g in args.groups.split(","):
        os.environ["MM_GROUP_M"] = g
        for _ in range(3):
            mm.gemm(A, B, out=C)
        torch.cuda.synchronize()
        time.sleep(1.0)  # cool down a little
        # burst: 5 launches
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5):
            mm.gemm(A, B, out=C)
        e1.record()
        e1.synchronize()
        burst = flops * 5 / (e0.elapsed_time(e1) * 1e-3) / 1e12
        # sustained for args.secs
        one = e0.elapsed_time(e1) / 5
        iters = max(5, int(args.secs * 1e3 / one))
        clk = ClockSampler(0)
        clk.start()
        time.sleep(0.1)
        e0.record()
        for _ in range(iters):
            mm.gemm(A, B, out=C)
        e1.record()
        e1.synchronize()
        c = clk.stop()
        sus = flops * iters / (e0.elapsed_time(e1) * 1e-3) / 1e12
        print(f"{args.dtype} N={N} group_m={g:>3}: burst {burst:7.1f} TF  sustained {sus:7.1f} TF  clocks {c}",
              flush=True)
    mm.sync_check()
    # cuBLAS reference, same protocol
    if args.dtype == "bf16":
        for _ in range(3):
            torch.matmul(A, B)
        torch.cuda.synchronize()
        time.sleep(1.0)
        iters = max(5, int(args.secs * 1e3 / one))
        clk = ClockSampler(0)
        clk.start()
        time.sleep(0.1)
        e0.record()
        for _ in range(iters):
            torch.matmul(A, B)
        e1.record()
        e1.synchronize()
        c = clk.stop()
        print(f"cuBLAS sustained {flops * iters / (e0.elapsed_time(e1) * 1e-3) / 1e12:7.1f} TF clocks {c}", flush=True)


if __name__ == "__main__":
    main()
