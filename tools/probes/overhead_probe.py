"""Host overhead and launch-mode probe (B200):
  * host microseconds per mm.gemm call (python binding) and per raw mm_gemm (ctypes), GPU kept busy
  * per-launch device time of a shape measured three ways: back-to-back (K launches between two
    events), single launch on an idle GPU (what the protocol's per-launch events see: includes
    the host call), single launch after an L2 flush (host call hidden behind the flush)
  * the same for cuBLAS (torch.matmul / torch._int_mm)
    python tools/overhead_probe.py [--cases bf16:4096,i8:4096,f64:256,...]
"""
import argparse
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402
from paper_2408_15384_b200 import _lib  # noqa: E402

DT = {"f64": (torch.float64, torch.float64), "bf16": (torch.bfloat16, torch.float32), "i8": (torch.int8, torch.int32)}


def make(dt, m, n, p):
    tin, tout = DT[dt]
    if dt == "i8":
        A = torch.randint(-127, 128, (m, n), dtype=torch.int8, device="cuda")
        B = torch.randint(-127, 128, (n, p), dtype=torch.int8, device="cuda")
    else:
        A = torch.randn(m, n, device="cuda").to(tin)
        B = torch.randn(n, p, device="cuda").to(tin)
    C = torch.empty(m, p, dtype=tout, device="cuda")
    return A, B, C


def b2b(fn, k):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / k


def single(fn, reps, flush=None):
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        else:
            torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def host_us(fn, k):
    # keep the GPU busy so launches never block, time the host side only
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / k * 1e6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="bf16:128,bf16:4096,bf16:8192,i8:4096,f64:256,f64:2000x1500x1750")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    lib = _lib.load()
    for case in args.cases.split(","):
        dt, shp = case.split(":")
        dims = [int(x) for x in shp.split("x")]
        m, n, p = dims if len(dims) == 3 else dims * 3
        A, B, C = make(dt, m, n, p)
        ctx = mm.context()
        s = torch.cuda.current_stream().cuda_stream
        code = {"f64": 0, "bf16": 1, "i8": 2}[dt]
        ap_, bp_, cp_ = A.data_ptr(), B.data_ptr(), C.data_ptr()
        ours = lambda: mm.gemm(A, B, out=C)  # noqa: E731
        raw = lambda: lib.mm_gemm(ctx.handle, m, n, p, code, ap_, bp_, cp_, s)  # noqa: E731
        ref = (lambda: torch._int_mm(A, B)) if dt == "i8" else (lambda: torch.matmul(A, B))  # noqa: E731
        flops = 2.0 * m * n * p
        row = {"case": case}
        row["host_us_py"] = round(host_us(ours, 200), 2)
        row["host_us_raw"] = round(host_us(raw, 200), 2)
        row["host_us_cublas"] = round(host_us(ref, 200), 2)
        for name, fn in (("ours", ours), ("cublas", ref)):
            t_b2b = b2b(fn, max(5, min(200, int(2e-3 / max(flops / 1.2e15, 1e-7)))))
            t_idle = single(fn, args.reps)
            t_fl = single(fn, args.reps, flush)
            row[name] = {"b2b_us": round(t_b2b * 1e3, 2), "idle_us": round(t_idle * 1e3, 2),
                         "flushed_us": round(t_fl * 1e3, 2), "tflops_b2b": round(flops / t_b2b / 1e9, 1)}
        mm.sync_check()
        print(row, flush=True)


if __name__ == "__main__":
    main()
