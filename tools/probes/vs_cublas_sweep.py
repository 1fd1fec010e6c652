"""Ours vs cuBLAS per launch (L2 flushed before each, interleaved, mean and median of N reps):
    python tools/probes/vs_cublas_sweep.py i8:4096,bf16:4096 [reps]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2408_15384_b200 as mm  # noqa: E402

cases = sys.argv[1].split(",")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for case in cases:
    dt, shp = case.split(":")
    d = [int(x) for x in shp.split("x")]
    m, n, p = d if len(d) == 3 else d * 3
    if dt == "i8":
        A = torch.randint(-127, 128, (m, n), dtype=torch.int8, device="cuda")
        B = torch.randint(-127, 128, (n, p), dtype=torch.int8, device="cuda")
        C = torch.empty(m, p, dtype=torch.int32, device="cuda")
        lib = lambda: torch._int_mm(A, B, out=C)  # noqa: E731
    elif dt == "bf16":
        A = torch.randn(m, n, device="cuda").bfloat16()
        B = torch.randn(n, p, device="cuda").bfloat16()
        C = torch.empty(m, p, dtype=torch.float32, device="cuda")
        lib = lambda: torch.mm(A, B, out_dtype=torch.float32, out=C)  # noqa: E731
    else:
        A = torch.randn(m, n, device="cuda", dtype=torch.float64)
        B = torch.randn(n, p, device="cuda", dtype=torch.float64)
        C = torch.empty(m, p, dtype=torch.float64, device="cuda")
        lib = lambda: torch.mm(A, B, out=C)  # noqa: E731
    ours = lambda: mm.gemm(A, B, out=C)  # noqa: E731
    for f in (ours, lib, ours, lib):
        f()
    torch.cuda.synchronize()
    big = (m * n + n * p) * A.element_size() > (256 << 20)
    ts = {"ours": [], "lib": []}
    for _ in range(reps):
        for k, f in (("ours", ours), ("lib", lib)):
            if not big:
                flush.zero_()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            f()
            e1.record()
            e1.synchronize()
            ts[k].append(e0.elapsed_time(e1) * 1e3)
    mm.sync_check()
    mo, ml = statistics.fmean(ts["ours"]), statistics.fmean(ts["lib"])
    fl = 2.0 * m * n * p
    print(f"{case:>22s}: ours {mo:9.2f} us ({fl / mo / 1e6:7.1f} TF) med {statistics.median(ts['ours']):8.1f} | "
          f"cuBLAS {ml:9.2f} us ({fl / ml / 1e6:7.1f} TF) med {statistics.median(ts['lib']):8.1f} | ours/lib speed {ml / mo:5.3f}",
          flush=True)
