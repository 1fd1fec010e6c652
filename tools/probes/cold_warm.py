"""Ours vs cuBLAS on one shape under three cache states (CUDA events around the product only):
warm (operands left in L2 by the previous call), after a 512-MB write flush (L2 full of dirty
lines), after a 512-MB read flush (L2 full of clean lines).
    python tools/cold_warm.py i8:4096 bf16:4096 ...
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402


def timeit(fn, prep, reps=30):
    ts = []
    for _ in range(reps):
        prep()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def main():
    wbuf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    rbuf = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
    sink = torch.empty(1, dtype=torch.float32, device="cuda")
    preps = {"warm": lambda: None, "wflush": lambda: wbuf.fill_(1), "rflush": lambda: torch.sum(rbuf, 0, out=sink[0])}
    for case in sys.argv[1:]:
        dt, n = case.split(":")
        n = int(n)
        if dt == "i8":
            A = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
            B = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
            C = torch.empty(n, n, dtype=torch.int32, device="cuda")
            lib = lambda: torch._int_mm(A, B, out=C)  # noqa: E731
        else:
            A = torch.randn(n, n, device="cuda").to(torch.bfloat16)
            B = torch.randn(n, n, device="cuda").to(torch.bfloat16)
            C = torch.empty(n, n, dtype=torch.float32, device="cuda")
            lib = lambda: torch.mm(A, B, out_dtype=torch.float32, out=C)  # noqa: E731
        ours = lambda: mm.gemm(A, B, out=C)  # noqa: E731
        for _ in range(5):
            ours(); lib()
        torch.cuda.synchronize()
        row = []
        for st, prep in preps.items():
            a = [timeit(ours, prep, 20) for _ in range(2)]
            b = [timeit(lib, prep, 20) for _ in range(2)]
            row.append(f"{st}: ours {min(a):6.1f} cublas {min(b):6.1f}")
        print(f"{case:>10}  " + " | ".join(row), flush=True)
    mm.sync_check()


if __name__ == "__main__":
    main()
