"""Run one product shape a few times (for ncu captures):  python tools/one_case.py i8:4096 [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402

dt, shp = sys.argv[1].split(":")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dims = [int(x) for x in shp.split("x")]
m, n, p = dims if len(dims) == 3 else dims * 3
tin, tout = {"f64": (torch.float64, torch.float64), "bf16": (torch.bfloat16, torch.float32),
             "i8": (torch.int8, torch.int32)}[dt]
if dt == "i8":
    A = torch.randint(-127, 128, (m, n), dtype=torch.int8, device="cuda")
    B = torch.randint(-127, 128, (n, p), dtype=torch.int8, device="cuda")
else:
    A = torch.randn(m, n, device="cuda").to(tin)
    B = torch.randn(n, p, device="cuda").to(tin)
C = torch.empty(m, p, dtype=tout, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if os.environ.get("FLUSH") else None
for _ in range(reps):
    if flush is not None:
        flush.fill_(1)  # (FLUSH=1: L2 full of other data before every call)
    if os.environ.get("LIB"):  # (LIB=1: the cuBLAS product on the same operands instead)
        if dt == "i8":
            torch._int_mm(A, B, out=C)
        elif dt == "bf16":
            torch.mm(A, B, out_dtype=torch.float32, out=C)
        else:
            torch.mm(A, B, out=C)
    else:
        mm.gemm(A, B, out=C)
mm.sync_check()
print("ok", dt, m, n, p)
