"""Run cuBLAS and ours on a few shapes (for an ncu launch list: kernel names + bytes).
    python tools/cublas_shapes.py [bf16:8192,i8:4096,...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402

cases = (sys.argv[1] if len(sys.argv) > 1 else "bf16:4096,bf16:8192,bf16:16384,i8:4096,i8:8192,f64:256,f64:8192").split(",")
for case in cases:
    dt, s = case.split(":")
    m = n = p = int(s)
    if dt == "i8":
        A = torch.randint(-127, 128, (m, n), dtype=torch.int8, device="cuda")
        B = torch.randint(-127, 128, (n, p), dtype=torch.int8, device="cuda")
        ref = lambda: torch._int_mm(A, B)  # noqa: E731
    else:
        t = torch.bfloat16 if dt == "bf16" else torch.float64
        A = torch.randn(m, n, device="cuda").to(t)
        B = torch.randn(n, p, device="cuda").to(t)
        ref = lambda: torch.matmul(A, B)  # noqa: E731
    for _ in range(2):
        ref()
        mm.gemm(A, B)
    torch.cuda.synchronize()
    del A, B
    torch.cuda.empty_cache()
print("ok")
