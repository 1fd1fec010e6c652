"""C3 (INT8 4096^3) once through the library and once through cuBLAS (torch._int_mm), after a
warm-up of each, for ncu captures:  ncu ... python tools/probes/c3_once.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2408_15384_b200 as mm  # noqa: E402

A = torch.randint(-127, 128, (4096, 4096), dtype=torch.int8, device="cuda")
B = torch.randint(-127, 128, (4096, 4096), dtype=torch.int8, device="cuda")
C = torch.empty(4096, 4096, dtype=torch.int32, device="cuda")
for _ in range(2):
    mm.gemm(A, B, out=C)
    torch._int_mm(A, B, out=C)
mm.sync_check()
print("ok")
