"""One MM_F64_EMU product of size N (after one warm-up) for ncu launch lists:
    ncu --metrics gpu__time_duration.sum python tools/probes/emu_once.py 8192"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2408_15384_b200 as mm  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = torch.rand(N, N, dtype=torch.float64, device="cuda") * 2 - 1
B = torch.rand(N, N, dtype=torch.float64, device="cuda") * 2 - 1
C = torch.empty(N, N, dtype=torch.float64, device="cuda")
for _ in range(2):
    mm.gemm(A, B, out=C, f64_emulation=True)
mm.sync_check()
print("ok", N)
