"""Run FP64 products of one shape (for ncu captures of the DMMA kernel).
    python tools/f64_probe.py M N K [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402
from synthgen import gpu as sgg  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
A = sgg.uniform_f64(4, 1, M, K)
B = sgg.uniform_f64(4, 2, K, N)
C = torch.empty(M, N, dtype=torch.float64, device="cuda")
for _ in range(reps):
    mm.gemm(A, B, out=C)
mm.sync_check()
print("ok")
