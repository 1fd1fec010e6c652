"""Run one BF16 product of a given shape (for ncu DRAM-traffic probes).
    python tools/dram_probe.py M N K [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(K, N, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.float32)
for _ in range(reps):
    mm.gemm(A, B, out=C)
mm.sync_check()
print("ok", M, N, K)
