"""Time mm_gemm_host on C4 (pinned host buffers) for several block splits."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = torch.randn(N, N).to(torch.bfloat16).pin_memory()
B = torch.randn(N, N).to(torch.bfloat16).pin_memory()
C = torch.empty(N, N, dtype=torch.float32).pin_memory()
for blocks in [int(x) for x in os.environ.get("BLOCKS", "1,2,4,8,16").split(",")]:
    os.environ["MM_HOST_BLOCKS"] = str(blocks)
    mm.gemm_host(A, B, out=C)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        mm.gemm_host(A, B, out=C)
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    print(f"blocks {blocks:2d}: {t*1e3:6.2f} ms  {2*N**3/t/1e12:6.1f} TFLOP/s e2e", flush=True)
