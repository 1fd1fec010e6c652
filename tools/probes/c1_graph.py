"""C1 (FP64 256^3) per product: single launches with L2 flushed (trimmed mean) and in a 100-product
CUDA graph, ours (default = gemm_f64_small, and MM_F64_SMALL=0 = the TMA kernel) vs cuBLAS."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2408_15384_b200 as mm  # noqa: E402

shapes = [tuple(int(x) for x in s.split("x")) for s in (sys.argv[1:] or ["256x256x256"])]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for (m, n, p) in shapes:
    A = torch.rand(m, n, dtype=torch.float64, device="cuda")
    B = torch.rand(n, p, dtype=torch.float64, device="cuda")
    C = torch.empty(m, p, dtype=torch.float64, device="cuda")
    out = {}
    for name, env, fn in (("small", None, lambda: mm.gemm(A, B, out=C)),
                          ("tma", "0", lambda: mm.gemm(A, B, out=C)),
                          ("cublas", None, lambda: torch.mm(A, B, out=C))):
        if env is not None:
            os.environ["MM_F64_SMALL"] = env
        try:
            res = []
            for _ in range(3):
                res.append((bench.per_launch_ms(fn, 40, flush) * 1e3, bench.graph_us(fn, 100, 5)))
            out[name] = (statistics.median(r[0] for r in res), statistics.median(r[1] for r in res))
        finally:
            os.environ.pop("MM_F64_SMALL", None)
    mm.sync_check()
    print(f"{m}x{n}x{p}: " + "  ".join(f"{k}: flushed {v[0]:6.2f} us, graph {v[1]:5.2f} us" for k, v in out.items()),
          flush=True)
