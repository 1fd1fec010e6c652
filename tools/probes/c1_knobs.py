"""C1 (FP64 256^3) in a 100-product CUDA graph and L2-flushed single launches under FP64 schedule
knob combinations, beside cuBLAS (medians of 3 rounds):  python tools/probes/c1_knobs.py"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2408_15384_b200 as mm  # noqa: E402

A = torch.rand(256, 256, dtype=torch.float64, device="cuda")
B = torch.rand(256, 256, dtype=torch.float64, device="cuda")
C = torch.empty(256, 256, dtype=torch.float64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
variants = [("default", {}), ("CK=1", {"MM_F64_CK": "1"}), ("KS=4", {"MM_F64_KS": "4", "MM_F64_CK": "1"}),
            ("KS=8", {"MM_F64_KS": "8", "MM_F64_CK": "1"}), ("KS=44", {"MM_F64_KS": "44", "MM_F64_CK": "1"}),
            ("KB=1", {"MM_F64_KB": "1"}), ("tile64", {"MM_F64_TILE": "64"})]
ref = torch.mm(A, B)
for name, env in variants + [("cublas", None)]:
    fn = (lambda: torch.mm(A, B, out=C)) if env is None else (lambda: mm.gemm(A, B, out=C))
    os.environ.update(env or {})
    try:
        res = [(bench.per_launch_ms(fn, 40, flush) * 1e3, bench.graph_us(fn, 100, 5)) for _ in range(3)]
        fn()
        torch.cuda.synchronize()
        ok = torch.allclose(C, ref, rtol=0, atol=1e-11)
        print(f"{name:10s} flushed {statistics.median(r[0] for r in res):6.2f} us  graph {statistics.median(r[1] for r in res):5.2f} us  ok={ok}", flush=True)
    finally:
        for k in (env or {}):
            os.environ.pop(k, None)
