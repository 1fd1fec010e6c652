"""Does the clock meter (mm_clock_meter) change a product's time?  C3 shape, L2 flushed, interleaved."""
import os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2408_15384_b200 as mm
A = torch.randint(-127, 128, (4096, 4096), dtype=torch.int8, device="cuda")
B = torch.randint(-127, 128, (4096, 4096), dtype=torch.int8, device="cuda")
C = torch.empty(4096, 4096, dtype=torch.int32, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
res = {"off": [], "on": []}
for _ in range(5):
    mm.gemm(A, B, out=C)
for r in range(60):
    for mode in ("off", "on"):
        if mode == "on":
            mm.clock_meter(True)
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); mm.gemm(A, B, out=C); e1.record(); e1.synchronize()
        res[mode].append(e0.elapsed_time(e1))
        if mode == "on":
            mm.clock_meter(False)
print({k: round(statistics.median(v) * 1e3, 2) for k, v in res.items()}, "us")
