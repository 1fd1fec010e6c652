"""MM_F64_EMU vs DMMA vs cuBLAS DGEMM: time per product (events, means) and the normalised
difference of the emulated product from DMMA's (|C_emu - C_dmma| / (|A|·|B|)):
    python tools/probes/f64_emu_probe.py 8192 32768"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2408_15384_b200 as mm  # noqa: E402


def t_ms(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.fmean(ts)


for N in [int(x) for x in sys.argv[1:]] or [8192]:
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.rand(N, N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    B = torch.rand(N, N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    C1 = torch.empty(N, N, dtype=torch.float64, device="cuda")
    C2 = torch.empty_like(C1)
    reps = 3 if N >= 16384 else 10
    te = t_ms(lambda: mm.gemm(A, B, out=C1, f64_emulation=True), reps)
    td = t_ms(lambda: mm.gemm(A, B, out=C2), reps)
    tc = t_ms(lambda: torch.mm(A, B, out=C2), reps)
    mm.gemm(A, B, out=C2)
    mm.sync_check()
    D = torch.mm(A.abs(), B.abs())
    diff = ((C1 - C2).abs() / D).max().item()
    fl = 2.0 * N ** 3
    print(f"FP64 {N}^3: emulated {te:9.2f} ms ({fl / te / 1e9:6.1f} TF)  DMMA {td:9.2f} ms ({fl / td / 1e9:5.1f} TF)  "
          f"cuBLAS {tc:9.2f} ms ({fl / tc / 1e9:5.1f} TF)  emu/cuBLAS speed {tc / te:5.2f}x  max |emu-dmma|/(|A||B|) {diff:.2e}",
          flush=True)
    del A, B, C1, C2, D
    torch.cuda.empty_cache()
