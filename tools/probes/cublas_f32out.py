"""cuBLAS bf16 x bf16 -> fp32 (torch.mm out_dtype) vs ours on C4-shaped operands: kernel names for
ncu and a sustained back-to-back comparison.   python tools/cublas_f32out.py [N] [steps]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
A = torch.randn(N, N, device="cuda").to(torch.bfloat16)
B = torch.randn(N, N, device="cuda").to(torch.bfloat16)
C1 = torch.empty(N, N, device="cuda", dtype=torch.float32)
C2 = torch.empty(N, N, device="cuda", dtype=torch.float32)
ours = lambda: mm.gemm(A, B, out=C1)  # noqa: E731
lib = lambda: torch.mm(A, B, out_dtype=torch.float32, out=C2)  # noqa: E731


def run(fn, k):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / k


for rnd in range(3):
    for name, fn in (("ours", ours), ("cublas", lib)):
        ms = run(fn, steps)
        print(f"round {rnd} {name:6s}: {ms:.3f} ms  {2 * N**3 / ms / 1e9:.1f} TFLOP/s", flush=True)
        time.sleep(0.5)
print("max |diff|", (C1 - C2).abs().max().item())
