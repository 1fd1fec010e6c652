"""PCIe probe: pinned H2D, D2H, and both directions concurrently (1 GiB each)."""
import time

import torch

N = 1 << 30
h1 = torch.empty(N, dtype=torch.uint8).pin_memory()
h2 = torch.empty(N, dtype=torch.uint8).pin_memory()
d1 = torch.empty(N, dtype=torch.uint8, device="cuda")
d2 = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


h2d = t(lambda: d1.copy_(h1, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


bo = t(both)
print(f"H2D {N/h2d/1e9:.1f} GB/s  D2H {N/d2h/1e9:.1f} GB/s  both-directions {2*N/bo/1e9:.1f} GB/s total "
      f"({bo*1e3:.1f} ms for 1 GiB each way)")
