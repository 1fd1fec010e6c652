"""MM_F64_EMU under schedule knobs of its INT8 products (one process, rounds in alternating order):
    python tools/probes/emu_knobs.py N [N ...]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2408_15384_b200 as mm  # noqa: E402

VARIANTS = [("default", {}), ("WAVE_SYNC=0", {"MM_WAVE_SYNC": "0"}), ("GROUP_M=8", {"MM_GROUP_M": "8"}),
            ("GROUP_M=32", {"MM_GROUP_M": "32"}), ("NT=1", {"MM_NT": "1"})]


def t(fn, reps):
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


for N in [int(x) for x in sys.argv[1:]] or [16384]:
    A = torch.rand(N, N, dtype=torch.float64, device="cuda")
    B = torch.rand(N, N, dtype=torch.float64, device="cuda")
    C = torch.empty_like(A)
    res = {}
    reps = 2 if N >= 32768 else 4
    for rnd in range(2):
        for name, env in (VARIANTS if rnd == 0 else VARIANTS[::-1]):
            os.environ.update(env)
            try:
                res.setdefault(name, []).append(t(lambda: mm.gemm(A, B, out=C, f64_emulation=True), reps))
            finally:
                for k in env:
                    os.environ.pop(k, None)
    base = statistics.fmean(res["default"])
    print(f"{N}^3: " + "  ".join(f"{k} {statistics.fmean(v):8.2f} ms ({base / statistics.fmean(v):5.3f}x)" for k, v in res.items()),
          flush=True)
    del A, B, C
    torch.cuda.empty_cache()
