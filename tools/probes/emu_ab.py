"""A/B of MM_F64_EMU between two builds of the library (ctypes, same operands, events, means after
one warm-up) plus both builds' normalised difference from DMMA (|C - C_dmma| / (|A|·|B|)):
    python tools/probes/emu_ab.py libA.so libB.so [shape ...]    shape = m,n,p or N"""
import ctypes
import statistics
import sys

import torch

vp, i64 = ctypes.c_void_p, ctypes.c_int64
libs = [ctypes.CDLL(p) for p in sys.argv[1:3]]
hs = []
for lib in libs:
    lib.mm_create.argtypes = [ctypes.c_int, vp, ctypes.c_size_t, ctypes.POINTER(vp)]
    lib.mm_gemm.argtypes = [vp, i64, i64, i64, ctypes.c_int, vp, vp, vp, vp]
    lib.mm_last_error.argtypes = [vp]
    lib.mm_last_error.restype = ctypes.c_char_p
    h = vp()
    assert lib.mm_create(0, None, 0, ctypes.byref(h)) == 0
    hs.append(h)
s = torch.cuda.current_stream().cuda_stream
shapes = [tuple(int(x) for x in a.split(",")) if "," in a else (int(a),) * 3 for a in sys.argv[3:]] or [(4096,) * 3]
for m, n, p in shapes:
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.rand(m, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    B = torch.rand(n, p, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    Cd = torch.empty(m, p, dtype=torch.float64, device="cuda")
    assert libs[1].mm_gemm(hs[1], m, n, p, 0, A.data_ptr(), B.data_ptr(), Cd.data_ptr(), s) == 0
    reps = 3 if m * n * p >= 16384 ** 3 else 10
    res = []
    for lib, h in zip(libs, hs):
        C = torch.empty(m, p, dtype=torch.float64, device="cuda")
        ts = []
        for r in range(reps + 1):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            st = lib.mm_gemm(h, m, n, p, 3, A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
            assert st == 0, lib.mm_last_error(h)
            e1.record()
            e1.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        diff = ((C - Cd).abs().max() / (A.abs().max() * B.abs().max() * n)).item()
        res.append((statistics.fmean(ts), diff))
        del C
    fl = 2.0 * m * n * p
    (ta, da), (tb, db) = res
    print(f"F64_EMU {m}x{n}x{p}: A {ta:9.3f} ms ({fl / ta / 1e9:6.1f} TF, diff {da:.1e})  "
          f"B {tb:9.3f} ms ({fl / tb / 1e9:6.1f} TF, diff {db:.1e})  B/A speed {ta / tb:5.3f}", flush=True)
    del A, B, Cd
    torch.cuda.empty_cache()
