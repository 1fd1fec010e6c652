"""PCIe copy rates for the host-operand path's shapes: contiguous vs 2-D strided blocks, one
vs two streams (copy engines), H2D and D2H, alone and together.  python tools/pcie_2d_probe.py"""
import ctypes
import glob
import os
import time

import torch

# cudaMemcpy2DAsync straight from the CUDA runtime (torch's copy_ of a strided view does not use it)
_rt = None
for pat in ("nvidia/cuda_runtime/lib/libcudart.so*",):
    for base in __import__("sys").path:
        hits = glob.glob(os.path.join(base, pat))
        if hits:
            _rt = ctypes.CDLL(hits[0])
            break
    if _rt:
        break
if _rt is None:
    _rt = ctypes.CDLL("libcudart.so")
_rt.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t,
                                  ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]


def copy2d(dst, dpitch, src, spitch, width, height, kind, stream):
    r = _rt.cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kind, stream.cuda_stream)
    assert r == 0, r

N = 16384
hC = torch.empty(N, N, dtype=torch.float32).pin_memory()
dC = torch.zeros(N, N, dtype=torch.float32, device="cuda")
hB = torch.empty(N, N, dtype=torch.bfloat16).pin_memory()
dB = torch.zeros(N, N, dtype=torch.bfloat16, device="cuda")
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def t(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def rate(nbytes, sec):
    return f"{nbytes / sec / 1e9:6.1f} GB/s"


blk = 4096
# D2H: contiguous 64 MB vs a 4096x4096 fp32 block of a 16384-wide matrix (16 KB rows)
c = t(lambda: hC.view(-1)[:blk * blk].copy_(dC.view(-1)[:blk * blk], non_blocking=True))
print("D2H contiguous 64 MB      ", rate(blk * blk * 4, c))
P4 = N * 4
D2H, H2D = 2, 1


def d2h_block(r0, rows, c0, cols, st):
    copy2d(hC.data_ptr() + (r0 * N + c0) * 4, P4, dC.data_ptr() + (r0 * N + c0) * 4, P4, cols * 4, rows, D2H, st)


c = t(lambda: d2h_block(0, blk, 0, blk, s1))
print("D2H 2-D 4096x4096 fp32    ", rate(blk * blk * 4, c))


def two_d2h():
    d2h_block(0, blk // 2, 0, blk, s1)
    d2h_block(blk // 2, blk // 2, 0, blk, s2)


print("D2H 2-D, two streams      ", rate(blk * blk * 4, t(two_d2h)))


def four_blocks_two_streams():
    for k in range(4):
        d2h_block(k * blk, blk, 0, blk, s1 if k % 2 == 0 else s2)


print("D2H 4 blocks on 2 streams ", rate(4 * blk * blk * 4, t(four_blocks_two_streams)))


def four_blocks_one_stream():
    for k in range(4):
        d2h_block(k * blk, blk, 0, blk, s1)


print("D2H 4 blocks on 1 stream  ", rate(4 * blk * blk * 4, t(four_blocks_one_stream)))
c = t(lambda: d2h_block(0, blk, 0, N, s1))
print("D2H full-width rows 256 MB", rate(blk * N * 4, c))
# H2D: B column panel 16384 x 4096 bf16 (8 KB rows) vs contiguous 128 MB
c = t(lambda: dB.view(-1)[:N * blk].copy_(hB.view(-1)[:N * blk], non_blocking=True))
print("H2D contiguous 128 MB     ", rate(N * blk * 2, c))
def h2d_panel(c0, cols, st):
    copy2d(dB.data_ptr() + c0 * 2, N * 2, hB.data_ptr() + c0 * 2, N * 2, cols * 2, N, H2D, st)


c = t(lambda: h2d_panel(0, blk, s3))
print("H2D 2-D panel 16384x4096  ", rate(N * blk * 2, c))


def both():
    h2d_panel(0, blk, s3)
    d2h_block(0, 2 * blk, 0, blk, s1)


print("H2D panel + D2H 2-D block ", rate(N * blk * 2 + 2 * blk * blk * 4, t(both)))


def both_contig():
    with torch.cuda.stream(s3):
        dB.view(-1)[:N * blk].copy_(hB.view(-1)[:N * blk], non_blocking=True)
    with torch.cuda.stream(s1):
        hC.view(-1)[:2 * blk * blk].copy_(dC.view(-1)[:2 * blk * blk], non_blocking=True)


print("H2D + D2H contiguous      ", rate(N * blk * 2 + 2 * blk * blk * 4, t(both_contig)))
