"""2-D (pitched) cudaMemcpy2DAsync rates over PCIe, as used by mm_gemm_host."""
import ctypes
import glob
import os
import time

import torch

cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
rt = ctypes.CDLL(cands[0] if cands else "libcudart.so.12")
rt.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t,
                                 ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
H2D, D2H = 1, 2
N = 16384
hB = torch.empty(N, N, dtype=torch.bfloat16).pin_memory()
dB = torch.empty(N, N, dtype=torch.bfloat16, device="cuda")
hC = torch.empty(N, N, dtype=torch.float32).pin_memory()
dC = torch.empty(N, N, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


for panels in (1, 2, 4, 8, 16, 32):
    w = N // panels

    def h2d():
        for j in range(panels):
            r = rt.cudaMemcpy2DAsync(dB.data_ptr() + j * w * 2, N * 2, hB.data_ptr() + j * w * 2, N * 2, w * 2, N, H2D, s)
            assert r == 0, r

    def d2h():
        for j in range(panels):
            r = rt.cudaMemcpy2DAsync(hC.data_ptr() + j * w * 4, N * 4, dC.data_ptr() + j * w * 4, N * 4, w * 4, N, D2H, s)
            assert r == 0, r
    a = t(h2d)
    b = t(d2h)
    print(f"panels {panels:2d} (rows of {w*2} B / {w*4} B): H2D {N*N*2/a/1e9:6.1f} GB/s  D2H {N*N*4/b/1e9:6.1f} GB/s",
          flush=True)
