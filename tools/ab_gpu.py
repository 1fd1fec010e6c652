"""A/B timing of two builds of libmm_b200.so in ONE process (interleaved reps, L2 flushed),
so box-to-box and thermal drift cancel:
    python tools/ab_gpu.py LIB_A LIB_B [--env-b KEY=VAL ...] [--cases bf16:4096,i8:4096,...]
Env overrides for side B are applied around its calls (getenv is read per call).
"""
import argparse
import ctypes
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

DT = {"f64": (0, torch.float64, torch.float64), "bf16": (1, torch.bfloat16, torch.float32),
      "i8": (2, torch.int8, torch.int32)}


def load(path):
    lib = ctypes.CDLL(path)
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    lib.mm_create.argtypes = [ctypes.c_int, vp, ctypes.c_size_t, ctypes.POINTER(vp)]
    lib.mm_gemm.argtypes = [vp, i64, i64, i64, ctypes.c_int, vp, vp, vp, vp]
    lib.mm_sync_check.argtypes = [vp, vp]
    h = vp()
    assert lib.mm_create(0, None, 0, ctypes.byref(h)) == 0
    return lib, h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib_a")
    ap.add_argument("lib_b")
    ap.add_argument("--env-a", nargs="*", default=[])
    ap.add_argument("--env-b", nargs="*", default=[])
    ap.add_argument("--cases", default="bf16:16384,bf16:8192,bf16:4096,i8:4096,i8:8192,f64:256,f64:2000x1500x1750")
    ap.add_argument("--reps", type=int, default=12)
    args = ap.parse_args()
    A_ = load(args.lib_a)
    B_ = load(args.lib_b)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def envset(kvs):
        old = {}
        for kv in kvs:
            k, v = kv.split("=", 1)
            old[k] = os.environ.get(k)
            os.environ[k] = v
        return old

    def envrestore(old):
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v

    for case in args.cases.split(","):
        dt, shape = case.split(":")
        dims = [int(x) for x in shape.split("x")]
        m, n, p = (dims * 3)[:3] if len(dims) == 1 else dims
        code, tin, tout = DT[dt]
        if dt == "i8":
            A = torch.randint(-127, 128, (m, n), device="cuda", dtype=torch.int8)
            B = torch.randint(-127, 128, (n, p), device="cuda", dtype=torch.int8)
        else:
            A = torch.randn(m, n, device="cuda").to(tin)
            B = torch.randn(n, p, device="cuda").to(tin)
        C = torch.empty(m, p, device="cuda", dtype=tout)
        big = m * n > (1 << 26)
        res = {"A": [], "B": []}
        for side, (lib, h), env in (("A", A_, args.env_a), ("B", B_, args.env_b)):
            old = envset(env)
            for _ in range(3):
                lib.mm_gemm(h, m, n, p, code, A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
            envrestore(old)
        torch.cuda.synchronize()
        for r in range(args.reps):
            for side, (lib, h), env in (("A", A_, args.env_a), ("B", B_, args.env_b)):
                old = envset(env)
                if not big:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record()
                st = lib.mm_gemm(h, m, n, p, code, A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
                e1.record()
                e1.synchronize()
                assert st == 0, st
                res[side].append(e0.elapsed_time(e1))
                envrestore(old)
        for side, (lib, h), _ in (("A", A_, None), ("B", B_, None)):
            assert lib.mm_sync_check(h, s) == 0
        fl = 2.0 * m * n * p
        ma, mb = statistics.median(res["A"]), statistics.median(res["B"])
        # CUDA event times on this pool come in ~2-us steps: the mean over reps resolves finer
        xa, xb = statistics.fmean(res["A"]), statistics.fmean(res["B"])
        print(f"{case:>22s}: A {ma*1e3:9.1f} us ({fl/ma/1e9:7.1f} TF)  B {mb*1e3:9.1f} us ({fl/mb/1e9:7.1f} TF)  "
              f"B/A speed {ma/mb:5.3f}  | means A {xa*1e3:9.2f} B {xb*1e3:9.2f} us, B/A speed {xa/xb:5.3f}", flush=True)
        del A, B, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
