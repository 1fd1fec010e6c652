"""A/B of the persistent-grid residency hazard: a product
launched while tests/libhog.so holds all but 16 SMs, with two builds of the library in one process.

    python tools/hazard_ab.py LIB_A LIB_B [--hold 3.0]

For each library and shape: the time from launch to completion of the product (device events),
whether the hog was still holding the SMs when the product finished, and the device error word
(mm_sync_check).  A library whose CTAs wait for non-resident CTAs finishes only after the hog
releases its SMs (or latches its 4-s pipeline time-out)."""
import argparse
import ctypes
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DT = {"f64": (0, torch.float64, torch.float64), "bf16": (1, torch.bfloat16, torch.float32),
      "i8": (2, torch.int8, torch.int32)}


def load(path):
    lib = ctypes.CDLL(path)
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    lib.mm_create.argtypes = [ctypes.c_int, vp, ctypes.c_size_t, ctypes.POINTER(vp)]
    lib.mm_gemm.argtypes = [vp, i64, i64, i64, ctypes.c_int, vp, vp, vp, vp]
    lib.mm_sync_check.argtypes = [vp, vp]
    lib.mm_last_error.argtypes = [vp]
    lib.mm_last_error.restype = ctypes.c_char_p
    h = vp()
    assert lib.mm_create(0, None, 0, ctypes.byref(h)) == 0
    return lib, h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--hold", type=float, default=3.0)
    ap.add_argument("--cases", default="bf16:8192x8192x8192,bf16:2560x2560x2560,f64:2000x1500x1750")
    args = ap.parse_args()
    hog = ctypes.CDLL(os.path.join(ROOT, "tests", "libhog.so"))
    hog.hog_launch.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p]
    hog.hog_started.restype = ctypes.c_uint
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks = sms - 16
    s_hog = torch.cuda.Stream()
    s = torch.cuda.current_stream().cuda_stream
    out = []
    for path in args.libs:
        lib, h = load(path)
        for case in args.cases.split(","):
            dt, shp = case.split(":")
            m, n, p = (int(x) for x in shp.split("x"))
            code, tin, tout = DT[dt]
            A = torch.randint(-2, 3, (m, n), device="cuda").to(tin)
            B = torch.randint(-2, 3, (n, p), device="cuda").to(tin)
            C = torch.empty(m, p, dtype=tout, device="cuda")
            lib.mm_gemm(h, m, n, p, code, A.data_ptr(), B.data_ptr(), C.data_ptr(), s)  # warm-up
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lib.mm_gemm(h, m, n, p, code, A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
            e1.record()
            e1.synchronize()
            idle_ms = e0.elapsed_time(e1)
            assert hog.hog_launch(blocks, int(args.hold * 1e9), ctypes.c_void_p(s_hog.cuda_stream)) == 0
            while hog.hog_started() < blocks:
                time.sleep(0.001)
            t0 = time.time()
            e0.record()
            lib.mm_gemm(h, m, n, p, code, A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
            e1.record()
            e1.synchronize()
            wall = time.time() - t0
            s_hog.synchronize()
            st = lib.mm_sync_check(h, s)
            ref = torch.mm(A.double(), B.double())
            ok = bool(torch.equal(C.double(), ref))
            rec = {"lib": os.path.basename(path), "case": case, "idle_ms": round(idle_ms, 3),
                   "held_ms": round(e0.elapsed_time(e1), 1), "wall_s": round(wall, 3),
                   "finished_before_hog_released": wall < args.hold - 0.2, "status": st,
                   "error": lib.mm_last_error(h).decode() if st else "", "correct": ok}
            print(json.dumps(rec), flush=True)
            out.append(rec)
    return 0


if __name__ == "__main__":
    sys.exit(main())
