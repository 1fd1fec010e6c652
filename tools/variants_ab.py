"""Schedule-knob variants of one shape against cuBLAS, in alternating windows (same thermal state):

    python tools/variants_ab.py bf16:16384 --window-s 2 --variants "base;MM_NT=1;MM_MC=2" [--flush]

Each round runs every variant (env knobs for the library) and cuBLAS for `window-s` seconds of
back-to-back products (or --reps single launches with an L2 flush before each, --flush); prints
per variant the median ms per product, TFLOP/s and the ratio to cuBLAS measured in the same round."""
import argparse
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402

TIN = {"f64": torch.float64, "bf16": torch.bfloat16, "i8": torch.int8}
TOUT = {"f64": torch.float64, "bf16": torch.float32, "i8": torch.int32}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--variants", default="base")
    ap.add_argument("--window-s", type=float, default=2.0)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--flush", action="store_true")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--graph", action="store_true", help="per-product time of 100 products replayed from a CUDA graph")
    args = ap.parse_args()
    dt, shp = args.case.split(":")
    dims = [int(x) for x in shp.split("x")]
    m, n, p = dims * 3 if len(dims) == 1 else dims
    if dt == "i8":
        A = torch.randint(-127, 128, (m, n), dtype=torch.int8, device="cuda")
        B = torch.randint(-127, 128, (n, p), dtype=torch.int8, device="cuda")
    else:
        A = torch.randn(m, n, device="cuda").to(TIN[dt])
        B = torch.randn(n, p, device="cuda").to(TIN[dt])
    C = torch.empty(m, p, dtype=TOUT[dt], device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if args.flush else None

    def lib():
        if dt == "i8":
            torch._int_mm(A, B, out=C)
        elif dt == "bf16":
            torch.mm(A, B, out_dtype=torch.float32, out=C)
        else:
            torch.mm(A, B, out=C)

    variants = [v.strip() for v in args.variants.split(";") if v.strip()]

    def run(fn, env):
        old = {}
        for kv in env:
            k, v = kv.split("=", 1)
            old[k] = os.environ.get(k)
            os.environ[k] = v
        try:
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            if args.graph:
                st = torch.cuda.Stream()
                st.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(st):
                    fn()
                torch.cuda.current_stream().wait_stream(st)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for _ in range(100):
                        fn()
                g.replay()
                torch.cuda.synchronize()
                ts = []
                for _ in range(args.reps):
                    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                    e0.record()
                    g.replay()
                    e1.record()
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1) / 100)
                return statistics.median(ts)
            if flush is not None:
                ts = []
                for _ in range(args.reps):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                    e0.record()
                    fn()
                    e1.record()
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1))
                return statistics.median(ts)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            k = max(3, int(args.window_s * 1e3 / max(e0.elapsed_time(e1), 1e-3)))
            e0.record()
            for _ in range(k):
                fn()
            e1.record()
            e1.synchronize()
            return e0.elapsed_time(e1) / k
        finally:
            for k2, v in old.items():
                if v is None:
                    os.environ.pop(k2, None)
                else:
                    os.environ[k2] = v

    res = {v: [] for v in variants}
    res["cublas"] = []
    for r in range(args.rounds):
        for v in variants:
            env = [] if v == "base" else [x for x in v.split(",") if "=" in x]
            res[v].append(run(lambda: mm.gemm(A, B, out=C), env))
            time.sleep(0.2)
        res["cublas"].append(run(lib, []))
        time.sleep(0.2)
    mm.sync_check()
    fl = 2.0 * m * n * p
    lib_ms = statistics.median(res["cublas"])
    mode = "graph x100" if args.graph else ("flush" if flush is not None else f"{args.window_s}s windows")
    print(f"{args.case} {mode}: cuBLAS {lib_ms:.4f} ms "
          f"({fl / lib_ms / 1e9:.1f} TF)")
    for v in variants:
        ms = statistics.median(res[v])
        print(f"  {v:40s} {ms:9.4f} ms {fl / ms / 1e9:8.1f} TF   vs cuBLAS {lib_ms / ms:6.3f}   rounds "
              + " ".join(f"{x:.4f}" for x in res[v]), flush=True)


if __name__ == "__main__":
    main()
