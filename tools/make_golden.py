"""Write tests/golden/oracle_fullsize.json: full-output checksums of the exact-integer
pin products at BASELINE.json's full config shapes, computed ONLY by the CPU oracle
(oracle/) on inputs from synthgen/.  Nothing here touches the CUDA path.

Exact-integer inputs: entries uniform on {-(K-1)/2..(K-1)/2}, so
every partial sum is an integer far below 2^24 (bf16->fp32) / 2^53 (fp64) and the
product is exact in any summation order: the GPU must match it bit for bit.

    python tools/make_golden.py [--only C1x,C2x,C3,C4x3,C4x9,C5x]
Entries are merged into the JSON as each finishes (long runs keep partial results).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synthgen as sg  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_fullsize.json")

CASES = {
    "C1x": dict(dtype="f64", m=256, n=256, p=256, seed=0, K=2049),
    "C2x": dict(dtype="f64", m=2000, n=1500, p=1750, seed=1, K=2049),
    "C3": dict(dtype="s8", m=4096, n=4096, p=4096, seed=2, K=255),
    "C4x3": dict(dtype="bf16", m=16384, n=16384, p=16384, seed=3, K=3),
    "C4x9": dict(dtype="bf16", m=16384, n=16384, p=16384, seed=3, K=9),
    "C5x": dict(dtype="f64", m=32768, n=32768, p=32768, seed=4, K=2049),
}


def compute(c):
    m, n, p, seed, K = c["m"], c["n"], c["p"], c["seed"], c["K"]
    if c["dtype"] == "s8":
        A, B = sg.uniform_i8(seed, 1, m, n), sg.uniform_i8(seed, 2, n, p)
    elif c["dtype"] == "bf16":
        A, B = sg.exact_bf16(seed, 1, K, m, n), sg.exact_bf16(seed, 2, K, n, p)
    else:
        A, B = sg.exact_f64(seed, 1, K, m, n), sg.exact_f64(seed, 2, K, n, p)
    cs = 0
    zeros = 0
    corners = {}
    block = max(1, min(m, (1 << 27) // (8 * p)))  # ~128 MiB of C per block
    for r0 in range(0, m, block):
        rows = np.arange(r0, min(m, r0 + block))
        if c["dtype"] == "s8":
            C = oracle.gemm_s8_rows(A, B, rows)
            assert np.abs(C).max() < 2 ** 31
            cs = (cs + sg.checksum_block(C.astype(np.int32), r0 * p, "i32")) % (1 << 64)
        elif c["dtype"] == "bf16":
            C, _ = oracle.gemm_bf16_rows(A, B, rows)
            assert np.all(np.abs(C) < 2 ** 24)
            cs = (cs + sg.checksum_block(C, r0 * p, "f64_as_f32")) % (1 << 64)
        else:
            C, _ = oracle.gemm_f64_rows(A, B, rows)
            assert np.all(np.abs(C) < 2 ** 53)
            cs = (cs + sg.checksum_block(C, r0 * p, "f64")) % (1 << 64)
        zeros += int((C == 0).sum())
        if r0 == 0:
            corners["C00"] = float(C[0, 0])
            corners["C0_last"] = float(C[0, -1])
        if r0 + len(rows) == m:
            corners["Clast_0"] = float(C[-1, 0])
            corners["Clast_last"] = float(C[-1, -1])
    return dict(c, checksum=f"0x{cs:016x}", zeros=zeros, **corners)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1x,C2x,C3,C4x3,C4x9")
    args = ap.parse_args()
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    data["_about"] = ("Full-output checksums (SURVEY.md §8 d1 checksum) of exact-integer pin products, "
                      "written by tools/make_golden.py calling only oracle/ and synthgen/. "
                      f"Oracle threads: {oracle.max_threads()}.")
    for name in args.only.split(","):
        t0 = time.time()
        res = compute(CASES[name])
        res["oracle_seconds"] = round(time.time() - t0, 1)
        data[name] = res
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
        print(name, res, flush=True)


if __name__ == "__main__":
    main()
