"""Small products through every kernel path, for compute-sanitizer (one tool per run):
    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
Covers: tcgen05 CTA pair / single CTA, 256- and 512-wide tiles, stream-K tail, TMA-store and
register-store epilogues (misaligned C), the pack path, FP64 stream-K with partial tiles."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2408_15384_b200 as mm  # noqa: E402
import synthgen as sg  # noqa: E402


def run(dt, m, n, p, env=None, misalign_c=False):
    env = env or {}
    for k, v in env.items():
        os.environ[k] = v
    try:
        if dt == "bf16":
            A, B = sg.exact_bf16(1, 1, 9, m, n), sg.exact_bf16(1, 2, 9, n, p)
            tA = torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).cuda()
            tB = torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).cuda()
            ref, _ = oracle.gemm_bf16(A, B)
            odt = torch.float32
        elif dt == "i8":
            A, B = sg.exact_i8(1, 1, 255, m, n), sg.exact_i8(1, 2, 255, n, p)
            tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
            ref = oracle.gemm_s8(A, B)
            odt = torch.int32
        else:
            A, B = sg.exact_f64(1, 1, 2049, m, n), sg.exact_f64(1, 2, 2049, n, p)
            tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
            ref = oracle.gemm_f64(A, B)
            odt = torch.float64
        if misalign_c:
            buf = torch.empty(m * p + 1, dtype=odt, device="cuda")
            C = buf[1:].view(m, p)
            mm.gemm(tA, tB, out=C)
        else:
            C = mm.gemm(tA, tB)
        mm.sync_check()
        ok = np.array_equal(C.cpu().numpy().astype(np.float64), np.asarray(ref, np.float64))
        print(f"{dt} {m}x{n}x{p} {env} misalignC={misalign_c}: {'ok' if ok else 'MISMATCH'}", flush=True)
        return ok
    finally:
        for k in env:
            os.environ.pop(k, None)


def main():
    ok = True
    for dt in ("bf16", "i8"):
        ok &= run(dt, 300, 200, 520, {"MM_FORCE_CG": "1"})
        ok &= run(dt, 300, 200, 520, {"MM_FORCE_CG": "2"})
        ok &= run(dt, 512, 1024, 1100, {"MM_FORCE_CG": "2", "MM_NT": "2"})
        ok &= run(dt, 512, 2048, 768, {"MM_FORCE_CG": "2", "MM_STREAMK": "1"})
        ok &= run(dt, 257, 130, 264, {"MM_FORCE_CG": "2"}, misalign_c=True)
        ok &= run(dt, 97, 61, 83)  # pack path (odd pitches)
    ok &= run("f64", 256, 256, 256)
    ok &= run("f64", 300, 2000, 260)  # stream-K partial tiles
    ok &= run("f64", 37, 19, 23)
    print("SANITIZE_CASES", "OK" if ok else "FAIL")


if __name__ == "__main__":
    main()
