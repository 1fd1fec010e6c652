"""Quick GPU diagnostics for the kernels: structured inputs whose products are
easy to read (identity, index patterns), printed mismatch maps.  Run on a B200:
    python tools/probe_gpu.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402
import oracle  # noqa: E402  (test infrastructure: diagnostics compare against it)
import synthgen as sg  # noqa: E402


def bf16_t(x):
    return torch.from_numpy(np.ascontiguousarray(x).astype(np.float32)).to(torch.bfloat16)


def run(A, B, cg=None):
    if cg:
        os.environ["MM_FORCE_CG"] = str(cg)
    else:
        os.environ.pop("MM_FORCE_CG", None)
    C = mm.gemm(A.cuda(), B.cuda())
    mm.sync_check()
    return C.cpu()


def report(name, got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    bad = got != ref
    print(f"{name}: shape {ref.shape} mismatches {bad.sum()} / {bad.size}", flush=True)
    if bad.any():
        idx = np.argwhere(bad)
        print("  first bad:", [(tuple(i), got[tuple(i)], ref[tuple(i)]) for i in idx[:6]])
        rows = np.unique(idx[:, 0])
        cols = np.unique(idx[:, 1])
        print(f"  bad rows {rows[:10]}.. ({rows.size}) bad cols {cols[:10]}.. ({cols.size})")
        print("  got[0,:8] =", got[0, :8], " ref[0,:8] =", ref[0, :8])
        if got.shape[0] > 1:
            print("  got[1,:8] =", got[1, :8], " ref[1,:8] =", ref[1, :8])
    return not bad.any()


def main():
    print(mm.version(), torch.cuda.get_device_name(0), flush=True)
    ok = True
    for dt in ("bf16", "i8"):
        for cg in (1, 2):
            for (m, n, p) in [(128 * cg, 128, 256), (256, 256, 512), (300, 200, 520)]:
                if dt == "bf16":
                    Ai = np.eye(m, n)
                    Bi = ((np.arange(n)[:, None] * 7 + np.arange(p)[None, :]) % 13 - 6).astype(np.float64)
                    A, B = bf16_t(Ai), bf16_t(Bi)
                else:
                    Ai = np.eye(m, n)
                    Bi = ((np.arange(n)[:, None] * 7 + np.arange(p)[None, :]) % 13 - 6).astype(np.float64)
                    A = torch.from_numpy(Ai.astype(np.int8))
                    B = torch.from_numpy(Bi.astype(np.int8))
                t0 = time.time()
                try:
                    C = run(A, B, cg)
                except Exception as e:  # noqa: BLE001
                    print(f"{dt} cg{cg} {m}x{n}x{p}: EXCEPTION {e}", flush=True)
                    ok = False
                    continue
                ok &= report(f"{dt} cg{cg} identity {m}x{n}x{p} ({time.time()-t0:.2f}s)", C.numpy(), Ai @ Bi)
                # random exact ints
                if dt == "bf16":
                    Ab = sg.exact_bf16(1, 1, 9, m, n)
                    Bb = sg.exact_bf16(1, 2, 9, n, p)
                    Cr, _ = oracle.gemm_bf16(Ab, Bb)
                    C = run(torch.from_numpy(Ab.view(np.int16)).view(torch.bfloat16),
                            torch.from_numpy(Bb.view(np.int16)).view(torch.bfloat16), cg)
                else:
                    Ab = sg.uniform_i8(1, 1, m, n)
                    Bb = sg.uniform_i8(1, 2, n, p)
                    Cr = oracle.gemm_s8(Ab, Bb)
                    C = run(torch.from_numpy(Ab), torch.from_numpy(Bb), cg)
                ok &= report(f"{dt} cg{cg} random-int {m}x{n}x{p}", C.numpy(), Cr)
    for (m, n, p) in [(128, 16, 128), (256, 256, 256), (2000, 1500, 1750), (37, 19, 23)]:
        A = sg.exact_f64(0, 1, 2049, m, n)
        B = sg.exact_f64(0, 2, 2049, n, p)
        try:
            C = run(torch.from_numpy(A), torch.from_numpy(B))
        except Exception as e:  # noqa: BLE001
            print(f"f64 {m}x{n}x{p}: EXCEPTION {e}", flush=True)
            ok = False
            continue
        ok &= report(f"f64 exact {m}x{n}x{p}", C.numpy(), oracle.gemm_f64(A, B))
    print("PROBE", "OK" if ok else "FAIL")


if __name__ == "__main__":
    main()
