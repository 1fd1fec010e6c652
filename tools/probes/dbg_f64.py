"""Debug: repeat one FP64 product and report mismatching tiles with their split-tile schedule.
   python tools/dbg_f64.py TILE STREAMK REPS [m n p]"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2408_15384_b200 as mm  # noqa: E402
import synthgen as sg  # noqa: E402

tile, streamk, reps = sys.argv[1], sys.argv[2], int(sys.argv[3])
m, n, p = (int(x) for x in sys.argv[4:7]) if len(sys.argv) > 6 else (1100, 768, 1700)
os.environ["MM_F64_TILE"] = tile
os.environ["MM_F64_STREAMK"] = streamk
bm = int(tile)
tm_, tn_, nkb = math.ceil(m / bm), math.ceil(p / bm), math.ceil(n / 16)
T = tm_ * tn_
nc = min(148, T * 4, max(1, T * nkb // 4))
W = T // nc
tail = T - W * nc
TI = tail * nkb
ntc = max(1, min(nc, tail * 4, TI // 4))
def coords(t, g=8):
    per = g * tn_
    gi = t // per
    first = gi * g
    gm = min(tm_ - first, g)
    r = t - gi * per
    return first + r % gm, r // gm
segs = {}
if streamk == "1" and tail:
    for c in range(ntc):
        it, end = c * TI // ntc, (c + 1) * TI // ntc
        while it < end:
            tt = it // nkb
            k0 = it - tt * nkb
            lim = min((tt + 1) * nkb, end)
            segs.setdefault(coords(W * nc + tt), []).append((c, k0, lim - tt * nkb))
            it = lim
A, B = sg.exact_f64(47, 1, 2049, m, n), sg.exact_f64(47, 2, 2049, n, p)
Cref = oracle.gemm_f64(A, B)
Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
nbad = 0
for rep in range(reps):
    C = mm.gemm(Ad, Bd)
    mm.sync_check()
    C = C.cpu().numpy()
    bad = np.argwhere(C != Cref)
    if len(bad):
        nbad += 1
        tiles = sorted(set((int(i) // bm, int(j) // bm) for i, j in bad))
        print(f"rep {rep}: {len(bad)} mismatches in tiles {tiles}")
        for t in tiles:
            sel = bad[(bad[:, 0] // bm == t[0]) & (bad[:, 1] // bm == t[1])]
            lr = sorted(set((sel[:, 0] % bm).tolist()))
            lc = sorted(set((sel[:, 1] % bm).tolist()))
            print(f"   tile {t}: segments (cta, kb0, kb1) {segs.get(t)}; local rows {lr[:12]}..; cols {lc[0]}..{lc[-1]} ({len(lc)})")
            # explain the error of one element by the segments' partial sums
            i, j = (int(x) for x in sel[0])
            d = C[i, j] - Cref[i, j]
            expl = []
            for (cc, k0, k1) in segs.get(t, []):
                part = float(A[i, k0 * 16:k1 * 16] @ B[k0 * 16:k1 * 16, j])
                expl.append((cc, k0, k1, part))
            print(f"     elem ({i},{j}) err {d}; segment partials {expl}")
print(f"tile {tile} streamk {streamk} shape {m}x{n}x{p}: {nbad}/{reps} launches wrong; T={T} nc={nc} W={W} tail={tail} ntc={ntc}")
