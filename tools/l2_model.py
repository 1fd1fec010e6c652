"""LRU model of the C4 kernel's DRAM operand reads at slab granularity (A slab = 256 rows x 64 k
bf16 = 32 KB, B slab = 64 k x 512 cols = 64 KB; 74 pair tiles per wave walking K in lockstep, as the
wave barrier enforces).  It reproduces the measured 6.59 GB/launch (ncu dram__bytes_read, group-16
raster) and compares rasters / K orders:
    python tools/l2_model.py [L2_MB=110]
Results (round 1): forward K, group 8/10/12/14/16/20/24: 6.98/6.74/6.71/6.49/6.59/7.35/7.53 GB;
reversing K on odd waves (group 16): 5.18 GB — not used: it changes the FP32 summation order of a
tile with its wave parity, which breaks the G-invariance contract (row blocks bit-identical to the
single product); K direction by column parity (G-invariant): 6.41-6.83 GB, no gain."""
import sys
from collections import OrderedDict

TM, TN, NKB = 64, 32, 256  # 16384/256 tile rows, 16384/512 tile cols, 16384/64 k-blocks
NC = 74                    # CTA pairs
L2 = int(float(sys.argv[1] if len(sys.argv) > 1 else 110) * 2**20)


def coords(t, g):
    per = g * TN
    gi = t // per
    first = gi * g
    gm = min(TM - first, g)
    r = t - gi * per
    return first + r % gm, r // gm


def dram_gb(g, direction):
    lru, size, miss = OrderedDict(), 0, 0
    T = TM * TN
    for wi, w0 in enumerate(range(0, T, NC)):
        tiles = [coords(t, g) for t in range(w0, min(T, w0 + NC))]
        dirs = [direction(wi, tm, tn) for tm, tn in tiles]
        for i in range(NKB):
            for (tm, tn), d in zip(tiles, dirs):
                k = i if d == 0 else NKB - 1 - i
                for key, sz in ((("A", tm, k), 32768), (("B", tn, k), 65536)):
                    if key in lru:
                        lru.move_to_end(key)
                    else:
                        miss += sz
                        lru[key] = sz
                        size += sz
                        while size > L2:
                            size -= lru.popitem(last=False)[1]
    return miss / 1e9


if __name__ == "__main__":
    for g in (8, 16):
        print(f"group {g:2d}: forward {dram_gb(g, lambda w, tm, tn: 0):.2f} GB | odd waves reversed "
              f"{dram_gb(g, lambda w, tm, tn: w & 1):.2f} GB | column-parity direction "
              f"{dram_gb(g, lambda w, tm, tn: tn & 1):.2f} GB", flush=True)
