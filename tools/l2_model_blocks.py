"""K direction by blocks of B tile columns (G-invariant: depends on the column only) in the LRU model of tools/l2_model.py.
Result (round 1): group 16: forward 6.59 GB, blocks of 3/4/5/6/8 columns 6.83/6.59/6.41/6.57/6.47 GB."""
import sys
sys.argv = ["x", "110"]
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
import l2_model as L
for g in (16, 8, 12):
    row = [f"group {g}: fwd {L.dram_gb(g, lambda w, tm, tn: 0):.2f}"]
    for B in (3, 4, 5, 6, 8):
        row.append(f"tn//{B} {L.dram_gb(g, lambda w, tm, tn, B=B: (tn // B) & 1):.2f}")
    row.append(f"tm//{g} {L.dram_gb(g, lambda w, tm, tn: (tm // 1) & 1):.2f}")
    print(" | ".join(row), flush=True)
