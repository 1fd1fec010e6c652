"""Per-kernel sums of an ncu launch list (gpu__time_duration.sum CSV), last `--last` launches:
    python tools/probes/launch_breakdown.py launches.csv [--last K]"""
import collections
import csv
import re
import sys

path = sys.argv[1]
last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else None
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ki, mi = h.index("Kernel Name"), h.index("Metric Value")
rows = rows[1:] if last is None else rows[-last:]
agg = collections.OrderedDict()
for r in rows:
    name = re.sub(r"\(.*", "", r[ki]).replace("void mmb::<unnamed>::", "").replace("mmb::<unnamed>::", "")
    name = re.sub(r"reduce_mod_kernel<\d+>", "reduce_mod_kernel<L>", name)
    agg.setdefault(name, []).append(float(r[mi].replace(",", "")) / 1e3)
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    print(f"{len(v):4d} x {k:45s} sum {sum(v):10.1f} us  mean {sum(v) / len(v):9.1f} us  {100 * sum(v) / tot:5.1f} %")
print(f"total {tot:.1f} us")
