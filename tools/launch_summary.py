"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel and grid: launches, total ns, share of all kernel time.
Usage: python tools/launch_summary.py launches.csv > summary.csv"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iv, ig = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    name = re.sub(r"^void |decmg_gpu::|\(anonymous namespace\)::|<unnamed>::|\(.*$", "", r[ik]).strip()
    a = agg[(name, r[ig])]
    a[0] += 1
    a[1] += float(r[iv].replace(",", ""))
tot = sum(a[1] for a in agg.values())
w = csv.writer(sys.stdout)
w.writerow(["kernel", "grid", "launches", "total_ns", "share"])
for (name, grid), (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    w.writerow([name, grid, n, int(t), round(t / tot, 5)])
