"""Print one V-cycle's launches (kernel, grid, us) from an ncu launch-list CSV
(--metrics gpu__time_duration.sum): the segment between the last two k_vtail
launches (or the last N launches). python tools/launch_cycle.py file.csv"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))


def short(n):
    n = re.sub(r"\(.*", "", n.replace("void ", ""))
    return re.sub(r"^.*?(?=k_|cub)", "", n)  # drop namespaces ("decmg_gpu::", "<unnamed>::" / "unnamed>::")


seq = [(short(d["Kernel Name"]), d["Grid Size"], float(d["Metric Value"]) / 1000) for d in data]
vt = [i for i, s in enumerate(seq) if s[0].startswith("k_vtail")]
a, b = vt[-2], vt[-1]
tot = 0.0
for s in seq[a + 1:b + 1]:
    print(f"{s[0][:40]:40s} {s[1]:>16s} {s[2]:8.1f}")
    tot += s[2]
print("cycle us", round(tot, 1))
