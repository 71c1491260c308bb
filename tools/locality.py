"""Access locality of the level-0 row kernels on a GPU-built hierarchy.

For the Morton row order `order` (row q of the ELL operators is vertex
order[q]) prints (1) how far apart in memory consecutive rows' vectors are in
the reference numbering (b / x' traffic), and (2) for the neighbour columns of
every row, the distance between the column's Morton position and the row's
position (how local the x gathers would be if vectors were stored in Morton
order). Usage: python tools/locality.py [nsub]
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2508_12501_b200 as d  # noqa: E402

nsub = int(sys.argv[1]) if len(sys.argv) > 1 else 10
h = d.MultigridHierarchy.from_base("ico", nsub)
order = h.export(0, "order")
n = order.size
rp = h.export(0, "L_row_ptr").astype(np.int64)
ci = h.export(0, "L_col_idx").astype(np.int64)
pos = np.empty(n, np.int64)
pos[order] = np.arange(n)
step = np.abs(np.diff(order.astype(np.int64)))
print(f"n={n}")
for k in (1, 2, 8, 64, 1024):
    print(f"  consecutive rows, |delta index| <= {k:5d}: {np.mean(step <= k):.3f}")
rows = np.repeat(np.arange(n), np.diff(rp))
dist = np.abs(pos[ci] - pos[rows])
for k in (0, 56, 224, 1024, 4096, 16384, 65536):
    print(f"  neighbour refs within +-{k:6d} Morton rows: {np.mean(dist <= k):.4f}")
dref = np.abs(ci - rows)
for k in (1024, 65536):
    print(f"  neighbour refs within +-{k:6d} reference rows: {np.mean(dref <= k):.4f}")

# restriction rows: R row of coarse vertex i gathers the fine residual at its
# copy (reference id i) and at the midpoints around it; distance of those
# columns from the copy's internal row (the window a fused residual +
# restriction pass would need)
Rrp = h.export(0, "R_row_ptr").astype(np.int64)
Rci = h.export(0, "R_col_idx").astype(np.int64)
nc = Rrp.size - 1
crow = np.repeat(np.arange(nc), np.diff(Rrp))
dR = pos[Rci] - pos[crow]
for lo, hi in ((-56, 56), (-112, 56), (-112, 112), (-224, 112), (-224, 224)):
    print(f"  R entries with column within [{lo}, +{hi}] rows of the copy: {np.mean((dR >= lo) & (dR <= hi)):.4f}")
rows_ok = np.zeros(nc, bool)
for lo, hi in ((-112, 56), (-224, 112)):
    ok = (dR >= lo) & (dR <= hi)
    allok = np.minimum.reduceat(ok.astype(np.int8), Rrp[:-1]) == 1
    print(f"  R rows with every column within [{lo}, +{hi}]: {np.mean(allok):.4f}")
