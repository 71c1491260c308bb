"""Device time of project_compatible (exact parallel chain vs the literal
chain, DECMG_PROJ_SEQ=1) on config 4's mesh with 16 RHS, and the fallback
count. Usage: python tools/proj_time.py [nsub] [nrhs]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_12501_b200 as d  # noqa: E402

nsub = int(sys.argv[1]) if len(sys.argv) > 1 else 10
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 16
h = d.MultigridHierarchy.from_base("ico", nsub, max_nrhs=nrhs)
B = h.make_rhs("uniform", 1, nrhs)
for rep in range(3):
    f0 = h.projection_fallbacks()
    h.set_timing(True)
    h.timing(-1)
    h.project_compatible(B)
    ms = h.timing(6)
    h.set_timing(False)
    segs = -(-h.n() // 256) * nrhs
    print(f"n={h.n()} nrhs={nrhs}: projection kernels {ms[1]:.2f} ms in {ms[0]} launches; "
          f"fallback segments {h.projection_fallbacks() - f0} of {segs}")
