"""Every BASELINE config on one GPU: setup time, V(2,2) cycle time (device, K
cycles in one run_cycles call), cycles and time to 1e-8 through gmg_solve
(host to host, pinned buffers), unknowns*cycles/s and the whole-cycle
fraction of the measured HBM peak (SURVEY 8(d) byte model). One JSON line per
config. Usage: python tools/configs_sweep.py [names...]"""
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_12501_b200 as d  # noqa: E402
from paper_2508_12501_b200 import _lib  # noqa: E402
from paper_2508_12501_b200.multigrid import _plan_struct  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
    else 6650.0
CONFIGS = {  # name: (base, nsub, dirichlet, rhs kind, nrhs)
    "config1": ("square", 4, True, "sinsin", 1),
    "config2": ("ico", 6, False, "ylm", 1),
    "config3": ("ico", 8, False, "uniform", 1),
    "config4": ("ico", 10, False, "uniform", 16),
    "config5a": ("square", 12, True, "uniform", 1),
    "config5b": ("ico", 11, False, "uniform", 1),
}


def b_alg(h, nrhs):
    L = h.levels()
    inf = [h.level_info(k) for k in range(L)]
    tot = 0.0
    for k in range(L - 1):
        nk, nc = inf[k]["nv"], inf[k + 1]["nv"]
        Mk = 12.0 * inf[k]["nnz_L"] + 4.0 * (nk + 1)
        sweep = Mk + 24.0 * nk * nrhs
        tot += 4 * sweep if k == 0 else 8.0 * nk + 16.0 * nk * nrhs + 3 * sweep
        tot += Mk + 16.0 * nk * nrhs + 12.0 * inf[k]["nnz_R"] + 4.0 * (nc + 1) + 8.0 * nc * nrhs
        tot += 12.0 * inf[k]["nnz_P"] + 4.0 * (nk + 1) + 8.0 * nc * nrhs + 16.0 * nk * nrhs
    return tot


lib = _lib.load()
for name in (sys.argv[1:] or list(CONFIGS)):
    base, nsub, dirichlet, kind, nrhs = CONFIGS[name]
    t0 = time.perf_counter()
    h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=dirichlet, max_nrhs=nrhs)
    setup = time.perf_counter() - t0
    n = h.n()
    B = h.make_rhs(kind, 1, nrhs) if nrhs > 1 else h.make_rhs(kind, 1)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    ps, keep = _plan_struct(plan, h.levels())
    Bd = torch.from_numpy(h.project_compatible(B) if not dirichlet else B).reshape(n, nrhs).cuda()
    Xd = torch.empty_like(Bd)
    K = 10 if n > 100000 else 50
    hist = torch.empty((K, nrhs), dtype=torch.float64, device="cuda")
    run = lambda k: _lib.check(lib.decmg_gpu_run_cycles_dev(h.ctx, C.byref(ps), nrhs, C.c_void_p(Bd.data_ptr()),
                                                           None, k, C.c_void_p(Xd.data_ptr()),
                                                           C.c_void_p(hist.data_ptr())), h.ctx)
    run(3)
    torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(h.stream())  # the context's stream: events must sit on it
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        e0.record(st)
        run(K)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / K)
    ms = min(ts)
    hb = torch.from_numpy(np.ascontiguousarray(B.reshape(n, nrhs))).pin_memory()
    hx = torch.empty_like(hb).pin_memory()
    hh = np.zeros((400, nrhs))
    done = np.zeros(nrhs, dtype=np.int32)
    fin = np.zeros(nrhs)
    solve = lambda: _lib.check(lib.decmg_gpu_solve(h.ctx, C.byref(ps), nrhs, C.c_void_p(hb.data_ptr()), None, 1e-8,
                                                   400, C.c_void_p(hx.data_ptr()), hh.ctypes.data_as(C.c_void_p),
                                                   done.ctypes.data_as(C.c_void_p),
                                                   fin.ctypes.data_as(C.c_void_p)), h.ctx)
    solve()
    t0 = time.perf_counter()
    solve()
    tsol = time.perf_counter() - t0
    ba = b_alg(h, nrhs)
    print(json.dumps({"config": name, "vertices": n, "levels": h.levels(), "nrhs": nrhs, "setup_s": round(setup, 3),
                      "ms_per_cycle": round(ms, 4), "unknowns_cycles_per_s": n * nrhs / (ms / 1e3),
                      "cycle_hbm_frac": round(ba / (ms / 1e3) / 1e9 / PEAK, 3), "b_alg_gb": round(ba / 1e9, 3),
                      "cycles_to_1e-8": int(done.max()), "time_to_1e-8_s": round(tsol, 4),
                      "final_rel_residual_max": float(fin.max())}), flush=True)
    del h
