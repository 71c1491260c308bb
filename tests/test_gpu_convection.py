"""The reference's downstream consumer on the GPU path.

oracle/_ref/convection_gpu is the reference's own physics.cpp and rk54.cpp,
unmodified, compiled with include/dropin ahead of the reference's headers
(`make -C oracle convection`): integrate_convection (physics.cpp:220-272) then
runs every pressure solve -- one warm-started gmg_solve per Runge-Kutta stage
(solve_pressure_rhs, physics.cpp:136-166) -- through libdecmg_gpu.so. The
goldens are the same main() linked against the reference itself on the CPU
(tests/golden/make_golden.py, CONVECTION).

gmg pressure solves: the temperature and pressure fields of every sample are
bit-identical to the reference's (the solver's iterates are; only the
residual norms differ in the last ulps). gmg_pcg: the CG scalars come from
tree sums instead of sequential ones, so fields agree to
rounding and the step statistics exactly.
"""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
EXE = ROOT / "oracle" / "_ref" / "convection_gpu"


def _run(stem):
    if not EXE.exists():
        pytest.skip("oracle/_ref/convection_gpu not built (needs /root/reference at build time)")
    g = json.loads((GOLDEN / f"{stem}.json").read_text())
    run = subprocess.run([str(EXE), *g["_argv"]], capture_output=True, text=True, timeout=900)
    assert run.returncode == 0, run.stderr
    return json.loads(run.stdout), g


@pytest.mark.parametrize("stem", ["convection_32_gs_w33", "convection_32_jacobi_v22", "convection_64_sgs_f21",
                                  "convection_256_gs_w33"])
def test_convection_gmg_bitwise(stem):
    out, g = _run(stem)
    for key in ("n", "accepted", "rejected", "rhs_evaluations", "pressure_solves"):
        assert out[key] == g[key], key
    assert len(out["samples"]) == len(g["samples"])
    for so, sg in zip(out["samples"], g["samples"]):
        assert so["t"] == sg["t"]
        assert so["fnv_T"] == sg["fnv_T"], f"temperature at t={so['t']} differs from the reference's"
        assert so["fnv_P"] == sg["fnv_P"], f"pressure at t={so['t']} differs from the reference's"
    np.testing.assert_allclose(out["max_pressure_residual"], g["max_pressure_residual"], rtol=1e-10)
    # ||delta q|| / ||rhs||: the reference's own host arithmetic on identical fields
    assert out["max_relative_divergence"] == g["max_relative_divergence"]


def test_convection_gmg_pcg():
    out, g = _run("convection_32_pcg")
    for key in ("n", "accepted", "rejected", "rhs_evaluations", "pressure_solves"):
        assert out[key] == g[key], key
    for so, sg in zip(out["samples"], g["samples"]):
        assert so["t"] == sg["t"]
        for key in ("T_mid", "P_mid", "T_absmax", "P_absmax"):
            np.testing.assert_allclose(so[key], sg[key], rtol=1e-9, err_msg=key)
    assert out["max_pressure_residual"] <= 1e-8
