"""The sweeps divide by a row's diagonal with the reciprocal refined once per
row (rowkernels.cuh div_seed / div_rn) instead of __ddiv_rn per right-hand
side. tools/check_div.cu compares the two bit for bit on the GPU over random
bit patterns, the V-cycle's value ranges and crossed special values."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def test_shared_divisor_division_is_ddiv_rn(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "check_div"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false", "-O3", "-std=c++17",
                    "-o", str(exe), str(ROOT / "tools" / "check_div.cu")], check=True, timeout=300)
    out = subprocess.run([str(exe), str(1 << 31)], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mismatches 0 of" in out.stdout
