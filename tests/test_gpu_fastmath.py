"""The kernel's branch-free float64 division / square root (csrc/dg_fastmath.cuh)
are bit-identical to the IEEE operators over the operand range the step uses
(2^-40 .. 2^40, exact integers, zeros): 2^30 random pairs per run."""

from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_ddiv_dsqrt_bitwise(tmp_path):
    exe = tmp_path / "divsqrt_check"
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                    "-fmad=false", "-o", str(exe), str(ROOT / "tools/microbench/divsqrt_check.cu")],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    first = out.splitlines()[0]
    assert "ddiv mismatches 0, dsqrt mismatches 0" in first, out
