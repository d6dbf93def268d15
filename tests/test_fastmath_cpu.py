"""The chi2 fast-mode exp (csrc/fastmath.cuh is __host__ __device__) compiled
for the host and checked against glibc exp: <= 1 ulp (measured; bound checked at 1.5) over [-745, 0],
correct subnormals.  CPU only."""
import os
import subprocess

from conftest import ROOT


def test_exp_nonpos_ulp(tmp_path):
    exe = tmp_path / "fastmath_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off",
                    "-I", os.path.join(ROOT, "paper_2203_06139_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpu", "fastmath_check.cpp"), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "max ulp" in out.stdout
