"""Drop-in integration: the reference-side binding (integration/adc_b200_bridge.cpp)
compiled against the UNMODIFIED reference library (oracle/_ref/libadc.a) and
the product's C ABI, and the header-only C++ mirror (include/adcx/adc_b200.hpp).
The CPU tests check the error contract (the reference's messages, refusal,
no CPU fallback); the GPU tests check parity of the bridged calls against the
reference's own adc::launch / FitEngine on the same inputs."""
import os
import subprocess

import pytest

from conftest import ROOT

BRIDGE = os.path.join(ROOT, "oracle", "_ref", "bridge_check")
LIBDIR = os.path.join(ROOT, "paper_2203_06139_b200")


def _run(args):
    r = subprocess.run(args, capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout + r.stderr


@pytest.fixture(scope="module")
def cxx_check(tmp_path_factory):
    exe = tmp_path_factory.mktemp("cxx") / "cxx_api_check"
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "restate"], check=True)
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(ROOT, "oracle"),
                    os.path.join(ROOT, "tests", "cpu", "cxx_api_check.cpp"),
                    os.path.join(ROOT, "oracle", "restate.c"), "-x", "none",
                    "-L", LIBDIR, "-ladc_b200", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe), "-lpthread"],
                   check=True)
    return str(exe)


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_cxx_mirror_error_contract(cxx_check):
    rc, out = _run([cxx_check, "gpu" if _has_gpu() else "cpu"])
    assert rc == 0, out


@pytest.mark.skipif(not os.path.exists(BRIDGE), reason="bridge_check not built (needs /root/reference)")
def test_bridge_error_contract():
    rc, out = _run([BRIDGE, "cpu"])
    assert rc == 0, out


@pytest.mark.gpu
def test_cxx_mirror_gpu(cxx_check):
    rc, out = _run([cxx_check, "gpu"])
    assert rc == 0, out


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BRIDGE), reason="bridge_check not built (needs /root/reference)")
def test_bridge_gpu_parity_with_reference():
    rc, out = _run([BRIDGE, "gpu"])
    print(out)
    assert rc == 0, out
