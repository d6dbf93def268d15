import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def restate():
    """The plain-C oracle (oracle/restate.c), built on demand with gcc."""
    from oracle import restate_lib
    return restate_lib.load()


def rel_err(a, b, floor=1e-300):
    """True relative difference per component: |a-b| / max(|a|,|b|)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
    return np.abs(a - b) / den


def pytest_collection_modifyitems(config, items):
    """GPU tests need a CUDA device; without one they are skipped, not failed
    (the driver runs `-m "not gpu"` here and `-m gpu` on a B200)."""
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
