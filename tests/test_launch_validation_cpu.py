"""Argument validation of the Python mirror (launch.py) before any device call
(ADVICE r01): every SoA buffer has x's (dim, n) shape, the shared-mean p / dp
are long enough, host and device buffers are never mixed, and the registry is
keyed by the fingerprint of the printed gradient when the module text is
supplied.  No GPU needed: each case raises before the C ABI is reached."""
import json
import os

import numpy as np
import pytest

import paper_2203_06139_b200 as adc
import importlib
L = importlib.import_module("paper_2203_06139_b200.launch")

from conftest import GOLDEN


def _soa(dim, n):
    return np.zeros((dim, n))


def test_launch_batch_rejects_short_slot_buffers():
    x, p = _soa(5, 100), _soa(5, 100)
    with pytest.raises(adc.AdcError) as e:
        adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, _soa(5, 100), _soa(4, 100))
    assert e.value.kind == "Launch" and "buffer 'dp' has shape (4, 100)" in str(e.value)
    with pytest.raises(adc.AdcError) as e:
        adc.launch_batch("gaussnd_grad_0_1", x, _soa(5, 99), 1.3, _soa(5, 100), _soa(5, 100))
    assert "buffer 'p'" in str(e.value)


def test_launch_batch_rejects_mixed_host_and_torch():
    torch = pytest.importorskip("torch")
    x = _soa(3, 10)
    with pytest.raises(adc.AdcError) as e:
        adc.launch_batch("gaussnd_grad_0_1", x, torch.zeros(3, 10, dtype=torch.float64), 1.3,
                         _soa(3, 10), _soa(3, 10))
    assert e.value.kind == "Launch"


def test_launch_rejects_cpu_torch_tensors():
    torch = pytest.importorskip("torch")
    n = 64
    arr = {k: torch.zeros(n, dtype=torch.float64) for k in ("x", "p", "dx", "dp")}
    with pytest.raises(adc.AdcError) as e:
        adc.launch("compute", adc.LaunchConfig(1, 64, n),
                   adc.BufferSet(arrays=arr, scalars={"sigma": 1.3}))
    assert e.value.kind == "Launch"


def test_launch_short_buffer_message_is_the_reference_one():
    n = 100
    arr = {k: np.zeros(n) for k in ("x", "p", "dx")}
    arr["dp"] = np.zeros(n - 1)
    with pytest.raises(adc.AdcError) as e:
        adc.launch("compute", adc.LaunchConfig(1, 128, n),
                   adc.BufferSet(arrays=arr, scalars={"sigma": 1.3}))
    # launch.cpp:281-284
    assert "buffer 'dp' has length 99 but is indexed by thread over 100 elements" in str(e.value)


def test_printed_gradient_fingerprint_is_the_registry_key():
    """The printed gauss_grad_0_1 cut out of the reference-printed module
    hashes to the fingerprint the reference-side bridge computes
    (tests/golden/gradient_fingerprints.json, written by the reference)."""
    module = str(np.load(os.path.join(GOLDEN, "jit_cases.npz"))["module"])
    fps = json.load(open(os.path.join(GOLDEN, "gradient_fingerprints.json")))
    text = L.printed_function(module, "gauss_grad_0_1")
    assert text.startswith("device host void gauss_grad_0_1(") and text.endswith("}\n")
    assert L.fingerprint_of(text) == int(fps["gauss_grad_0_1"], 16)
    # a changed generated gradient is a registry miss: Error(Launch)
    bad = module.replace("_d_p[0] += -_r5;", "_d_p[0] += _r5;")
    arr = {k: np.zeros(8) for k in ("x", "p", "dx", "dp")}
    with pytest.raises(adc.AdcError) as e:
        adc.launch("compute", adc.LaunchConfig(1, 8, 8),
                   adc.BufferSet(arrays=arr, scalars={"sigma": 1.3}), module=bad)
    assert e.value.kind == "Launch"
