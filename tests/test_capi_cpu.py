"""CPU-only checks of the C ABI boundary: the library loads, exports every
symbol include/adc_cuda.h declares, validates arguments like the reference,
keeps the registry in sync with the reference's generated gradients, and
refuses to compute without a GPU (no CPU fallback)."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

import paper_2203_06139_b200 as adc
from paper_2203_06139_b200 import _capi

HEADER = os.path.join(ROOT, "include", "adc_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(adc_(?:cuda|chi2|fit|nccl|comm|jit|histogram)_\w+)\s*\(", text)))


def test_every_declared_symbol_is_exported_and_bound():
    syms = declared_symbols()
    assert len(syms) >= 25
    lib = ctypes.CDLL(_capi.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_capi.SIGNATURES), set(syms) ^ set(_capi.SIGNATURES)
    assert _capi.lib.adc_cuda_abi_version() == 1


def test_registry_matches_reference_fingerprints():
    with open(os.path.join(GOLDEN, "gradient_fingerprints.json")) as fh:
        fps = {k: int(v, 16) for k, v in json.load(fh).items()}
    lib = _capi.lib
    names = {lib.adc_cuda_registry_name(i).decode(): lib.adc_cuda_registry_fingerprint(i)
             for i in range(lib.adc_cuda_registry_size())}
    assert names == fps
    for name, fp in fps.items():
        assert adc.registry_find(name, fp) >= 0
    with pytest.raises(adc.AdcError) as e:
        adc.registry_find("gauss_grad_0_1", fps["gauss_grad_0_1"] ^ 1)
    assert e.value.kind == "Launch" and "differs" in str(e.value)
    with pytest.raises(adc.AdcError) as e:
        adc.registry_find("poly_grad", 0)
    assert e.value.kind == "Launch" and "no B200 kernel registered for 'poly_grad'" in str(e.value)


def test_fingerprint_is_fnv1a64():
    assert _capi.lib.adc_cuda_fingerprint(b"", 0) == 0xCBF29CE484222325
    assert _capi.lib.adc_cuda_fingerprint(b"a", 1) == 0xAF63DC4C8601EC8C


@pytest.mark.parametrize("grid,block,n,msg", [
    (0, 256, 512, "launch configuration must be positive (grid 0, block 256, n 512)"),
    (1, 256, 512, "grid 1 x block 256 does not cover problem size 512"),
])
def test_config_validation_messages(grid, block, n, msg):
    # LaunchConfig::validate, launch.cpp:9-19 — checked before any device use.
    rc = _capi.lib.adc_cuda_compute_gauss(grid, block, n, None, None, 1.0, None, None, None)
    assert rc == 4 and _capi.lib.adc_cuda_last_error().decode() == msg
    with pytest.raises(adc.AdcError) as e:
        adc.LaunchConfig(grid, block, n).validate()
    assert str(e.value) == msg and e.value.kind == "Launch"


def test_buffer_validation_messages():
    # launch.cpp:271-284 messages (test_launch.cpp:168-182).
    b = adc.BufferSet(arrays={"x": np.zeros(10), "p": np.zeros(512), "dx": np.zeros(512),
                              "dp": np.zeros(512)}, scalars={"sigma": 1.0})
    with pytest.raises(adc.AdcError, match="length"):
        adc.launch("compute", adc.LaunchConfig(3, 256, 512), b)
    del b.arrays["x"]
    with pytest.raises(adc.AdcError, match="missing buffer 'x'"):
        adc.launch("compute", adc.LaunchConfig(3, 256, 512), b)


def test_hazardous_kernel_refused():
    # launch.cpp:261-267 / acceptance criterion 6.
    b = adc.BufferSet()
    with pytest.raises(adc.AdcError) as e:
        adc.launch("compute_shared", adc.LaunchConfig(1, 32, 32), b)
    assert e.value.kind == "Launch" and "launch refused" in str(e.value)


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    x = np.zeros(8)
    rc = _capi.lib.adc_cuda_compute_gauss_host(1, 8, 8, x.ctypes.data, x.ctypes.data, 1.0,
                                               x.ctypes.data, x.ctypes.data)
    assert rc == 6 and "no CUDA device" in _capi.lib.adc_cuda_last_error().decode()
    rc = _capi.lib.adc_cuda_gaussnd_grad_host(8, 1, 8, x.ctypes.data, x.ctypes.data, 1.0,
                                              x.ctypes.data, x.ctypes.data)
    assert rc == 6


def test_chi2_layout_shards_whole_chunks():
    for bins in (1, 1000, 10**6, (1 << 22) + 5, 10**8):
        L1 = adc.chi2_layout(bins)
        assert L1.bin_begin == 0 and L1.bin_end == bins and L1.chunk_end == L1.nchunks
        chunk_bins = L1.tile_bins * L1.chunk_tiles
        assert (L1.nchunks - 1) * chunk_bins < bins <= L1.nchunks * chunk_bins
        for world in (2, 3, 4, 8):
            spans = [adc.chi2_layout(bins, world, r) for r in range(world)]
            assert spans[0].bin_begin == 0 and spans[-1].bin_end == bins
            for a, b in zip(spans, spans[1:]):
                assert a.chunk_end == b.chunk_begin and a.bin_end == b.bin_begin
                assert a.bin_end == min(bins, a.chunk_end * chunk_bins)
    L = adc.chi2_layout(10**8)
    # 84 bins per thread: 4651 tiles = 15.7 waves of 296 CTAs on one GPU, and
    # at most 12 chunks x 49 tiles = 588 tiles = 1.99 waves per rank on eight
    assert L.tile_bins == 84 * 256 and L.chunk_tiles == 49 and L.nchunks == 95
    per_rank = [(lambda s: (s.chunk_end - s.chunk_begin) * L.chunk_tiles)(
        adc.chi2_layout(10**8, 8, r)) for r in range(8)]
    assert max(per_rank) <= 2 * 296


def test_host_communicator_without_device():
    # The host transport needs no device; compute still refuses without one.
    import paper_2203_06139_b200 as adc
    comm = adc.Comm.host(3, 2, lambda a: np.tile(a, 3))
    assert comm.info() == (3, 2, 2)
    with pytest.raises(adc.AdcError) as e:
        adc.Comm.host(2, 2, lambda a: a)
    assert e.value.kind == "Arg"
    rc = _capi.lib.adc_cuda_chi2_plan_set_comm(None, comm._p)
    assert rc == 7
    comm.close()
