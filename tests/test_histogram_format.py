"""The histogram ingest format (include/adc_cuda.h "ADCHIST1"; the
reference's Histogram, fit.hpp:23-34, on disk): written and read by the
product (host and device counts), read independently by the oracle (numpy in
oracle/restate_lib.py, and ref_tool chi2-file, which feeds the file to the
reference's own chi2 / chi2_gradient formula)."""
import os
import subprocess

import numpy as np
import pytest

from conftest import REF_TOOL

import paper_2203_06139_b200 as adc  # noqa: E402
from oracle import restate_lib  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402


def test_write_then_read_host(tmp_path):
    counts, ev = synth.histogram(5000, events=1e6, seed=9)
    h = adc.Histogram(5000, -5.0, 5.0, ev, counts)
    path = str(tmp_path / "h.adchist")
    h.save(path)
    bins, lo, hi, events, c = restate_lib.read_histogram(path)
    assert (bins, lo, hi, events) == (5000, -5.0, 5.0, ev)
    assert c.tobytes() == counts.tobytes()
    assert os.path.getsize(path) == 40 + 8 * 5000
    back = adc.Histogram.load(path)
    assert (back.bins, back.lo, back.hi, back.events) == (5000, -5.0, 5.0, ev)
    assert back.counts.tobytes() == counts.tobytes()


def test_bad_files_are_arg_errors(tmp_path):
    p = tmp_path / "bad.adchist"
    p.write_bytes(b"NOTAHIST" + bytes(40))
    with pytest.raises(adc.AdcError) as e:
        adc.Histogram.load(str(p))
    assert e.value.kind == "Arg" and "ADCHIST1" in str(e.value)
    good = tmp_path / "short.adchist"
    adc.Histogram(10, 0.0, 1.0, 45.0, np.arange(10.0)).save(str(good))
    good.write_bytes(good.read_bytes()[:-8])
    with pytest.raises(adc.AdcError) as e:
        adc.Histogram.load(str(good))
    assert e.value.kind == "Arg"


@pytest.mark.skipif(not os.path.exists(REF_TOOL), reason="ref_tool not built")
def test_reference_reads_the_same_file(tmp_path):
    """ref_tool chi2-file (the reference's formula on the file's histogram)
    equals ref_tool chi2-in on the raw counts: the format carries the
    reference's Histogram exactly."""
    counts, ev = synth.histogram(3000, events=3e5, seed=4)
    path = str(tmp_path / "h.adchist")
    adc.Histogram(3000, -5.0, 5.0, ev, counts).save(path)
    q = [str(v) for v in synth.GPOLY_INIT]
    out1, out2, raw = (str(tmp_path / n) for n in ("o1.bin", "o2.bin", "c.bin"))
    subprocess.run([REF_TOOL, "chi2-file", "gpoly", path, out1, *q], check=True,
                   capture_output=True)
    counts.tofile(raw)
    subprocess.run([REF_TOOL, "chi2-in", "gpoly", "3000", "-5", "5", raw, out2, "1", *q],
                   check=True, capture_output=True)
    assert np.fromfile(out1).tobytes() == np.fromfile(out2).tobytes()


@pytest.mark.gpu
def test_device_histogram_round_trip(tmp_path, restate):
    import torch
    h = adc.sample_histogram("gpoly", synth.GPOLY_TRUTH, 2_000_003, -5.0, 5.0, 2e8, seed=8,
                             zero_every=100, device="cuda")
    path = str(tmp_path / "d.adchist")
    h.save(path)  # device counts: pinned pieces
    _, _, _, events, c = restate_lib.read_histogram(path)
    assert events == h.events and c.tobytes() == h.counts.cpu().numpy().tobytes()
    back = adc.Histogram.load(path, device="cuda")
    assert torch.equal(back.counts, h.counts)
    q = list(synth.GPOLY_INIT)
    g0, c0 = adc.Chi2Plan("gpoly", 6, h).gradient(q)
    g1, c1 = adc.Chi2Plan("gpoly", 6, back).gradient(q)
    assert np.asarray(g0).tobytes() == np.asarray(g1).tobytes() and c0 == c1
