"""Pins the plain-C oracle (oracle/restate.c) to the reference itself: every
golden fixture was written by the unmodified reference library
(tests/golden/make_golden.py -> oracle/_ref/ref_tool).  CPU only."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, rel_err


def test_gauss_grad_kat(restate):
    # test_reverse.cpp:69-82: gauss(1,0,1) -> dx = -0.2419707245191434 = -dp.
    g = golden("gauss1d_cases.npz")
    x, p = g["kat_x"].copy(), g["kat_p"].copy()
    dx, dp = np.zeros(1), np.zeros(1)
    restate.gauss_grad(x, p, 1.0, dx, dp)
    assert dx[0] == g["kat_dx"][0] and dp[0] == g["kat_dp"][0]
    assert abs(dx[0] - -0.2419707245191434) < 1e-16 and dx[0] == -dp[0]


def test_gauss_grad_listing1_bitexact(restate):
    # acceptance.cpp:160-211 analog: N=512, seed 0x5EED, sigma 1.3.
    g = golden("gauss1d_n512.npz")
    dx, dp = np.zeros(512), np.zeros(512)
    restate.gauss_grad(g["x"], g["p"], float(g["sigma"]), dx, dp)
    assert np.array_equal(dx, g["dx"]) and np.array_equal(dp, g["dp"])
    assert int(g["active"]) == 512 and int(g["idle"]) == 256


@pytest.mark.parametrize("case", ["accum300", "edges"])
def test_gauss_grad_accumulate_bitexact(restate, case):
    g = golden("gauss1d_cases.npz")
    dx, dp = g[f"{case}_dx0"].copy(), g[f"{case}_dp0"].copy()
    restate.gauss_grad(g[f"{case}_x"], g[f"{case}_p"], float(g[f"{case}_sigma"]), dx, dp)
    # bit-exact including the sign of zero
    assert dx.tobytes() == g[f"{case}_dx"].tobytes()
    assert dp.tobytes() == g[f"{case}_dp"].tobytes()


@pytest.mark.parametrize("key", ["d100_n64", "d1000_n8", "d1_n33", "d37_n70", "d128_n40",
                                 "d129_n5"])
def test_gaussnd_grad_bitexact(restate, key):
    g = golden("gaussnd_cases.npz")
    dx, dp = g[f"{key}_dx0"].copy(), g[f"{key}_dp0"].copy()
    restate.gaussnd_grad(g[f"{key}_x"], g[f"{key}_p"], float(g[f"{key}_sigma"]), dx, dp)
    assert dx.tobytes() == g[f"{key}_dx"].tobytes()
    assert dp.tobytes() == g[f"{key}_dp"].tobytes()


@pytest.mark.parametrize("key", ["gpoly_b2000", "gsum1_b1000", "gsum2_b1500"])
def test_chi2_bitexact_and_compensated(restate, key):
    g = golden("chi2_cases.npz")
    model = str(g[f"{key}_model"])
    counts, q, ev = g[f"{key}_counts"], g[f"{key}_q"], float(g[f"{key}_events"])
    # The sequential restatement is the reference's own arithmetic: bit-exact.
    assert restate.chi2(model, counts, -5.0, 5.0, ev, q) == g[f"{key}_chi2"]
    assert np.array_equal(restate.chi2_gradient(model, counts, -5.0, 5.0, ev, q), g[f"{key}_grad"])
    # The compensated variant (accuracy reference for reordered GPU sums)
    # differs from the sequential sums by rounding only.
    gc, scale = restate.chi2_gradient_compensated(model, counts, -5.0, 5.0, ev, q)
    assert np.all(np.abs(gc - g[f"{key}_grad"]) <= 1e-12 * scale)
    vc, vscale = restate.chi2_compensated(model, counts, -5.0, 5.0, ev, q)
    assert abs(vc - g[f"{key}_chi2"]) <= 1e-12 * vscale


def test_fingerprints_file():
    with open(os.path.join(GOLDEN, "gradient_fingerprints.json")) as fh:
        fps = json.load(fh)
    assert set(fps) == {"gauss_grad", "gauss_grad_0_1", "gaussnd_grad_0_1", "gpoly_grad_1",
                        "gsum_grad_1"}


@pytest.mark.parametrize("case", ["n100", "n4097"])
def test_gauss_shared_sequential_bitexact(restate, case):
    # compute_shared forced sequential (test_launch.cpp:148-153): the restatement
    # is the reference's own arithmetic and order, bit for bit.
    g = golden("gauss_shared_cases.npz")
    dx, dp, ds = g[f"{case}_dx0"].copy(), g[f"{case}_dp0"].copy(), g[f"{case}_dsigma0"].copy()
    restate.gauss_grad_shared(g[f"{case}_x"], g[f"{case}_p"], float(g[f"{case}_sigma"]), dx, dp, ds)
    assert dx.tobytes() == g[f"{case}_dx"].tobytes()
    assert dp.tobytes() == g[f"{case}_dp"].tobytes()
    assert ds.tobytes() == g[f"{case}_dsigma"].tobytes()
    tot, scale = restate.gauss_shared_dsigma_compensated(g[f"{case}_x"], g[f"{case}_p"],
                                                         float(g[f"{case}_sigma"]))
    assert abs((g[f"{case}_dsigma0"][0] + tot) - g[f"{case}_dsigma"][0]) <= 1e-12 * (scale + 0.25)


@pytest.mark.parametrize("key", ["gpoly_b2000", "gsum1_b1000", "gsum2_b1500"])
def test_chi2_numeric_provider_bitexact(restate, key):
    # GradientProvider::Numeric (fit.cpp:187-190, central_gradient numdiff.cpp:38-87):
    # the reference's value for gsum comes from the unmodified FitEngine.
    g = golden("chi2_numeric_cases.npz")
    model = str(g[f"{key}_model"])
    counts, q, ev = g[f"{key}_counts"], g[f"{key}_q"], float(g[f"{key}_events"])
    assert np.array_equal(restate.chi2_gradient_numeric(model, counts, -5.0, 5.0, ev, q),
                          g[f"{key}_grad"])
    gc, scale, fd = restate.chi2_gradient_numeric_compensated(model, counts, -5.0, 5.0, ev, q)
    assert np.all(np.abs(gc - g[f"{key}_grad"]) <= 1e-12 * scale)
    assert np.all(fd > 0) and np.all(fd < 1e-6 * scale)
    # numeric and AD agree to finite-difference accuracy (test_fit.cpp:62-79: 1e-6)
    ad, _ = restate.chi2_gradient_compensated(model, counts, -5.0, 5.0, ev, q)
    assert np.all(np.abs(gc - ad) <= 1e-6 * scale)


@pytest.mark.parametrize("key", ["d100_n64", "d37_n150", "d1_n40", "d300_n33"])
def test_gaussnd_shared_p_bitexact(restate, key):
    # one p and one dp slot for every point, points in order: the reference's
    # Program::eval run sequentially (ref_tool gaussnd-shared-p-in)
    g = golden("gaussnd_shared_p_cases.npz")
    dx, dp = g[f"{key}_dx0"].copy(), g[f"{key}_dp0"].copy()
    restate.gaussnd_grad_shared_p(np.ascontiguousarray(g[f"{key}_x"]), g[f"{key}_p"], 1.3, dx, dp)
    assert dx.tobytes() == g[f"{key}_dx"].tobytes()
    assert dp.tobytes() == g[f"{key}_dp"].tobytes()
