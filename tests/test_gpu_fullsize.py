"""GPU parity at the BASELINE configs' FULL sizes.

The per-point kernels at 10M x 100 and 1M x 1000 run their real grid-stride
schedule (all tiles, all CTAs) over device-generated inputs; the output is
checked against the C oracle on a subsample of every 997th point (the
per-point results are independent, so a subsample is a complete check of the
points it covers).  The 1e8-bin chi2 pass (4651 tiles, 96 chunks, the
layout the bench times) is checked over EVERY bin against the compensated
restatement of fit.cpp:206-259, and through size-independent properties:
linearity of the accumulate-only slots (two launches == 2x one launch up to
one rounding), and the chi2 value of the multi-candidate pass equal bit for
bit to the single pass.

Tolerances: per-point 1e-12 relative per component; reductions
1e-12 * sum_j |w_j dm_j/dq_i| (the summation-order change).
"""
import numpy as np
import pytest

from conftest import rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402

REL = 1e-12
STRIDE = 997


def _points(dim, n, spread, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    p = torch.rand((dim, n), dtype=torch.float64, device="cuda", generator=g) * 4 - 2
    x = p + spread * torch.randn((dim, n), dtype=torch.float64, device="cuda", generator=g)
    return x, p


def _check_subsample(restate, x, p, dx, dp, stride=STRIDE):
    idx = torch.arange(0, x.shape[1], stride, device="cuda")
    xs, ps, dxs, dps = (t[:, idx].cpu().numpy() for t in (x, p, dx, dp))
    rdx, rdp = np.zeros_like(xs), np.zeros_like(xs)
    restate.gaussnd_grad(np.ascontiguousarray(xs), np.ascontiguousarray(ps), 1.3, rdx, rdp)
    assert rel_err(dxs, rdx).max() <= REL
    assert rel_err(dps, rdp).max() <= REL
    return xs.shape[1]


@pytest.mark.parametrize("dim,n,spread", [(100, 10_000_000, 0.1), (1000, 1_000_000, 0.03)],
                         ids=["cfg2_d100_10M", "cfg4_d1000_1M"])
def test_gaussnd_full_size_subsample(restate, dim, n, spread):
    x, p = _points(dim, n, spread, seed=2024 + dim)
    dx, dp = torch.zeros_like(x), torch.zeros_like(x)
    adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, dx, dp)
    torch.cuda.synchronize()
    checked = _check_subsample(restate, x, p, dx, dp)
    assert checked == (n + STRIDE - 1) // STRIDE
    # accumulate-only slots at full size: a second launch adds the same
    # gradient again (x + x is exact, so the sums are exactly 2x)
    once = dx[:, ::STRIDE].clone(), dp[:, ::STRIDE].clone()
    adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, dx, dp)
    torch.cuda.synchronize()
    assert torch.equal(dx[:, ::STRIDE], 2 * once[0])
    assert torch.equal(dp[:, ::STRIDE], 2 * once[1])
    # the tail of the last tile (points not covered by the stride) too
    tail = slice(n - 300, n)
    xs, ps = x[:, tail].cpu().numpy(), p[:, tail].cpu().numpy()
    rdx, rdp = np.zeros_like(xs), np.zeros_like(xs)
    restate.gaussnd_grad(np.ascontiguousarray(xs), np.ascontiguousarray(ps), 1.3, rdx, rdp)
    assert rel_err(dx[:, tail].cpu().numpy(), 2 * rdx).max() <= 2 * REL
    assert rel_err(dp[:, tail].cpu().numpy(), 2 * rdp).max() <= 2 * REL


def test_gauss1d_1M_every_point(restate):
    n = 1_000_000
    x, p = synth.points_1d(n, seed=0x5EED)
    X, P = torch.from_numpy(x).cuda(), torch.from_numpy(p).cuda()
    dx = torch.zeros(n, dtype=torch.float64, device="cuda")
    dp = torch.zeros_like(dx)
    st = adc.launch("compute", adc.LaunchConfig(n // 256 + 1, 256, n),
                    adc.BufferSet(arrays={"x": X, "p": P, "dx": dx, "dp": dp},
                                  scalars={"sigma": 1.3}))
    assert st.active == n
    rdx, rdp = np.zeros(n), np.zeros(n)
    restate.gauss_grad(x, p, 1.3, rdx, rdp)
    assert rel_err(dx.cpu().numpy(), rdx).max() <= REL
    assert rel_err(dp.cpu().numpy(), rdp).max() <= REL


@pytest.fixture(scope="module")
def hist_1e8():
    bins = 100_000_000
    h = adc.sample_histogram("gpoly", synth.GPOLY_TRUTH, bins, -5.0, 5.0, bins * 100.0, seed=77,
                             zero_every=100, device="cuda")
    yield h, h.counts.cpu().numpy()
    del h
    torch.cuda.empty_cache()


def test_chi2_1e8_gradient_every_bin(restate, hist_1e8):
    h, counts = hist_1e8
    assert np.all(counts[::100] == 0.0) and counts.sum() == h.events
    q = list(synth.GPOLY_INIT)
    plan = adc.Chi2Plan("gpoly", 6, h)
    assert plan.layout.nchunks > 64  # the multi-chunk layout the bench times
    g, c2 = plan.gradient(q)
    ref, scale = restate.chi2_gradient_compensated("gpoly", counts, -5.0, 5.0, h.events, q)
    assert np.all(np.abs(np.asarray(g) - ref) <= REL * scale), (g, ref)
    cref, cscale = restate.chi2_compensated("gpoly", counts, -5.0, 5.0, h.events, q)
    assert abs(c2 - cref) <= REL * cscale
    # the value pass (line search) within the same bound; the batched
    # line-search pass equal to it bit for bit
    v = plan.chi2(q)
    assert abs(v - cref) <= REL * cscale
    qs = np.array([q, [qi * 0.999 for qi in q]])
    vm = plan.chi2_multi(qs)
    assert vm[0] == v
    assert vm[1] == plan.chi2(list(qs[1]))
    plan.close()


def test_chi2_1e8_numeric_provider(restate, hist_1e8):
    h, counts = hist_1e8
    q = list(synth.GPOLY_INIT)
    plan = adc.Chi2Plan("gpoly", 6, h)
    plan.set_provider(adc.GradientProvider.Numeric)
    g, _ = plan.gradient(q)
    ref, scale, fd = restate.chi2_gradient_numeric_compensated("gpoly", counts, -5.0, 5.0,
                                                               h.events, q)
    assert np.all(np.abs(np.asarray(g) - ref) <= REL * scale + 16 * fd)
    plan.close()
