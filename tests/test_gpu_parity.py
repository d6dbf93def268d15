"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the C oracle.  Tolerances:
  * per-point outputs: |g - r| <= 1e-12 * max(|g|, |r|)  (true relative)
  * reductions (chi2, its gradient): |g - r| <= 1e-12 * sum_j |term_j|
    against the Neumaier-compensated restatement of fit.cpp:206-259.
"""
import numpy as np
import pytest

from conftest import golden, rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402
from paper_2203_06139_b200.launch import set_gaussnd_variant  # noqa: E402

REL = 1e-12
DEV = "cuda"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def host(a):
    torch.cuda.synchronize()
    return a.cpu().numpy()


# ---------------------------------------------------------------------------- K1
def test_listing1_n512_device_and_host():
    g = golden("gauss1d_n512.npz")
    for path in ("device", "host"):
        if path == "device":
            x, p = t(g["x"]), t(g["p"])
            dx, dp = torch.zeros(512, dtype=torch.float64, device=DEV), torch.zeros(
                512, dtype=torch.float64, device=DEV)
        else:
            x, p = g["x"].copy(), g["p"].copy()
            dx, dp = np.zeros(512), np.zeros(512)
        st = adc.launch("compute", adc.LaunchConfig(512 // 256 + 1, 256, 512),
                        adc.BufferSet(arrays={"x": x, "p": p, "dx": dx, "dp": dp},
                                      scalars={"sigma": 1.3}))
        assert st.active == 512 and st.idle == 256 and st.thread_statements.size == 768
        gx = host(dx) if path == "device" else dx
        gp = host(dp) if path == "device" else dp
        assert rel_err(gx, g["dx"]).max() <= REL
        assert rel_err(gp, g["dp"]).max() <= REL
        assert np.array_equal(gx, -gp)  # dx == -dp exactly from zero slots
        # most components are bit-identical (exp may round differently by 1 ulp)
        assert np.mean(gx == g["dx"]) > 0.9


@pytest.mark.parametrize("case", ["kat", "accum300", "edges"])
def test_listing1_cases(case):
    g = golden("gauss1d_cases.npz")
    n = g[f"{case}_x"].size
    block = int(g[f"{case}_block"])
    dx, dp = t(g[f"{case}_dx0"]), t(g[f"{case}_dp0"])
    adc.launch("compute", adc.LaunchConfig(n // block + 1, block, n),
               adc.BufferSet(arrays={"x": t(g[f"{case}_x"]), "p": t(g[f"{case}_p"]), "dx": dx,
                                     "dp": dp}, scalars={"sigma": float(g[f"{case}_sigma"])}))
    assert acc_err(host(dx), g[f"{case}_dx"], g[f"{case}_dx0"]).max() <= REL
    assert acc_err(host(dp), g[f"{case}_dp"], g[f"{case}_dp0"]).max() <= REL
    if case == "kat":
        assert host(dx)[0] == pytest.approx(-0.2419707245191434, rel=1e-15)


def acc_err(g, r, init):
    """Accumulated slots: the increment is compared relative to the larger of
    the result and the initial slot value (a 1-ulp difference in the increment
    is amplified by cancellation against the slot otherwise)."""
    g, r, init = (np.asarray(a, dtype=np.float64) for a in (g, r, init))
    den = np.maximum(np.maximum(np.abs(g), np.abs(r)), np.abs(init))
    return np.abs(g - r) / np.maximum(den, 1e-300)


def test_listing1_1m_vs_oracle(restate):
    n = 10**6
    x, p = synth.points_1d(n)
    dx0 = np.random.default_rng(3).standard_normal(n)
    dp0 = np.random.default_rng(4).standard_normal(n)
    ox, op = dx0.copy(), dp0.copy()
    restate.gauss_grad(x, p, 1.3, ox, op)
    dx, dp = t(dx0), t(dp0)
    adc.launch("compute", adc.LaunchConfig(n // 256 + 1, 256, n),
               adc.BufferSet(arrays={"x": t(x), "p": t(p), "dx": dx, "dp": dp},
                             scalars={"sigma": 1.3}))
    assert acc_err(host(dx), ox, dx0).max() <= REL and acc_err(host(dp), op, dp0).max() <= REL
    # odd length + unaligned views take the scalar path
    dx2 = torch.zeros(n + 1, dtype=torch.float64, device=DEV)
    dp2 = torch.zeros(n + 1, dtype=torch.float64, device=DEV)
    xs, ps = t(np.concatenate([[0.0], x])), t(np.concatenate([[0.0], p]))
    m = n - 1
    adc.launch("compute", adc.LaunchConfig(m // 256 + 1, 256, m),
               adc.BufferSet(arrays={"x": xs[1:1 + m], "p": ps[1:1 + m], "dx": dx2[1:1 + m],
                                     "dp": dp2[1:1 + m]}, scalars={"sigma": 1.3}))
    ox2, op2 = np.zeros(m), np.zeros(m)
    restate.gauss_grad(x[:m].copy(), p[:m].copy(), 1.3, ox2, op2)
    assert rel_err(host(dx2)[1:1 + m], ox2).max() <= REL


def test_listing1_domain_error():
    z = torch.zeros(4, dtype=torch.float64, device=DEV)
    with pytest.raises(adc.AdcError) as e:
        adc.launch("compute", adc.LaunchConfig(1, 4, 4),
                   adc.BufferSet(arrays={"x": z, "p": z, "dx": z, "dp": z}, scalars={"sigma": 0.0}))
    assert e.value.kind == "Eval" and "division by zero" in str(e.value)


# ---------------------------------------------------------------------------- K2
ND_KEYS = ["d100_n64", "d1000_n8", "d1_n33", "d37_n70", "d128_n40", "d129_n5"]


@pytest.mark.parametrize("variant", [0, 2, 3, 10, 100, 102])
@pytest.mark.parametrize("key", ND_KEYS)
def test_gaussnd_golden(key, variant):
    g = golden("gaussnd_cases.npz")
    set_gaussnd_variant(variant)
    try:
        dx, dp = t(g[f"{key}_dx0"]), t(g[f"{key}_dp0"])
        adc.launch_batch("gaussnd_grad_0_1", t(g[f"{key}_x"]), t(g[f"{key}_p"]),
                         float(g[f"{key}_sigma"]), dx, dp)
        assert acc_err(host(dx), g[f"{key}_dx"], g[f"{key}_dx0"]).max() <= REL
        assert acc_err(host(dp), g[f"{key}_dp"], g[f"{key}_dp0"]).max() <= REL
    finally:
        set_gaussnd_variant(0)


def test_gaussnd_host_path():
    g = golden("gaussnd_cases.npz")
    key = "d37_n70"
    dx, dp = g[f"{key}_dx0"].copy(), g[f"{key}_dp0"].copy()
    adc.launch_batch("gaussnd_grad_0_1", g[f"{key}_x"].copy(), g[f"{key}_p"].copy(),
                     float(g[f"{key}_sigma"]), dx, dp)
    assert acc_err(dx, g[f"{key}_dx"], g[f"{key}_dx0"]).max() <= REL
    assert acc_err(dp, g[f"{key}_dp"], g[f"{key}_dp0"]).max() <= REL


@pytest.mark.parametrize("dim,n", [(100, 200_003), (100, 200_010), (64, 4096), (1000, 20_011),
                                   (5, 77), (300, 1000), (2, 4097), (3, 1000), (4, 2049),
                                   (6, 640), (8, 1001), (12, 777), (16, 3000), (110, 513)])
def test_gaussnd_vs_oracle(restate, dim, n):
    # variant 0 = auto (K2: 8 neighbouring tiles per CTA up to 112 dims, the
    # row batch U following the dims; dims over the warps of a CTA above;
    # spans claimed in order), 3 = K2 one warp per 32-point tile, 2 = K2 with
    # the dims over the warps of a CTA, 10 = K2v (double2) forced; + 100 =
    # the static grid-stride schedule
    x, p = synth.points_nd(dim, n, seed=dim)
    ox, op = np.zeros((dim, n)), np.zeros((dim, n))
    restate.gaussnd_grad(x, p, 1.3, ox, op)
    for variant in (0, 2, 3, 10, 100, 102, 103):
        set_gaussnd_variant(variant)
        try:
            dx = torch.zeros((dim, n), dtype=torch.float64, device=DEV)
            dp = torch.zeros_like(dx)
            adc.launch_batch("gaussnd_grad_0_1", t(x), t(p), 1.3, dx, dp)
            hx, hp = host(dx), host(dp)
            assert rel_err(hx, ox).max() <= REL, variant
            assert rel_err(hp, op).max() <= REL, variant
            assert np.array_equal(hx, -hp)
        finally:
            set_gaussnd_variant(0)


def test_gaussnd_accumulates_twice():
    # accumulate-only slots: two launches double the first (test_reverse.cpp:335-348).
    x, p = synth.points_nd(64, 4096, seed=5)
    dx = torch.zeros((64, 4096), dtype=torch.float64, device=DEV)
    dp = torch.zeros_like(dx)
    X, P = t(x), t(p)
    adc.launch_batch("gaussnd_grad_0_1", X, P, 0.9, dx, dp)
    once = host(dx).copy()
    adc.launch_batch("gaussnd_grad_0_1", X, P, 0.9, dx, dp)
    assert np.array_equal(host(dx), 2 * once)


def _nd_repeat(variant, X, P, launches, sigma=1.1):
    set_gaussnd_variant(variant)
    try:
        dx = torch.zeros_like(X)
        dp = torch.zeros_like(X)
        for _ in range(launches):
            adc.launch_batch("gaussnd_grad_0_1", X, P, sigma, dx, dp)
        return host(dx), host(dp)
    finally:
        set_gaussnd_variant(0)


@pytest.mark.parametrize("dim,n", [(2, 400_003), (37, 200_001), (300, 30_011)])
def test_gaussnd_claimed_spans_match_static(dim, n):
    # Claimed spans (auto) and the static grid-stride schedule (+100) run the
    # same per-point arithmetic: bit-identical, with more spans than CTAs so
    # claiming engages (dim 2: ~1.5k spans of 256 points).
    x, p = synth.points_nd(dim, n, seed=dim + 1)
    X, P = t(x), t(p)
    a = _nd_repeat(0, X, P, 1)
    b = _nd_repeat(100, X, P, 1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_gaussnd_claim_ring_wraps():
    # 4100 launches walk every pair of the 4096-slot claim ring and reuse some:
    # each launch's last CTA must leave its pair at zero, or a reused pair
    # would skip spans.  The accumulated slots equal the static schedule's.
    x, p = synth.points_nd(2, 400_003, seed=11)
    X, P = t(x), t(p)
    a = _nd_repeat(0, X, P, 4100)
    b = _nd_repeat(100, X, P, 4100)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_gaussnd_claimed_spans_concurrent_threads():
    # four host threads, each on its own stream with its own buffers, launch
    # at the same time: each launch takes its own claim pair from the ring, so
    # every thread's slots equal the single-thread result bit for bit
    import threading
    x, p = synth.points_nd(37, 200_001, seed=8)
    X, P = t(x), t(p)
    ref = _nd_repeat(0, X, P, 5)
    out, errs = {}, []

    def work(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                dx = torch.zeros_like(X)
                dp = torch.zeros_like(X)
                for _ in range(5):
                    adc.launch_batch("gaussnd_grad_0_1", X, P, 1.1, dx, dp)
            s.synchronize()
            out[k] = (host(dx), host(dp))
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    ths = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errs, errs
    for k in range(4):
        assert np.array_equal(out[k][0], ref[0]) and np.array_equal(out[k][1], ref[1]), k


def test_gaussnd_claimed_spans_in_cuda_graph():
    # a captured launch keeps one claim pair; the kernel resets it, so graph
    # replays accumulate exactly like eager launches
    x, p = synth.points_nd(37, 200_001, seed=4)
    X, P = t(x), t(p)
    eager = _nd_repeat(0, X, P, 3)
    dx = torch.zeros_like(X)
    dp = torch.zeros_like(X)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        adc.launch_batch("gaussnd_grad_0_1", X, P, 1.1, dx, dp)  # warm-up outside capture
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    dx.zero_()
    dp.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        adc.launch_batch("gaussnd_grad_0_1", X, P, 1.1, dx, dp)
    for _ in range(3):
        g.replay()
    assert np.array_equal(host(dx), eager[0]) and np.array_equal(host(dp), eager[1])


# ---------------------------------------------------------------------------- chi2
CHI2_KEYS = ["gpoly_b2000", "gsum1_b1000", "gsum2_b1500"]


@pytest.mark.parametrize("fast", [0, 1, 2])
@pytest.mark.parametrize("key", CHI2_KEYS)
def test_chi2_golden(restate, key, fast):
    g = golden("chi2_cases.npz")
    model = str(g[f"{key}_model"])
    counts, q, ev = g[f"{key}_counts"], g[f"{key}_q"], float(g[f"{key}_events"])
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)
    plan = adc.Chi2Plan(model, q.size, h)
    plan.set_precision(fast)
    grad, c2 = plan.gradient(q)
    ref, scale = restate.chi2_gradient_compensated(model, counts, -5.0, 5.0, ev, q)
    assert np.all(np.abs(grad - ref) <= 1e-12 * scale), (grad, ref, scale)
    # and against the reference's own (sequential) numbers
    assert np.all(np.abs(grad - g[f"{key}_grad"]) <= 1e-12 * scale)
    vref, vscale = restate.chi2_compensated(model, counts, -5.0, 5.0, ev, q)
    assert abs(c2 - vref) <= 1e-12 * vscale
    assert abs(plan.chi2(q) - g[f"{key}_chi2"]) <= 1e-12 * vscale


def test_chi2_config3_1e6(restate):
    counts, ev = synth.histogram(10**6, events=1e8)
    q = np.array(synth.GPOLY_INIT)
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)
    plan = adc.Chi2Plan("gpoly", 6, h)
    grad, c2 = plan.gradient(q)
    ref, scale = restate.chi2_gradient_compensated("gpoly", counts, -5.0, 5.0, ev, q)
    assert np.all(np.abs(grad - ref) <= 1e-12 * scale)
    vref, vscale = restate.chi2_compensated("gpoly", counts, -5.0, 5.0, ev, q)
    assert abs(c2 - vref) <= 1e-12 * vscale


@pytest.mark.parametrize("model,q", [
    ("gpoly", synth.GPOLY_INIT),
    ("gsum", (0.9, 0.1, 1.4)),
    ("gsum", (0.7, -1.0, 1.2, 0.4, 1.5, 0.8)),
])
def test_chi2_gaussian_recurrence(restate, model, q):
    """Precision mode 2 (default): gradient passes take each thread's Gaussian
    factors from the anchored product recurrence (bpt >= 16 from ~1.2M bins
    here 2M bins, 28 per thread).  Against the compensated oracle within the
    reduction tolerance and within ~1e-13 of mode 1's per-bin table exp; the
    same for the value pass, and the batched line-search pass repeats the
    value pass bit for bit per candidate."""
    bins = 2_000_000
    q = np.array(q)
    counts, ev = synth.histogram(bins, events=2e8, seed=21, model=model, q=q)
    h = adc.Histogram(bins, -5.0, 5.0, ev, counts)
    plan = adc.Chi2Plan(model, q.size, h)
    assert plan.layout.tile_bins // 256 >= 16
    g2, c2 = plan.gradient(q)
    ref, scale = restate.chi2_gradient_compensated(model, counts, -5.0, 5.0, ev, q)
    assert np.all(np.abs(g2 - ref) <= 1e-12 * scale)
    v2 = plan.chi2(q)
    vref, vscale = restate.chi2_compensated(model, counts, -5.0, 5.0, ev, q)
    assert abs(v2 - vref) <= 1e-12 * vscale
    g = np.linspace(0.5, 1.5, q.size) * 1e-3 * np.abs(q)
    qs = np.stack([q - 2.0 ** -k * g for k in range(9)])
    assert plan.chi2_multi(qs).tobytes() == np.array([plan.chi2(qk) for qk in qs]).tobytes()
    plan.set_precision(1)
    g1, c1 = plan.gradient(q)
    assert np.all(np.abs(g2 - g1) <= 1e-13 * scale)
    assert abs(plan.chi2(q) - v2) <= 1e-13 * vscale
    # the recurrence really ran: the chunk records (before the final rounding
    # of the closed form) are not mode 1's
    R = adc.record_len(q.size, True)
    recs = []
    for mode in (2, 1):
        plan.set_precision(mode)
        r = torch.zeros(plan.layout.nchunks * R, dtype=torch.float64, device="cuda")
        plan.partials(list(q), True, r)
        recs.append(host(r))
    assert recs[0].tobytes() != recs[1].tobytes()


@pytest.mark.parametrize("bins,model,np_", [(100_003, "gpoly", 6), (2_000_000, "gpoly", 6),
                                            (300_000, "gsum", 12)])
def test_chi2_gradient_batch_bitwise_equals_single(bins, model, np_):
    """adc_cuda_chi2_gradient_multi runs its members as ONE batched launch
    (blockIdx.y = member); each member's gradient is bit-identical to a single
    gradient pass."""
    if model == "gpoly":
        q = np.array(synth.GPOLY_INIT)
    else:
        q = np.array(adc.perturbed_init(adc.default_truth(np_ // 3)))
    counts, ev = synth.histogram(bins, events=100.0 * bins, seed=31, model=model,
                                 q=adc.default_truth(np_ // 3) if model == "gsum" else synth.GPOLY_TRUTH)
    h = adc.Histogram(bins, -5.0, 5.0, ev, counts)
    plan = adc.Chi2Plan(model, np_, h)
    qs = np.stack([q * (1.0 + 1e-3 * k) for k in range(2 * np_)])
    batch = plan.gradient_multi(qs)
    single = np.stack([plan.gradient(qk)[0] for qk in qs])
    assert batch.tobytes() == single.tobytes()


def test_chi2_recurrence_skipped_for_wide_runs():
    """When a thread's run of bins spans more than one sigma (|D| bpt > 1) the
    recurrence is not used: mode 2 is bitwise mode 1."""
    bins = 2_000_000
    q = np.array([1.0, 0.3, 0.004, 0.2, -0.01, 0.003])  # sigma = 0.004: D = 0.32, bpt 28
    counts, ev = synth.histogram(bins, events=2e8, seed=23, model="gpoly", q=q)
    h = adc.Histogram(bins, -5.0, 5.0, ev, counts)
    plan = adc.Chi2Plan("gpoly", 6, h)
    g2, _ = plan.gradient(q)
    plan.set_precision(1)
    g1, _ = plan.gradient(q)
    assert g2.tobytes() == g1.tobytes()


def test_chi2_sharding_bitwise_invariant():
    # Any split of whole chunks over ranks gives the same bits (fixed trees).
    counts, ev = synth.histogram(3_000_000, events=3e8, seed=9)
    q = np.array(synth.GPOLY_INIT)
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)
    full = adc.Chi2Plan("gpoly", 6, h)
    g1, c1 = full.gradient(q)
    R = adc.record_len(6, True)
    for world in (2, 3, 4, 8):
        recs = []
        for rank in range(world):
            pl = adc.Chi2Plan("gpoly", 6, h, world=world, rank=rank)
            nloc = pl.layout.chunk_end - pl.layout.chunk_begin
            buf = torch.zeros(max(1, nloc) * R, dtype=torch.float64, device=DEV)
            pl.partials(q, True, buf)
            torch.cuda.synchronize()
            recs.append(buf.cpu().numpy()[:nloc * R])
            pl.close()
        gw, cw = adc.finalize(6, ev, np.concatenate(recs), True)
        assert np.array_equal(gw, g1) and cw == c1, world


def test_chi2_domain_error():
    counts, ev = synth.histogram(1000, events=1e5)
    h = adc.Histogram(1000, -5.0, 5.0, ev, counts)
    with pytest.raises(adc.AdcError) as e:
        adc.FitEngine("gpoly", 6).chi2_gradient(h, [1, 0, 0.0, 0, 0, 0])
    assert e.value.kind == "Eval"


# ---------------------------------------------------------------------------- fit
@pytest.mark.parametrize("key", ["gpoly_b400", "gsum1_b300", "gpoly_b400_hess",
                                 "gsum1_b300_hess"])
def test_fit_iterates_match_reference(key):
    """Fit iterates against the reference's FitEngine::fit (fit.cpp:315-425).

    Steepest descent: every traced iterate within 1e-9.  Numeric-Hessian Newton
    steps difference the gradient over ~6e-6 and solve a nearly singular system
    (chi2 normalises by S, so the overall amplitude scale is unidentified and
    the Hessian is singular along it): the reference's own iterate-sequence
    precedent, 1e-5 (test_fit.cpp:95-109), applies to the identified shape
    parameters; the final chi2 must agree to 1e-6."""
    g = golden("fit_cases.npz")
    model = str(g[f"{key}_model"])
    init = g[f"{key}_init"]
    counts = g[f"{key}_counts"]
    hess = bool(g[f"{key}_hessian"])
    h = adc.Histogram(counts.size, -5.0, 5.0, float(counts.sum()), counts)
    eng = adc.FitEngine(model, init.size)
    res = eng.fit(h, init, adc.FitOptions(budget=12, trace_iterates=10, use_hessian=hess))
    ref_its = g[f"{key}_iterates"]
    n_ref = min(10, int(g[f"{key}_iterations"]) + 1)
    assert len(res.iterates) == n_ref
    assert res.iterations == int(g[f"{key}_iterations"])
    assert rel_err(res.chi2, g[f"{key}_chi2"]) <= (1e-6 if hess else 1e-10)
    if not hess:
        cols, tol = slice(None), 1e-9
    else:
        cols, tol = ([1, 2] if model == "gsum" else slice(None)), 1e-5
    for k in range(n_ref):
        assert rel_err(np.asarray(res.iterates[k])[cols], ref_its[k][cols]).max() <= tol, k
    assert rel_err(np.asarray(res.params)[cols], g[f"{key}_params"][cols]).max() <= tol


def test_chi2_multi_bitwise_equals_single():
    # The batched line-search pass gives each candidate exactly the single pass's bits.
    for bins in (2000, 1_000_000, 5_000_000):
        counts, ev = synth.histogram(bins, events=100.0 * bins, seed=bins)
        h = adc.Histogram(bins, -5.0, 5.0, ev, counts)
        pl = adc.Chi2Plan("gpoly", 6, h)
        q = np.array(synth.GPOLY_INIT)
        g = np.array([1e3, -2e3, 5e2, 10.0, -3.0, 1.0])
        qs = np.stack([q - 2.0 ** -k * g for k in range(32)])
        multi = pl.chi2_multi(qs)
        single = np.array([pl.chi2(qk) for qk in qs])
        assert np.array_equal(multi, single), bins
        assert np.array_equal(pl.chi2_multi(qs[:5]), single[:5])
        gm = pl.gradient_multi(qs[:12])
        for k in range(12):
            assert np.array_equal(gm[k], pl.gradient(qs[k])[0]), (bins, k)


def test_fit_1e6_newton_converges_to_truth():
    # Plain steepest descent (the reference default) crawls on this badly scaled
    # 6-parameter problem; the reference's numeric-Hessian Newton option converges.
    counts, ev = synth.histogram(10**6, events=1e8, seed=11)
    h = adc.Histogram(10**6, -5.0, 5.0, ev, counts)
    r = adc.FitEngine("gpoly", 6).fit(h, synth.GPOLY_INIT,
                                      adc.FitOptions(budget=400, use_hessian=True))
    # the Gaussian's position and width are identified (the overall scale is
    # not: chi2 normalises by S, fit.cpp:231-245)
    # Gaussian parameters recovered to the reference's bounds (test_fit.cpp:81-93)
    assert abs(r.params[1] - synth.GPOLY_TRUTH[1]) < 0.05
    assert abs(r.params[2] - synth.GPOLY_TRUTH[2]) < 0.05


# ---------------------------------------------------------------------------- Numeric provider
@pytest.mark.parametrize("key", ["gpoly_b2000", "gsum1_b1000", "gsum2_b1500"])
@pytest.mark.parametrize("fast", [True, False])
def test_chi2_numeric_provider(restate, key, fast):
    """GradientProvider::Numeric (fit.cpp:187-190 -> central_gradient,
    numdiff.cpp:38-87) against the reference's own numbers and the compensated
    restatement.  Tolerance: the reduction bound 1e-12 * sum|terms| plus the
    finite-difference amplification of the primal's last-ulp differences
    (libdevice / table exp vs glibc): K ulps of m_j times |w_j| / (2h_i),
    K = 4 faithful, 16 fast (reciprocal multiplies add ulps to z and m)."""
    g = golden("chi2_numeric_cases.npz")
    model = str(g[f"{key}_model"])
    counts, q, ev = g[f"{key}_counts"], g[f"{key}_q"], float(g[f"{key}_events"])
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)
    eng = adc.FitEngine(model, q.size)
    eng._plan(h).set_precision(fast)
    grad = eng.chi2_gradient(h, q, adc.GradientProvider.Numeric)
    ref, scale, fd = restate.chi2_gradient_numeric_compensated(model, counts, -5.0, 5.0, ev, q)
    tol = 1e-12 * scale + (16.0 if fast else 4.0) * fd
    assert np.all(np.abs(grad - ref) <= tol), (grad - ref, tol)
    assert np.all(np.abs(grad - g[f"{key}_grad"]) <= tol + 1e-12 * scale)
    # the AD provider is a different (exact) gradient of the same chi2
    ad = eng.chi2_gradient(h, q, adc.GradientProvider.AdReverse)
    assert np.all(np.abs(ad - grad) <= 1e-6 * scale)
    assert not np.array_equal(ad, grad)


@pytest.mark.parametrize("key", ["gpoly_b2000", "gsum1_b1000", "gsum2_b1500"])
def test_fit_numeric_provider_matches_reference(key):
    """FitEngine::fit(h, Numeric, ...) iterates (fit-in <model>:numeric, budget 12)."""
    g = golden("chi2_numeric_cases.npz")
    model = str(g[f"{key}_model"])
    counts, q, ev = g[f"{key}_counts"], g[f"{key}_q"], float(g[f"{key}_events"])
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)
    res = adc.FitEngine(model, q.size).fit(h, q, adc.FitOptions(budget=12, trace_iterates=10),
                                           provider=adc.GradientProvider.Numeric)
    assert res.iterations == int(g[f"{key}_fit_iterations"])
    assert rel_err(res.chi2, g[f"{key}_fit_chi2"]) <= 1e-9
    its = g[f"{key}_fit_iterates"]
    for k in range(min(10, res.iterations + 1)):
        assert rel_err(np.asarray(res.iterates[k]), its[k]).max() <= 1e-6, k


def test_numeric_provider_probe_domain_error():
    # a width whose probe q - h hits 0 is the interpreter's division by zero
    counts, ev = synth.histogram(1000, events=1e5)
    h = adc.Histogram(1000, -5.0, 5.0, ev, counts)
    h0 = np.cbrt(2.220446049250313e-16)
    with pytest.raises(adc.AdcError) as e:
        adc.FitEngine("gpoly", 6).chi2_gradient(h, [1, 0, h0, 0, 0, 0], adc.GradientProvider.Numeric)
    assert e.value.kind == "Eval"


# ---------------------------------------------------------------------------- compute_shared
@pytest.mark.parametrize("case", ["n100", "n4097"])
@pytest.mark.parametrize("device", [True, False])
def test_compute_shared_forced_deterministic(restate, case, device):
    """compute_shared (kernels.dsl:16-21) forced: dx, dp per point within 1e-12
    (as `compute`); dsigma = dsigma0 + a fixed-order sum of all contributions,
    within 1e-12 * sum|contributions| of the compensated total and within the
    reference's own 1e-9 (test_launch.cpp:165) of its sequential result;
    identical bits on every run."""
    g = golden("gauss_shared_cases.npz")
    n, sigma, block = g[f"{case}_x"].size, float(g[f"{case}_sigma"]), int(g[f"{case}_block"])
    cfg = adc.LaunchConfig(n // block + 1, block, n)

    def run():
        arrs = {k: g[f"{case}_{k}"].copy() for k in ("x", "p")}
        arrs.update(dx=g[f"{case}_dx0"].copy(), dp=g[f"{case}_dp0"].copy(),
                    dsigma=g[f"{case}_dsigma0"].copy())
        if device:
            arrs = {k: t(v) for k, v in arrs.items()}
        adc.launch("compute_shared", cfg, adc.BufferSet(arrays=arrs, scalars={"sigma": sigma}),
                   adc.LaunchOptions(unsafe=True))
        return {k: host(v) if device else v for k, v in arrs.items()}

    a = run()
    assert rel_err(a["dx"], g[f"{case}_dx"]).max() <= REL
    assert rel_err(a["dp"], g[f"{case}_dp"]).max() <= REL
    tot, scale = restate.gauss_shared_dsigma_compensated(g[f"{case}_x"], g[f"{case}_p"], sigma)
    d0 = g[f"{case}_dsigma0"][0]
    assert abs(a["dsigma"][0] - (d0 + tot)) <= 1e-12 * (scale + abs(d0))
    assert rel_err(a["dsigma"][0], g[f"{case}_dsigma"][0]) <= 1e-9
    b = run()
    assert a["dsigma"].tobytes() == b["dsigma"].tobytes()


def test_compute_shared_large_vs_oracle(restate):
    n = 3_000_017
    rng = np.random.Generator(np.random.PCG64(4))
    x, p = rng.uniform(-3, 3, n), rng.uniform(-2, 2, n)
    dx, dp, ds = np.zeros(n), np.zeros(n), np.zeros(1)
    bufs = {"x": t(x), "p": t(p), "dx": t(dx), "dp": t(dp), "dsigma": t(ds)}
    adc.launch("compute_shared", adc.LaunchConfig(n // 256 + 1, 256, n),
               adc.BufferSet(arrays=bufs, scalars={"sigma": 1.1}), adc.LaunchOptions(unsafe=True))
    rx, rp, rs = np.zeros(n), np.zeros(n), np.zeros(1)
    restate.gauss_grad_shared(x, p, 1.1, rx, rp, rs)
    assert rel_err(host(bufs["dx"]), rx).max() <= REL
    tot, scale = restate.gauss_shared_dsigma_compensated(x, p, 1.1)
    assert abs(host(bufs["dsigma"])[0] - tot) <= 1e-12 * scale


def test_compute_shared_refused_without_unsafe():
    n = 64
    bufs = {k: t(np.zeros(n)) for k in ("x", "p", "dx", "dp")}
    bufs["dsigma"] = t(np.zeros(1))
    with pytest.raises(adc.AdcError) as e:
        adc.launch("compute_shared", adc.LaunchConfig(1, 64, n),
                   adc.BufferSet(arrays=bufs, scalars={"sigma": 1.0}))
    assert e.value.kind == "Launch" and str(e.value).startswith("launch refused")


def test_plan_refresh_after_counts_change(restate):
    # The plan snapshots what depends on the counts alone (1/c, C0, linear
    # sums); refresh() picks up an in-place change of device counts.
    counts, ev = synth.histogram(50_000, events=5e6, seed=31)
    dc = t(counts)
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, dc)
    pl = adc.Chi2Plan("gpoly", 6, h)
    q = np.array(synth.GPOLY_INIT)
    g1, c1 = pl.gradient(q)
    dc[::7] += 3.0
    torch.cuda.synchronize()
    pl.refresh()
    g2, c2 = pl.gradient(q)
    c_new = host(dc)
    ref, scale = restate.chi2_gradient_compensated("gpoly", c_new, -5.0, 5.0, ev, q)
    assert np.all(np.abs(g2 - ref) <= 1e-12 * scale)
    assert not np.array_equal(g1, g2)


# ---------------------------------------------------------------------------- histogram sampling
@pytest.mark.parametrize("events", [1e8, 3e6])
def test_sample_histogram_statistics_and_determinism(events):
    """K6: counts ~ Poisson(E m_j / S) (PTRS for large means, multiplication
    below 10): standardised residuals have mean 0 and variance 1; the same
    seed gives the same bits; Histogram.events is the exact count total."""
    bins = 1_000_000
    q = np.array(synth.GPOLY_TRUTH)
    h = adc.sample_histogram("gpoly", q, bins, -5.0, 5.0, events, seed=7)
    c = host(h.counts)
    assert np.all(c == np.floor(c)) and np.all(c >= 0)
    assert h.events == c.sum()
    x = -5.0 + (np.arange(bins) + 0.5) * (10.0 / bins)
    m = np.array([0.0] * bins)
    z = (x - q[1]) / q[2]
    m = q[0] * np.exp(-0.5 * z * z) + q[3] + q[4] * x + q[5] * x * x
    lam = events * m / m.sum()
    r = (c - lam) / np.sqrt(lam)
    assert abs(r.mean()) < 5 / np.sqrt(bins)
    assert abs(r.var() - 1.0) < 0.01
    h2 = adc.sample_histogram("gpoly", q, bins, -5.0, 5.0, events, seed=7)
    assert host(h2.counts).tobytes() == c.tobytes()
    h3 = adc.sample_histogram("gpoly", q, bins, -5.0, 5.0, events, seed=8)
    assert not np.array_equal(host(h3.counts), c)


def test_sample_histogram_zero_every_and_fit():
    h = adc.sample_histogram("gpoly", synth.GPOLY_TRUTH, 1_000_000, -5.0, 5.0, 1e8, seed=3,
                             zero_every=100)
    c = host(h.counts)
    assert np.all(c[::100] == 0) and np.all(c[1::100] > 0)
    r = adc.FitEngine("gpoly", 6).fit(h, synth.GPOLY_INIT,
                                      adc.FitOptions(budget=200, use_hessian=True))
    assert abs(r.params[1] - synth.GPOLY_TRUTH[1]) < 0.05
    assert abs(r.params[2] - synth.GPOLY_TRUTH[2]) < 0.05


def test_bench_scaling_rows():
    rows = adc.bench_scaling(k_list=(1, 2), bins=20_000, events=2e6,
                             opts=adc.FitOptions(budget=30))
    assert [(r.k, r.provider) for r in rows] == [(1, "ad-reverse"), (1, "numeric"),
                                                  (2, "ad-reverse"), (2, "numeric")]
    assert all(r.grad_evals > 0 and r.median_wall_ns > 0 for r in rows)
    csv = adc.bench_csv(rows)
    assert csv.splitlines()[0].startswith("K,params,provider")


# ---------------------------------------------------------------------------- shared mean vector
@pytest.mark.parametrize("key", ["d100_n64", "d37_n150", "d1_n40", "d300_n33"])
def test_gaussnd_shared_p_golden(restate, key):
    """One p and one shared dp slot for every point: dx per point within 1e-12
    (as K2); dp = dp0 + a fixed-order sum of every point's -_r6, within
    1e-12 * sum|terms| of the compensated total, within the reference's 1e-9
    (test_launch.cpp:165) of its sequential result, bitwise repeatable."""
    g = golden("gaussnd_shared_p_cases.npz")
    x, p = g[f"{key}_x"], g[f"{key}_p"]

    def run():
        dx, dp = t(g[f"{key}_dx0"]), t(g[f"{key}_dp0"])
        adc.launch_batch_shared_p("gaussnd_grad_0_1", t(x), t(p), 1.3, dx, dp,
                                  adc.LaunchOptions(unsafe=True))
        return host(dx), host(dp)

    dx, dp = run()
    scale = np.maximum(np.abs(g[f"{key}_dx0"]), 0)
    assert (np.abs(dx - g[f"{key}_dx"]) <= REL * np.maximum(
        np.maximum(np.abs(dx), np.abs(g[f"{key}_dx"])), scale)).all()
    tot, ab = restate.gaussnd_shared_p_dp_compensated(np.ascontiguousarray(x), p, 1.3)
    dp0 = g[f"{key}_dp0"]
    assert np.all(np.abs(dp - (dp0 + tot)) <= 1e-12 * (ab + np.abs(dp0)))
    assert rel_err(dp, g[f"{key}_dp"]).max() <= 1e-9
    dx2, dp2 = run()
    assert dp2.tobytes() == dp.tobytes() and dx2.tobytes() == dx.tobytes()


def test_gaussnd_shared_p_large_and_refusal(restate):
    dim, n = 100, 200_003
    x, _ = synth.points_nd(dim, n, seed=5)
    p = np.linspace(-1, 1, dim)
    x = p[:, None] + 0.1 * np.random.Generator(np.random.PCG64(6)).standard_normal((dim, n))
    dp = t(np.zeros(dim))
    with pytest.raises(adc.AdcError) as e:
        adc.launch_batch_shared_p("gaussnd_grad_0_1", t(x), t(p), 1.3, None, dp)
    assert e.value.kind == "Launch" and str(e.value).startswith("launch refused")
    adc.launch_batch_shared_p("gaussnd_grad_0_1", t(x), t(p), 1.3, None, dp,
                              adc.LaunchOptions(unsafe=True))
    tot, ab = restate.gaussnd_shared_p_dp_compensated(np.ascontiguousarray(x), p, 1.3)
    assert np.all(np.abs(host(dp) - tot) <= 1e-12 * ab)


@pytest.mark.parametrize("dim,n", [(100, 200_006), (37, 64 * 700), (128, 5_000), (2, 10_001),
                                   (3, 6_400), (5, 4_099), (12, 3_000), (24, 7_001), (25, 3_333),
                                   (256, 1_100), (257, 650)])
def test_gaussnd_shared_p_with_dx_paths(restate, dim, n):
    """With private dx slots: up to 24 dims K2sr (a thread per point, any
    layout); up to 256 dims the staged-tile form (4 or 8 warps per 32-point
    tile, ragged tail through K2s) — the aligned layout with 2-D tensor
    loads, an odd-offset view with cp.async copies; K2s above.  dx per point
    within 1e-12 of the restatement in both; dp within 1e-12 * sum|terms| of
    the compensated total in both (the paths sum in different fixed orders);
    each path bitwise repeatable."""
    rng = np.random.Generator(np.random.PCG64(dim))
    p = rng.uniform(-1, 1, dim)
    x = p[:, None] + 0.1 * rng.standard_normal((dim, n))
    dx0 = rng.standard_normal((dim, n))
    dp0 = rng.standard_normal(dim)
    rdx, rdp = dx0.copy(), dp0.copy()
    restate.gaussnd_grad_shared_p(np.ascontiguousarray(x), p, 1.3, rdx, rdp)
    tot, ab = restate.gaussnd_shared_p_dp_compensated(np.ascontiguousarray(x), p, 1.3)
    o = adc.LaunchOptions(unsafe=True)
    wide = np.zeros((dim, n + 1))
    per_offset = []
    for offset in (0, 1):
        X = t(np.ascontiguousarray(x)) if offset == 0 else t(wide)[:, 1:]
        if offset:
            X.copy_(t(x))
        runs = []
        for _ in range(2):
            DX = t(dx0) if offset == 0 else t(np.zeros((dim, n + 1)))[:, 1:]
            if offset:
                DX.copy_(t(dx0))
            DP = t(dp0)
            adc.launch_batch_shared_p("gaussnd_grad_0_1", X, t(p), 1.3, DX, DP, o)
            runs.append((host(DX), host(DP)))
        (gdx, gdp), (gdx2, gdp2) = runs
        assert gdx.tobytes() == gdx2.tobytes() and gdp.tobytes() == gdp2.tobytes()
        assert acc_err(gdx, rdx, dx0).max() <= REL, offset
        assert np.all(np.abs(gdp - (dp0 + tot)) <= 1e-12 * (ab + np.abs(dp0))), offset
        per_offset.append(gdx)
    # a point's dx bits do not depend on which form its layout selected (K2s
    # sums the forward in the TMA form's warp chunks)
    assert per_offset[0].tobytes() == per_offset[1].tobytes()


def test_gaussnd_strided_views(restate):
    # a (dim, n) view of a wider SoA buffer: the row stride comes from the view
    dim, n, big = 50, 3000, 3200
    x, p = synth.points_nd(dim, big, seed=44)
    X, P = t(x), t(p)
    DX = torch.zeros_like(X)
    DP = torch.zeros_like(X)
    adc.launch_batch("gaussnd_grad_0_1", X[:, 64:64 + n], P[:, 64:64 + n], 1.3,
                     DX[:, 64:64 + n], DP[:, 64:64 + n])
    ox, op = np.zeros((dim, n)), np.zeros((dim, n))
    restate.gaussnd_grad(np.ascontiguousarray(x[:, 64:64 + n]),
                         np.ascontiguousarray(p[:, 64:64 + n]), 1.3, ox, op)
    hx = host(DX)
    assert rel_err(hx[:, 64:64 + n], ox).max() <= REL
    assert np.all(hx[:, :64] == 0) and np.all(hx[:, 64 + n:] == 0)
    with pytest.raises(adc.AdcError):
        adc.launch_batch("gaussnd_grad_0_1", X[:, ::2], P[:, ::2], 1.3, DX[:, ::2], DP[:, ::2])


@pytest.mark.parametrize("case", ["gpoly_1e6", "gpoly_1e6_b1", "gpoly_1e6_b3", "gsum1", "gsum2",
                                  "gsum4", "gpoly_1e6_newton", "gsum2_newton", "gsum4_newton",
                                  "gsum2_numeric", "gsum1_numeric_newton",
                                  "gpoly_1e6_b3_numeric"])
def test_device_fit_loop_bitwise_equals_host_loop(case):
    """The device-resident loop (one graph, a WHILE node around the
    steepest-descent body: gradient pass, finalize, Armijo trials, multi pass,
    selection, loop control; the host only continues searches longer than a
    batch) takes exactly the host-driven loop's steps: same iterates, chi2 and
    counters, bit for bit — also when the budget ends the loop early, with the
    Newton option (2 np probe gradient passes, Hessian, damped solve) and with
    the numeric gradient provider."""
    import os
    newton = case.endswith("_newton")
    numeric = "_numeric" in case
    case = case.replace("_newton", "").replace("_numeric", "")
    if case.startswith("gpoly_1e6"):
        counts, ev = synth.histogram(10**6, events=1e8, seed=11)
        budget = {"gpoly_1e6": 400, "gpoly_1e6_b1": 1, "gpoly_1e6_b3": 3}[case]
        model, init = "gpoly", list(synth.GPOLY_INIT)
    else:
        k = int(case[-1])
        truth = adc.default_truth(k)
        counts, ev = synth.histogram(20_000, -5.0, 5.0, 2e6, "gsum", truth, seed=k)
        model, init, budget = "gsum", adc.perturbed_init(truth), 200
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)
    out = {}
    for mode in ("0", "1"):
        r = adc.FitEngine(model, len(init)).fit(
            h, init, adc.FitOptions(budget=budget, trace_iterates=budget + 1,
                                    use_hessian=newton, host_loop=mode == "0"),
            provider=adc.GradientProvider.Numeric if numeric else
            adc.GradientProvider.AdReverse)
        out[mode] = r
    a, b = out["0"], out["1"]
    assert a.iterations == b.iterations and a.gradient_evals == b.gradient_evals
    assert a.chi2_evals == b.chi2_evals and a.sigma_clamps == b.sigma_clamps
    assert a.converged == b.converged
    assert np.array(a.params).tobytes() == np.array(b.params).tobytes()
    assert a.chi2 == b.chi2
    assert np.array(a.iterates).tobytes() == np.array(b.iterates).tobytes()


# ---------------------------------------------------------------------------- high counts per bin
@pytest.mark.parametrize("bins,events", [(1000, 1e8), (100, 1e11), (20_000, 1e9)])
def test_chi2_value_high_counts_residual(restate, bins, events):
    """the single pass's chi2 = C0 - 2a A1 + a^2 A2 loses ~eps * E
    (relative ~5 eps kappa, kappa = counts per bin).  Plans with kappa > 256
    compute chi2 values as sum (c - a m)^2 / c directly (K3r).  Checked
    against the compensated oracle RELATIVE TO chi2 itself (not the ~4E sum of
    the expanded terms), through every value entry point, and the batched
    line search still equals the single value pass bit for bit."""
    counts, ev = synth.histogram(bins, events=events, seed=bins)
    h = adc.Histogram(bins, -5.0, 5.0, ev, counts)
    plan = adc.Chi2Plan("gpoly", 6, h)
    resid, kappa = plan.value_mode()
    assert resid and kappa > 256
    q = np.array(synth.GPOLY_INIT)
    cref, _ = restate.chi2_compensated("gpoly", counts, -5.0, 5.0, ev, q)
    v = plan.chi2(q)
    assert abs(v - cref) <= 1e-12 * abs(cref), (v, cref, abs(v - cref) / cref)
    g, c2 = plan.gradient(q)
    assert abs(c2 - cref) <= 1e-12 * abs(cref)  # (its S is the gradient pass's: other bits)
    ref, scale = restate.chi2_gradient_compensated("gpoly", counts, -5.0, 5.0, ev, q)
    assert np.all(np.abs(g - ref) <= 1e-12 * scale)
    qs = np.stack([q, q * (1 + 1e-4), q * (1 - 1e-4)])
    vm = plan.chi2_multi(qs)
    assert vm[0] == v
    for k in range(3):
        ck, _ = restate.chi2_compensated("gpoly", counts, -5.0, 5.0, ev, qs[k])
        assert abs(vm[k] - ck) <= 1e-12 * abs(ck)
    # the fit runs (host loop in this mode) and agrees with the reference's bound
    r = adc.FitEngine("gpoly", 6).fit(h, synth.GPOLY_INIT, adc.FitOptions(budget=60, use_hessian=True))
    assert np.isfinite(r.chi2) and r.chi2 <= v


def test_chi2_value_mode_baseline_histograms_stay_single_pass():
    counts, ev = synth.histogram(1_000_000, events=1e8, seed=11)  # configs[2]: ~100 per bin
    plan = adc.Chi2Plan("gpoly", 6, adc.Histogram(1_000_000, -5.0, 5.0, ev, counts))
    resid, kappa = plan.value_mode()
    assert not resid and 50 < kappa < 256
