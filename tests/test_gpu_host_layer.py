"""Host layer on the GPU: the multi-GPU
host-buffer form, thread safety of the launch path (the reference's launch is
safe from several threads on distinct buffer sets), the
per-thread kernel selection, and the FitEngine plan cache following the
histogram it snapshots."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402
from paper_2203_06139_b200.launch import set_gaussnd_variant  # noqa: E402


def _soa(dim, n, seed):
    rng = np.random.default_rng(seed)
    p = rng.uniform(-2, 2, (dim, n))
    x = p + 0.1 * rng.standard_normal((dim, n))
    return x, p


@pytest.mark.parametrize("dim,n", [(100, 20_011), (3, 100_003), (150, 4_099)])
def test_multi_gpu_host_form_equals_single_device(dim, n):
    x, p = _soa(dim, n, dim)
    dx0, dp0 = np.full((dim, n), 0.25), np.full((dim, n), -0.5)
    a = (dx0.copy(), dp0.copy())
    b = (dx0.copy(), dp0.copy())
    adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, *a)
    adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, *b, devices=[0])
    assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()


def test_multi_gpu_listing1_equals_single_device():
    n = 1_000_003
    rng = np.random.default_rng(3)
    x, p = rng.uniform(-3, 3, n), rng.uniform(-2, 2, n)
    cfg = adc.LaunchConfig(n // 256 + 1, 256, n)
    outs = []
    for devices in (None, [0]):
        bufs = {"x": x, "p": p, "dx": np.zeros(n), "dp": np.zeros(n)}
        adc.launch("compute", cfg, adc.BufferSet(arrays=bufs, scalars={"sigma": 1.3}),
                   devices=devices)
        outs.append((bufs["dx"].tobytes(), bufs["dp"].tobytes()))
    assert outs[0] == outs[1]


def test_multi_gpu_bad_device_lists():
    x, p = _soa(4, 64, 1)
    for devs, msg in (([0, 0], "listed twice"), ([0, 4096], "does not exist")):
        with pytest.raises(adc.AdcError) as e:
            adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, np.zeros_like(x), np.zeros_like(x),
                             devices=devs)
        assert msg in str(e.value)


def test_threads_on_distinct_buffers_are_bitwise_sequential():
    """8 threads: host-buffer and device-buffer calls at once, each thread
    with its own buffers; one thread forces a different kernel (dims over the
    warps of a CTA, a regrouped forward sum) for itself only — the selection is
    per thread, so the others keep the auto kernel's bits."""
    dim, n = 100, 30_000
    x, p = _soa(dim, n, 7)
    ref = [np.zeros((dim, n)), np.zeros((dim, n))]
    adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, *ref)
    forced = [np.zeros((dim, n)), np.zeros((dim, n))]
    set_gaussnd_variant(2)
    try:
        adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, *forced)
    finally:
        set_gaussnd_variant(0)
    xd, pd = torch.from_numpy(x).cuda(), torch.from_numpy(p).cuda()
    results, errors = {}, []

    def work(t):
        try:
            for _ in range(3):
                if t % 2 == 0:
                    out = [np.zeros((dim, n)), np.zeros((dim, n))]
                    if t == 4:
                        set_gaussnd_variant(2)
                    adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, *out)
                    got = out
                else:
                    out = [torch.zeros((dim, n), dtype=torch.float64, device="cuda")
                           for _ in range(2)]
                    s = torch.cuda.Stream()
                    with torch.cuda.stream(s):
                        adc.launch_batch("gaussnd_grad_0_1", xd, pd, 1.3, *out)
                    s.synchronize()
                    got = [o.cpu().numpy() for o in out]
                results.setdefault(t, []).append(got)
        except Exception as ex:  # noqa: BLE001
            errors.append(repr(ex))
        finally:
            set_gaussnd_variant(0)

    th = [threading.Thread(target=work, args=(t,)) for t in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for t, runs in results.items():
        want = forced if t == 4 else ref
        for got in runs:
            assert got[0].tobytes() == want[0].tobytes(), t
            assert got[1].tobytes() == want[1].tobytes(), t


def test_fit_engine_follows_inplace_changes_of_device_counts():
    counts, ev = synth.histogram(200_000, events=2e7, seed=4)
    q = list(synth.GPOLY_INIT)
    dc = torch.from_numpy(counts.copy()).cuda()
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, dc)
    eng = adc.FitEngine("gpoly", 6)
    g0 = eng.chi2_gradient(h, q)
    dc[::7] += 3.0  # in place: the plan's 1/c and C0 must be rebuilt
    fresh = adc.FitEngine("gpoly", 6).chi2_gradient(
        adc.Histogram(counts.size, -5.0, 5.0, ev, dc.clone()), q)
    g1 = eng.chi2_gradient(h, q)
    assert g1.tobytes() == fresh.tobytes() and g1.tobytes() != g0.tobytes()


def test_fit_engine_freezes_host_counts():
    counts, ev = synth.histogram(50_000, events=5e6, seed=5)
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)
    eng = adc.FitEngine("gpoly", 6)
    eng.chi2(h, synth.GPOLY_INIT)
    with pytest.raises(ValueError):
        counts[0] = 1.0  # the snapshot would silently go stale
    h.events = ev + 100.0  # a reassigned field rebuilds the plan
    want = adc.FitEngine("gpoly", 6).chi2(adc.Histogram(counts.size, -5.0, 5.0, ev + 100.0,
                                                        counts.copy()), synth.GPOLY_INIT)
    assert eng.chi2(h, synth.GPOLY_INIT) == want
