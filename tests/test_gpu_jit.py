"""Generic lowering on the B200: every corpus gradient, called from a
Listing-style kernel, against the reference's own adc::launch on the same
inputs (tests/golden/jit_cases.npz, written by the unmodified reference).

Tolerances: per-point slots 1e-12 true-relative (the initial slot value in the
scale), bit-exact where the gradient uses only + - * / (rational, poly,
looped); forced hazardous kernels (atomic accumulation in an unspecified
order) 1e-9 relative to max|slot| (test_launch.cpp:165 precedent), except
sumn whose every thread adds identical values (bit-exact up to libm)."""
import numpy as np
import pytest

from conftest import golden, rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2203_06139_b200 as adc  # noqa: E402

G = golden("jit_cases.npz")
MODULE = str(G["module"])
EXACT = {"rational", "poly", "looped"}


def _run(key, device, counts=False, **kw):
    kern = str(G[f"{key}_kernel"])
    n = int(G[f"{key}_n"])
    unsafe = str(G[f"{key}_mode"]) == "unsafe"
    m = adc.JitModule(MODULE, kern, unsafe=unsafe, **kw)
    bufs = adc.BufferSet()
    arrays = []
    for i, (name, kind) in enumerate(m.params):
        v = G[f"{key}_in{i}"]
        if kind == "real[]":
            a = v.copy()
            if device:
                a = torch.from_numpy(a).cuda()
            bufs.arrays[name] = a
            arrays.append(name)
        elif kind == "real":
            bufs.scalars[name] = float(v)
        else:
            bufs.integers[name] = int(v)
    st = m.launch(adc.LaunchConfig(n // 256 + 1, 256, n), bufs, counts=counts)
    assert st.active == n
    outs = [bufs.arrays[a] for a in arrays]
    if device:
        torch.cuda.synchronize()
        outs = [o.cpu().numpy() for o in outs]
    return (outs, st) if counts else outs


@pytest.mark.parametrize("key", ["gauss", "rational", "branchy", "poly", "looped", "gsum",
                                 "sumn", "hess"])
@pytest.mark.parametrize("device", [True, False])
def test_corpus_gradient_matches_reference_launch(key, device):
    outs = _run(key, device)
    ins = [G[f"{key}_in{i}"] for i in range(int(G[f"{key}_nparams"]))]
    ins = [v for v in ins if v.ndim == 1]
    for i, (got, ref) in enumerate(zip(outs, [G[f"{key}_out{j}"] for j in range(len(outs))])):
        if key in EXACT:
            assert got.tobytes() == ref.tobytes(), (key, i)
        elif key == "gsum":
            assert np.abs(got - ref).max() <= 1e-9 * np.abs(ref).max(), (key, i)
        else:
            scale = np.maximum(np.maximum(np.abs(got), np.abs(ref)), np.abs(ins[i]))
            assert (np.abs(got - ref) <= 1e-12 * np.maximum(scale, 1e-300)).all(), (key, i)


@pytest.mark.parametrize("key", ["gauss", "rational", "branchy", "poly", "looped", "gsum",
                                 "sumn", "hess"])
@pytest.mark.parametrize("device", [True, False])
def test_launch_stats_equal_reference(key, device):
    """LaunchStats from the counting variant equal the reference launch's:
    the OpCounters sums over all threads (data-dependent branches and loops:
    branchy, looped, sumn) and every thread's kernel-frame statement count;
    the results are those of the plain variant."""
    outs, st = _run(key, device, counts=True)
    assert tuple(st.counts.values()) == tuple(int(v) for v in G[f"{key}_counts"])
    assert st.thread_statements.tobytes() == G[f"{key}_stm"].astype(np.uint32).tobytes()
    if key in EXACT:
        for i, got in enumerate(outs):
            assert got.tobytes() == G[f"{key}_out{i}"].tobytes(), (key, i)


def test_domain_error_is_eval():
    with pytest.raises(adc.AdcError) as e:
        _run("gauss_div0", True)
    assert e.value.kind == "Eval" and "division by zero" in str(e.value)
    assert "division by zero" in str(G["gauss_div0_error"])


def test_tape_deeper_than_default_capacity():
    """looped_grad with 300 iterations pushes more than the default 256 tape
    entries per thread.  The reference's tapes are unbounded: the host-buffer
    path redoes the launch from the caller's data with a larger tape (the same
    bits as the reference); a device-buffer launch reports the overflow as an
    Eval error naming the remedy."""
    outs, st = _run("looped_deep", False, counts=True)
    assert outs[-1].tobytes() == G["looped_deep_out1"].tobytes()
    assert tuple(st.counts.values()) == tuple(int(v) for v in G["looped_deep_counts"])
    with pytest.raises(adc.AdcError) as e:
        _run("looped_deep", True)
    assert e.value.kind == "Eval" and "tape capacity" in str(e.value)
    outs = _run("looped_deep", True, tape_capacity=1024)
    assert outs[-1].tobytes() == G["looped_deep_out1"].tobytes()


def test_integer_overflow_is_eval():
    # int64 arithmetic raises like the interpreter (eval.cpp:601-628)
    with pytest.raises(adc.AdcError) as e:
        _run("iovf", True)
    assert e.value.kind == "Eval" and "integer overflow" in str(e.value)
    assert "integer overflow" in str(G["iovf_error"])


def test_index_out_of_range_is_eval():
    m = adc.JitModule(MODULE, "k_sumn", unsafe=True)
    x = torch.zeros(64, dtype=torch.float64, device="cuda")
    dx = torch.zeros_like(x)
    with pytest.raises(adc.AdcError) as e:
        m.launch(adc.LaunchConfig(1, 32, 32),
                 adc.BufferSet(arrays={"x": x, "dx": dx}, integers={"n": 65}))
    assert e.value.kind == "Eval" and "index 64 out of range" in str(e.value)


def test_tape_capacity():
    n = 256
    x = torch.linspace(-2, 3, n, dtype=torch.float64, device="cuda")
    small = adc.JitModule(MODULE, "k_looped", tape_capacity=64)
    with pytest.raises(adc.AdcError) as e:
        small.launch(adc.LaunchConfig(1, n, n), adc.BufferSet(
            arrays={"x": x, "dx": torch.zeros_like(x)}, integers={"n": 100}))
    assert e.value.kind == "Eval" and "tape capacity" in str(e.value)
    big = adc.JitModule(MODULE, "k_looped")  # default: 256 entries per tape
    dx = torch.zeros_like(x)
    big.launch(adc.LaunchConfig(1, n, n), adc.BufferSet(arrays={"x": x, "dx": dx},
                                                        integers={"n": 100}))
    # d/dx of the loop: each step halves (s > 1) or maps s -> 1.5 s + x; finite, nonzero
    assert torch.isfinite(dx).all() and (dx != 0).any()


def test_launch_module_cache_and_compute_equivalence():
    # The JIT's gauss_grad_0_1 and the hand-written K1 agree within 1e-12
    # (K1 hoists the two pow() calls to the host libm).
    n = 100_003
    rng = np.random.Generator(np.random.PCG64(3))
    x, p = rng.uniform(-3, 3, n), rng.uniform(-2, 2, n)
    a = {"x": x.copy(), "p": p.copy(), "dx": np.zeros(n), "dp": np.zeros(n)}
    b = {"x": x.copy(), "p": p.copy(), "dx": np.zeros(n), "dp": np.zeros(n)}
    cfg = adc.LaunchConfig(n // 256 + 1, 256, n)
    adc.launch_module(MODULE, "k_gauss", cfg, adc.BufferSet(arrays=a, scalars={"sigma": 1.3}))
    adc.launch_module(MODULE, "k_gauss", cfg, adc.BufferSet(arrays=a, scalars={"sigma": 1.3}))
    adc.launch("compute", cfg, adc.BufferSet(arrays=b, scalars={"sigma": 1.3}))
    adc.launch("compute", cfg, adc.BufferSet(arrays=b, scalars={"sigma": 1.3}))
    assert rel_err(a["dx"], b["dx"]).max() <= 1e-12
    assert rel_err(a["dp"], b["dp"]).max() <= 1e-12
