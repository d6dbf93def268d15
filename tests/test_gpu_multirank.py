"""Native multi-GPU driver (include/adc_cuda.h, adc_comm): a sharded chi2 plan
with a communicator runs kernels + the record all-gather + the fixed-order
finalize inside the library, so gradient / chi2 / the batched line search /
the fit loop are bitwise identical to the single-device plan on every rank.

The box has one GPU: NCCL is exercised at world size 1 (same enqueue and
graph-capture code as at N > 1), and world sizes 2 and 3 run as separate
processes sharing the GPU over the host-callback transport (gloo) and over the
peer-memory transport (CUDA IPC buffers, GPU-side publish + flags)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402

from conftest import ROOT  # noqa: E402

BINS = 3 * (1 << 20) + 4321  # 3 chunks + a partial one -> uneven shards


def _problem(bins=BINS, seed=5):
    counts, ev = synth.histogram(bins, events=100.0 * bins, seed=seed)
    q = np.array(synth.GPOLY_INIT)
    g = np.array([1e3, -2e3, 5e2, 10.0, -3.0, 1.0])
    qs = np.stack([q - 2.0 ** -k * g for k in range(9)])
    return counts, ev, q, qs


def _results(plan, eng, h, q, qs):
    out = {}
    for k in range(3):  # eager first pass, then graph capture, then replay
        out[f"grad{k}"], out[f"c2g{k}"] = plan.gradient(q)
    out["c2"] = plan.chi2(q)
    out["multi"] = plan.chi2_multi(qs)
    out["gmulti"] = plan.gradient_multi(qs[:5])
    r = eng.fit(h, q, adc.FitOptions(budget=15, trace_iterates=6))
    out["fit_params"] = np.array(r.params)
    out["fit_chi2"] = r.chi2
    out["fit_its"] = np.array(r.iterates)
    r = eng.fit(h, q, adc.FitOptions(budget=3, use_hessian=True))
    out["newton_params"] = np.array(r.params)
    r = eng.fit(h, q, adc.FitOptions(budget=4, trace_iterates=5),
                provider=adc.GradientProvider.Numeric)
    out["numeric_its"] = np.array(r.iterates)
    return {k: np.asarray(v).tobytes() for k, v in out.items()}


def _single_device(counts, ev, q, qs):
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)
    return _results(adc.Chi2Plan("gpoly", 6, h), adc.FitEngine("gpoly", 6), h, q, qs)


def test_nccl_world1_bitwise_equals_single_device():
    counts, ev, q, qs = _problem()
    ref = _single_device(counts, ev, q, qs)
    comm = adc.Comm.nccl(1, 0, adc.Comm.unique_id())
    assert comm.info() == (1, 0, 1)
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)
    got = _results(adc.Chi2Plan("gpoly", 6, h, comm=comm), adc.FitEngine("gpoly", 6, comm=comm),
                   h, q, qs)
    for k in ref:
        assert got[k] == ref[k], k
    # one-call form for a rank holding only its shard
    L = adc.chi2_layout(counts.size, 1, 0)
    shard = torch.from_numpy(counts[L.bin_begin:L.bin_end].copy()).cuda()
    pl = adc.Chi2Plan.sharded("gpoly", 6, h, shard, comm)
    assert pl.gradient(q)[0].tobytes() == ref["grad0"][:48]
    pl.close()
    comm.close()


def test_peer_comm_world1_bitwise_equals_single_device():
    counts, ev, q, qs = _problem(bins=900_001, seed=12)
    ref = _single_device(counts, ev, q, qs)
    comm = adc.Comm.peer(1, 0, lambda a: a.copy())
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)
    got = _results(adc.Chi2Plan("gpoly", 6, h, comm=comm), adc.FitEngine("gpoly", 6, comm=comm),
                   h, q, qs)
    assert got == ref


def test_peer_fit_trace_grows_between_fits_on_one_plan():
    """The device fit loop on a peer-sharded plan reallocates only its iterate
    trace when a later fit asks for more iterates (the compact
    all-rank record buffers stay allocated; the rebuilt graph must not point
    at freed memory).  Each fit equals the single-device fit bit for bit."""
    counts, ev, q, _ = _problem(bins=600_001, seed=21)
    h1 = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)
    ref_eng = adc.FitEngine("gpoly", 6)
    comm = adc.Comm.peer(1, 0, lambda a: a.copy())
    h2 = adc.Histogram(counts.size, -5.0, 5.0, ev, counts.copy())
    eng = adc.FitEngine("gpoly", 6, comm=comm)
    for trace in (2, 10, 40, 5, 41):
        o = adc.FitOptions(budget=40, trace_iterates=trace)
        a, b = ref_eng.fit(h1, q, o), eng.fit(h2, q, o)
        assert np.array(a.params).tobytes() == np.array(b.params).tobytes(), trace
        assert np.array(a.iterates).tobytes() == np.array(b.iterates).tobytes(), trace
        assert a.chi2 == b.chi2 and a.iterations == b.iterations
    comm.close()


def test_host_comm_world1_identity():
    counts, ev, q, qs = _problem(bins=700_001, seed=8)
    ref = _single_device(counts, ev, q, qs)
    comm = adc.Comm.host(1, 0, lambda a: a.copy())
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)
    got = _results(adc.Chi2Plan("gpoly", 6, h, comm=comm), adc.FitEngine("gpoly", 6, comm=comm),
                   h, q, qs)
    assert got == ref


def test_sharded_plan_without_comm_is_refused():
    counts, ev, q, _ = _problem(bins=3 * (1 << 20), seed=2)
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)
    pl = adc.Chi2Plan("gpoly", 6, h, world=2, rank=1)
    with pytest.raises(adc.AdcError) as e:
        pl.gradient(q)
    assert e.value.kind == "Arg" and "communicator" in str(e.value)


def test_failing_host_callback_is_reported():
    counts, ev, q, _ = _problem(bins=100_000, seed=2)
    h = adc.Histogram(counts.size, -5.0, 5.0, ev, counts)

    def boom(_a):
        raise RuntimeError("link down")

    comm = adc.Comm.host(1, 0, boom)
    pl = adc.Chi2Plan("gpoly", 6, h, comm=comm)
    with pytest.raises(adc.AdcError) as e:
        pl.gradient(q)
    assert e.value.kind == "Nccl"


def _worker(rank, world, port, out_q, transport="host", bins=BINS):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_2203_06139_b200 as adc_
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        counts, ev, q, qs = _problem(bins)
        comm = adc_.Comm.from_torch(transport)
        h = adc_.Histogram(counts.size, -5.0, 5.0, ev, counts)
        L = adc_.chi2_layout(counts.size, world, rank)
        shard = torch.from_numpy(counts[L.bin_begin:L.bin_end].copy()).cuda()
        plan = adc_.Chi2Plan.sharded("gpoly", 6, h, shard, comm)
        res = _results(plan, adc_.FitEngine("gpoly", 6, comm=comm), h, q, qs)
        out_q.put((rank, res, None))
    except Exception as e:  # noqa: BLE001
        out_q.put((rank, None, repr(e)))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,transport,bins", [(2, "host", BINS), (3, "host", BINS),
                                                  (2, "peer", BINS), (3, "peer", BINS),
                                                  (3, "peer", 200_001)])
def test_ranks_share_gpu_bitwise(world, transport, bins):
    """Several ranks on the one GPU: the host transport (gloo all-gather) and
    the peer transport (CUDA IPC buffers on the device, GPU-side publish and
    flags — the multi-GPU path without NCCL) both give every rank the
    single-device bits; 200,001 bins over 3 ranks leaves a rank without
    chunks (it only takes part in the exchanges)."""
    import torch.multiprocessing as mp
    counts, ev, q, qs = _problem(bins)
    ref = _single_device(counts, ev, q, qs)
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out_q, transport, bins))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [out_q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, got, err in res:
        assert err is None, (rank, err)
        for k in ref:
            assert got[k] == ref[k], (rank, k)


def _absent_peer_worker(rank, world, port, out_q):
    import sys
    import time
    sys.path.insert(0, ROOT)
    os.environ["ADC_PEER_TIMEOUT_S"] = "3"
    import torch.distributed as dist
    import paper_2203_06139_b200 as adc_
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    err = None
    try:
        counts, ev, q, _ = _problem(BINS)
        comm = adc_.Comm.from_torch("peer")
        h = adc_.Histogram(counts.size, -5.0, 5.0, ev, counts)
        L = adc_.chi2_layout(counts.size, world, rank)
        shard = torch.from_numpy(counts[L.bin_begin:L.bin_end].copy()).cuda()
        plan = adc_.Chi2Plan.sharded("gpoly", 6, h, shard, comm)
        if rank == 0:  # rank 1 never runs the pass
            t0 = time.monotonic()
            try:
                plan.gradient(q)
                torch.cuda.synchronize()
            except Exception as e:  # noqa: BLE001
                err = (e.kind if hasattr(e, "kind") else type(e).__name__, time.monotonic() - t0)
        out_q.put((rank, err))
    except Exception as e:  # noqa: BLE001
        out_q.put((rank, ("setup", repr(e))))
    dist.barrier()
    os._exit(0)  # rank 0's CUDA context is gone after the trap


def test_absent_peer_fails_instead_of_hanging():
    """Peer transport: a rank whose peers never reach the pass gets an error
    after ADC_PEER_TIMEOUT_S (the flag wait traps) — it does not spin on the
    GPU forever."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_absent_peer_worker, args=(r, 2, port, out_q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(out_q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    assert res[1] is None
    assert res[0] is not None and res[0][0] != "setup", res[0]
    assert res[0][0] == "Cuda" and 2.5 < res[0][1] < 120, res[0]


# ---- shared mean vector over ranks (dp all-reduce) ---------------
def _sp_problem(dim=100, n=50_003, seed=3):
    rng = np.random.Generator(np.random.PCG64(seed))
    p = rng.uniform(-1, 1, dim)
    x = p[:, None] + 0.1 * rng.standard_normal((dim, n))
    dp0 = rng.standard_normal(dim)
    return x, p, dp0


def _sp_run(x, p, dp0, comm=None):
    X = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    P = torch.from_numpy(p).cuda()
    DX = torch.zeros_like(X)
    DP = torch.from_numpy(dp0.copy()).cuda()
    adc.launch_batch_shared_p("gaussnd_grad_0_1", X, P, 1.3, DX, DP,
                              adc.LaunchOptions(unsafe=True), comm=comm)
    torch.cuda.synchronize()
    return DX.cpu().numpy(), DP.cpu().numpy()


def test_shared_p_comm_world1_bitwise_equals_single_device():
    x, p, dp0 = _sp_problem()
    dx1, dp1 = _sp_run(x, p, dp0)
    for comm in (adc.Comm.nccl(1, 0, adc.Comm.unique_id()), adc.Comm.host(1, 0, lambda a: a.copy()),
                 adc.Comm.peer(1, 0, lambda a: a.copy())):
        dx, dp = _sp_run(x, p, dp0, comm)
        assert dx.tobytes() == dx1.tobytes() and dp.tobytes() == dp1.tobytes()
        comm.close()


def _sp_worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_2203_06139_b200 as adc_  # noqa: F401
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, p, dp0 = _sp_problem()
        n = x.shape[1]
        lo, hi = n * rank // world, n * (rank + 1) // world
        comm = adc_.Comm.from_torch("host")
        runs = [_sp_run(x[:, lo:hi], p, dp0, comm) for _ in range(2)]
        out_q.put((rank, runs[0][0].tobytes(), runs[0][1].tobytes(), runs[1][1].tobytes(), None))
    except Exception as e:  # noqa: BLE001
        out_q.put((rank, None, None, None, repr(e)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shared_p_ranks_share_gpu(restate, world):
    """Each rank holds a contiguous slice of the points and the same p: its dx
    rows are the single-device ones bit for bit, and every rank ends with the
    same dp — within 1e-12 * sum|terms| of the compensated total, repeatable."""
    import torch.multiprocessing as mp
    x, p, dp0 = _sp_problem()
    dx1, _ = _sp_run(x, p, dp0)
    tot, ab = restate.gaussnd_shared_p_dp_compensated(np.ascontiguousarray(x), p, 1.3)
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sp_worker, args=(r, world, port, out_q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([out_q.get(timeout=600) for _ in procs])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    n = x.shape[1]
    dps = set()
    for rank, dxb, dpb, dpb2, err in res:
        assert err is None, (rank, err)
        lo, hi = n * rank // world, n * (rank + 1) // world
        dx = np.frombuffer(dxb).reshape(x.shape[0], hi - lo)
        assert dx.tobytes() == np.ascontiguousarray(dx1[:, lo:hi]).tobytes()
        assert dpb == dpb2
        dps.add(dpb)
    assert len(dps) == 1
    dp = np.frombuffer(dps.pop())
    assert np.all(np.abs(dp - (dp0 + tot)) <= 1e-12 * (ab + np.abs(dp0)))


# ---- the forced compute_shared launch over ranks (the dsigma slot) ---------------
def _cs_problem(n=200_003, seed=9):
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-3, 3, n), rng.uniform(-2, 2, n)


def _cs_run(x, p, comm=None):
    n = x.size
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    X, P = t(x), t(p)
    DX, DP = torch.zeros_like(X), torch.zeros_like(X)
    DS = torch.full((1,), 0.25, dtype=torch.float64, device="cuda")
    adc.launch("compute_shared", adc.LaunchConfig(n // 256 + 1, 256, n),
               adc.BufferSet(arrays={"x": X, "p": P, "dx": DX, "dp": DP, "dsigma": DS},
                             scalars={"sigma": 1.3}),
               adc.LaunchOptions(unsafe=True), comm=comm)
    torch.cuda.synchronize()
    return DX.cpu().numpy(), DS.cpu().numpy()


def test_compute_shared_comm_world1_bitwise_equals_single_device():
    x, p = _cs_problem()
    dx1, ds1 = _cs_run(x, p)
    for comm in (adc.Comm.nccl(1, 0, adc.Comm.unique_id()), adc.Comm.host(1, 0, lambda a: a.copy())):
        dx, ds = _cs_run(x, p, comm)
        assert dx.tobytes() == dx1.tobytes() and ds.tobytes() == ds1.tobytes()
        comm.close()


def _cs_worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_2203_06139_b200 as adc_
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, p = _cs_problem()
        n = x.size
        lo, hi = n * rank // world, n * (rank + 1) // world
        comm = adc_.Comm.from_torch("peer")
        dx, ds = _cs_run(x[lo:hi], p[lo:hi], comm)
        out_q.put((rank, dx.tobytes(), ds.tobytes(), None))
    except Exception as e:  # noqa: BLE001
        out_q.put((rank, None, None, repr(e)))
    dist.barrier()
    dist.destroy_process_group()


def test_compute_shared_ranks_share_gpu(restate):
    """Two ranks (peer transport's callback), each with half the points: the
    same dsigma on both, within 1e-12 * sum|terms| of the compensated total;
    dx per point bit-identical to one device."""
    import torch.multiprocessing as mp
    x, p = _cs_problem()
    dx1, _ = _cs_run(x, p)
    tot, ab = restate.gauss_shared_dsigma_compensated(x, p, 1.3)
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cs_worker, args=(r, 2, port, out_q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted([out_q.get(timeout=600) for _ in procs])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    n = x.size
    dss = set()
    for rank, dxb, dsb, err in res:
        assert err is None, (rank, err)
        lo, hi = n * rank // 2, n * (rank + 1) // 2
        assert np.frombuffer(dxb).tobytes() == dx1[lo:hi].tobytes()
        dss.add(dsb)
    assert len(dss) == 1
    ds = np.frombuffer(dss.pop())[0]
    assert abs(ds - (0.25 + tot)) <= 1e-12 * (ab + 0.25)
