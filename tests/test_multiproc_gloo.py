"""Multi-rank host logic on CPU (world_size 2, gloo): each rank owns a range
of whole chunks (adc_chi2_make_layout), chunk records are exchanged with ONE
all_gather, every rank runs the fixed-order finalize (adc_chi2_finalize).
The result must be bitwise identical on every rank and to the single-rank
run, and match the reference formula (fit.cpp:224-259) within the reduction
tolerance.  The per-chunk records here come from a numpy restatement of the
record definition (include/adc_cuda.h) — the GPU produces them in bench.py /
tests/test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from conftest import ROOT  # noqa: E402


def gpoly_terms(x, q):
    z = (x - q[1]) / q[2]
    e = np.exp(-0.5 * z * z)
    m = q[0] * e + q[3] + q[4] * x + q[5] * x * x
    dz = (-0.5 * z) * (q[0] * e) + -0.5 * ((q[0] * e) * z)
    bg = np.stack([e, -(dz / q[2]), -((dz * z) / q[2]), np.ones_like(x), x, x * x])
    return m, bg


def chunk_records(counts, lo, hi, q, layout, chunk_begin, chunk_end):
    bins = counts.size
    chunk_bins = layout.tile_bins * layout.chunk_tiles
    recs = []
    for c in range(chunk_begin, chunk_end):
        a, b = c * chunk_bins, min(bins, (c + 1) * chunk_bins)
        j = np.arange(a, b, dtype=np.float64)
        x = lo + (j + 0.5) * ((hi - lo) / bins)
        m, bg = gpoly_terms(x, q)
        cc = counts[a:b]
        pos = cc > 0
        mc = np.where(pos, m / np.where(pos, cc, 1.0), 0.0)
        rec = [m.sum(), m[pos].sum(), (m * mc).sum(), cc[pos].sum()]
        rec += list(bg.sum(axis=1)) + list(bg[:, pos].sum(axis=1)) + list((bg * mc).sum(axis=1))
        recs.append(rec)
    return np.array(recs, dtype=np.float64).reshape(-1)


def _worker(rank, world, port, counts, q, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import paper_2203_06139_b200 as adc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = adc.chi2_layout(counts.size, world, rank)
    R = adc.record_len(6, True)
    mine = chunk_records(counts, -5.0, 5.0, q, L, L.chunk_begin, L.chunk_end)
    per = (L.nchunks + world - 1) // world
    buf = torch.zeros(per * R, dtype=torch.float64)
    buf[:mine.size] = torch.from_numpy(mine)
    gathered = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf)   # the one exchange step
    sizes = [adc.chi2_layout(counts.size, world, r) for r in range(world)]
    rec = np.concatenate([gathered[r].numpy()[:(s.chunk_end - s.chunk_begin) * R]
                          for r, s in enumerate(sizes)])
    g, c2 = adc.finalize(6, float(counts.sum()), rec, True)
    out_q.put((rank, g.tobytes(), c2))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_chi2_two_ranks_gloo_bitwise(restate):
    import sys
    sys.path.insert(0, ROOT)
    import paper_2203_06139_b200 as adc
    from paper_2203_06139_b200 import synth
    bins = 5 * (1 << 20) + 123              # 5 chunks of ~1 Mi bins (the last partial)
    counts, ev = synth.histogram(bins, events=2e8, seed=3)
    q = np.array(synth.GPOLY_INIT)
    L = adc.chi2_layout(bins)
    assert L.nchunks == 5  # odd: the two ranks own 2 and 3 chunks
    g1, c1 = adc.finalize(6, ev, chunk_records(counts, -5.0, 5.0, q, L, 0, L.nchunks), True)
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, counts, q, out_q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [out_q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, gb, c2 in res:
        assert np.frombuffer(gb).tobytes() == g1.tobytes(), rank
        assert c2 == c1
    ref, scale = restate.chi2_gradient_compensated("gpoly", counts, -5.0, 5.0, ev, q)
    assert np.all(np.abs(g1 - ref) <= 1e-12 * scale)
