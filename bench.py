"""Benchmark driver (contract in the task statement; workloads in DESIGN.md §5).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload gaussnd100|gaussnd1000|gauss1d|chi2|fit]
                    [--transport peer|nccl] [--no-configs] [--no-e2e]

Default workload (BASELINE.json configs[1]): batched reverse-mode gradient of
the 100-dim Gaussian over 10M points per GPU, FP64, structure-of-arrays,
inputs resident in HBM (32 GB per GPU >> the 126 MB L2, so no flush is needed
between steps).  A step = one launch of gaussnd_grad_0_1 over all points of
the rank.  Multi-GPU: points are independent, each rank owns its own 10M
points (weak scaling), no collective on the data path.

`--workload chi2` (BASELINE configs[4]) makes the line the chi2 fit gradient
over 1e8 bins, strong-scaled: the histogram is split into contiguous chunk
ranges over the ranks and every pass ends in the one exchange step inside the
library (an all-gather of the chunk records, then the same fixed-order
finalize on every rank); value = gradient passes of the whole histogram per
second.  `--workload fit` is configs[2] (1e6 bins, the fit loop).

Besides the headline, the default line carries `configs`: one compact record
per BASELINE config (value, roofline with the measured peak, cpu_baseline =
the unmodified reference on this box's host cores, parity against the oracle
at the config's full size), so every config is in the driver-parsed line.

`--gpus N` without torchrun re-executes itself under torch.distributed.run
(one process per GPU) and fails if the world size differs from N.

Rank 0 prints ONE JSON line.  `--impl reference` times the reference's own
CPU implementation (oracle/_ref/ref_tool over the unmodified reference
library) on the host cores instead.

The oracle (oracle/) is used here only as the checker (the `parity` blocks,
outside every timed region) and for the CPU baselines; the measured path is
libadc_b200.so alone.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
FP64_PROBE = os.path.join(ROOT, "build", "fp64_peak")
METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]

WORKLOADS = {
    # name: (dim, points per GPU, description)
    "gaussnd100": (100, 10_000_000, "N-dim Gaussian gradient gaussnd_grad_0_1, dim=100, "
                                    "10M points per GPU, FP64 SoA (BASELINE configs[1])"),
    "gaussnd1000": (1000, 1_000_000, "N-dim Gaussian gradient, dim=1000, 1M points per GPU "
                                     "(BASELINE configs[3])"),
    "gauss1d": (1, 1_000_000, "Listing-1 compute -> gauss_grad_0_1 over 1M points "
                              "(BASELINE configs[0])"),
    "chi2": (0, 100_000_000, "chi2 fit gradient, gpoly (Gaussian + quadratic background), 1e8 "
                             "bins split over the GPUs, one record all-gather per pass "
                             "(BASELINE configs[4])"),
    "fit": (0, 1_000_000, "chi2 fit of gpoly over 1e6 bins, fit loop of fit.cpp:315-425 "
                          "(BASELINE configs[2])"),
}
CHI2_BINS = 100_000_000
FIT_BINS = 1_000_000
REL_TOL = 1e-12  # per component, relative


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def traffic_for(key):
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(key)
    except Exception:
        return None


HBM_NOMINAL_GBS = 7700.0  # B200 HGX figure (B200_PROFILING.md)


def hbm_roofline(alg_bytes, kernel_ms, traffic_key):
    pk = peaks()
    achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9
    r = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
         "frac": achieved / pk["hbm_gbs"], "traffic": traffic_for(traffic_key),
         "algorithmic_bytes_per_launch": alg_bytes, "kernel_ms": kernel_ms,
         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if not pk.get("_fallback")
         else "fallback 6650 GB/s (B200_PROFILING.md)",
         "frac_of_nominal": achieved / HBM_NOMINAL_GBS}
    if r["frac"] > 1.0:
        r["note"] = ("above the measured copy peak: that peak is a 1:1 read:write stream and "
                     "read-heavier mixes (this path reads 2 bytes per byte written) run faster; "
                     "frac_of_nominal is against the 7.7 TB/s HGX figure")
    return r


_FP64 = None


def fp64_peak(device):
    """The FP64 pipe peak MEASURED on this box in this run (tools/fp64_peak.cu:
    DFMA chains over every SM, best of 5 launches).  Falls back to SMs x 64
    lanes x max clock only when the probe binary is missing."""
    global _FP64
    if _FP64 is None:
        try:
            r = subprocess.run([FP64_PROBE, str(device), "5"], capture_output=True, text=True,
                               timeout=120, check=True)
            _FP64 = json.loads(r.stdout.strip().splitlines()[-1])
            _FP64["source"] = "measured: build/fp64_peak (tools/fp64_peak.cu), this run"
        except Exception as ex:  # noqa: BLE001
            import torch
            sms = torch.cuda.get_device_properties(device).multi_processor_count
            mhz = peaks().get("sm_max_mhz", 1965.0)
            _FP64 = {"tinstr_s": sms * 64 * mhz * 1e6 / 1e12, "sm_mhz": mhz,
                     "source": f"theoretical {sms} SMs x 64 lanes x {mhz:.0f} MHz "
                               f"(probe unavailable: {repr(ex)[:80]})"}
    return _FP64


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region (NVML polled
    every 5 ms from a thread; nvidia-smi's own polling is too coarse for a
    sub-second region)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index, self.samples, self.reasons, self.max_mhz = index, [], set(), None
        self._stop = threading.Event()
        self._thread = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for nm, b in self.REASONS.items():
                            if bits & b:
                                self.reasons.add(nm)
                    except Exception:
                        pass
                    self._stop.wait(0.005)
            self._thread = threading.Thread(target=poll, daemon=True)
            self._thread.start()
        except Exception:
            self._thread = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=2)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "NVML, 5 ms polling"}


# ---------------------------------------------------------------------------- distributed
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def respawn_under_torchrun(gpus):
    """`python bench.py --gpus N` (no torchrun): one process per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__), *sys.argv[1:]]
    log("bench: re-executing under torch.distributed.run:", " ".join(cmd[1:6]))
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


BACKEND = "nccl"


def device_index(local):
    """One process per GPU; with --dist-backend gloo on a box with fewer GPUs
    than ranks (path testing only) ranks share devices round-robin."""
    import torch
    return local % max(1, torch.cuda.device_count())


def maybe_init_pg(world, local, backend="nccl"):
    import torch
    import torch.distributed as dist
    global BACKEND
    BACKEND = backend
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group(backend, device_id=torch.device("cuda", device_index(local)))
        else:
            dist.init_process_group(backend)
    return dist if world > 1 else None


def coll_device():
    """Collectives run on the GPU with NCCL, on host copies with gloo."""
    return "cuda" if BACKEND == "nccl" else "cpu"


def barrier_sync(dist):
    import torch
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
        torch.cuda.synchronize()


def max_over_ranks(dist, value):
    import torch
    if dist is None:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def event_time(fn, stream):
    import torch
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    fn()
    b.record(stream)
    return a, b


# ---------------------------------------------------------------------------- checker (oracle)
def rel_err(g, r):
    """|g - r| / max(|g|, |r|), denormal floor 1e-300."""
    import numpy as np
    g, r = np.asarray(g, dtype=np.float64), np.asarray(r, dtype=np.float64)
    den = np.maximum(np.maximum(np.abs(g), np.abs(r)), 1e-300)
    return float(np.max(np.abs(g - r) / den)) if g.size else 0.0


def parity_points(dim, x_sub, p_sub, dx_sub, dp_sub, stride, note):
    """Per-point parity of a subsample (every `stride`-th point) against the C
    restatement of the generated gradient (oracle/restate.c)."""
    import numpy as np
    from oracle import restate_lib
    rs = restate_lib.load()
    rdx, rdp = np.zeros_like(x_sub), np.zeros_like(x_sub)
    if dim == 1:
        rs.gauss_grad(x_sub, p_sub, 1.3, rdx, rdp)
    else:
        rs.gaussnd_grad(np.ascontiguousarray(x_sub), np.ascontiguousarray(p_sub), 1.3, rdx, rdp)
    e = max(rel_err(dx_sub, rdx), rel_err(dp_sub, rdp))
    return {"max_rel": e, "n_checked": int(x_sub.size), "tol": REL_TOL, "ok": e <= REL_TOL,
            "oracle": "oracle/restate.c (C restatement of the generated gradient)",
            "sample": note}


# ---------------------------------------------------------------------------- reference (CPU)
def run_ref_tool(args, timeout=900):
    r = subprocess.run([REF_TOOL, *map(str, args)], capture_output=True, text=True,
                       timeout=timeout, check=True)
    return json.loads(r.stdout.strip().splitlines()[-1])


def ref_points(workload, per_step=None):
    """The unmodified reference on the host: adc::launch(compute) for gauss1d,
    Program::eval(gaussnd_grad_0_1) on an nproc thread pool otherwise.
    Returns (pt*param/s, cores, sample text)."""
    dim = WORKLOADS[workload][0]
    if workload == "gauss1d":
        n = per_step or 1_000_000
        out = run_ref_tool(["gauss1d-bench", n, 1])
        return 2 * n / out["seconds"], out["workers"], \
            f"{n} points through adc::launch(compute) (default workers)"
    total = per_step or (200_000 if dim <= 100 else 20_000)
    uniq = min(total, 100_000 if dim <= 100 else 10_000)
    out = run_ref_tool(["gaussnd-bench", dim, uniq, total, 1.3, 42, 0])
    return total * 2 * dim / out["seconds"], out["workers"], \
        f"{total} points ({uniq} distinct) x dim {dim} through Program::eval(gaussnd_grad_0_1) " \
        f"on an nproc thread pool"


def ref_chi2_slice(bins):
    """The reference's chi2_gradient (fit.cpp:224-259; single-threaded, as it
    is) over a `bins`-bin slice.  Returns bins/s."""
    from paper_2203_06139_b200 import synth
    out = run_ref_tool(["chi2-bench", "gpoly", bins, 1, *synth.GPOLY_INIT])
    return bins / out["seconds"], out


def ref_port_points(dim, npts):
    """No reference build on this host: the C restatement, one core."""
    import numpy as np
    from oracle import restate_lib
    from paper_2203_06139_b200 import synth
    rs = restate_lib.load()
    if dim == 1:
        x, p = synth.points_1d(npts)
    else:
        x, p = synth.points_nd(dim, npts, seed=7)
    dx, dp = np.zeros_like(x), np.zeros_like(x)
    t0 = time.perf_counter()
    (rs.gauss_grad if dim == 1 else rs.gaussnd_grad)(x, p, 1.3, dx, dp)
    return npts * 2 * dim / (time.perf_counter() - t0)


def cpu_baseline_for(workload):
    cores = os.cpu_count()
    try:
        if workload in ("chi2", "fit"):
            if not os.path.exists(REF_TOOL):
                return {"error": "oracle/_ref/ref_tool not built"}
            sl = 2_000_000 if workload == "chi2" else FIT_BINS
            bps, out = ref_chi2_slice(sl)
            total = CHI2_BINS if workload == "chi2" else FIT_BINS
            return {"value": bps / total, "unit": "gradient passes/s", "cores": 1,
                    "kind": "reference",
                    "sample": f"one chi2_gradient pass over a {sl}-bin slice through the "
                              f"reference's FitEngine formula (ref_tool chi2-bench, single "
                              f"thread as fit.cpp:224-259 is), scaled to {total:.0e} bins "
                              f"(linear in bins): {out['seconds']:.2f} s",
                    "bins_per_s": bps}
        if os.path.exists(REF_TOOL):
            rate, workers, sample = ref_points(workload)
            return {"value": rate, "unit": "pt*param/s", "cores": workers, "kind": "reference",
                    "sample": sample}
        dim = WORKLOADS[workload][0]
        return {"value": ref_port_points(dim, 20000), "unit": "pt*param/s", "cores": 1,
                "kind": "port", "sample": "20000 points through oracle/restate.c, one core"}
    except Exception as ex:  # noqa: BLE001
        return {"error": repr(ex)[:200], "cores": cores}


def reference_arm(a, world, rank):
    """bench.py --impl reference: the reference's own CPU path on the host
    cores, same metric/unit/config as our arm, a bounded sample per step."""
    if rank != 0:
        return
    dim, npts, desc = WORKLOADS[a.workload]
    kind = "reference" if os.path.exists(REF_TOOL) else "port"
    rates, cores, sample = [], 1, ""
    for s in range(a.warmup + a.steps):
        if a.workload in ("chi2", "fit"):
            sl = 1_000_000 if a.workload == "chi2" else FIT_BINS // 4
            bps, out = ref_chi2_slice(sl)
            rate = bps / (CHI2_BINS if a.workload == "chi2" else FIT_BINS)
            sample = f"chi2_gradient over a {sl}-bin slice per step (single thread, as " \
                     "fit.cpp:224-259), scaled linearly to the full histogram"
        elif kind == "reference":
            per = 1_000_000 if a.workload == "gauss1d" else (100_000 if dim <= 100 else 10_000)
            rate, cores, sample = ref_points(a.workload, per)
        else:
            rate, cores = ref_port_points(max(dim, 1), 20000), 1
            sample = "20000 points through oracle/restate.c, one core"
        if s >= a.warmup:
            rates.append(rate)
    value = statistics.median(rates)
    unit = "gradient passes/s" if a.workload in ("chi2", "fit") else "pt*param/s"
    units_per_step = 1.0 if unit != "pt*param/s" else npts * 2 * max(dim, 1)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": unit,
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": units_per_step / value * 1e3, "higher_is_better": True,
        "scaling": "strong" if a.workload == "chi2" else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "sample_per_step": sample},
        "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- per-point configs
def make_points(workload, rank, dev):
    import torch
    dim, npts, _ = WORKLOADS[workload]
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    if workload == "gauss1d":
        x = torch.rand(npts, dtype=torch.float64, device=dev, generator=g) * 6 - 3
        p = torch.rand(npts, dtype=torch.float64, device=dev, generator=g) * 4 - 2
    else:
        spread = 0.1 if dim <= 100 else 0.03
        p = torch.rand((dim, npts), dtype=torch.float64, device=dev, generator=g) * 4 - 2
        x = p + spread * torch.randn((dim, npts), dtype=torch.float64, device=dev, generator=g)
    return x, p


def point_step(workload, x, p, dx, dp):
    import paper_2203_06139_b200 as adc
    n = x.shape[-1]
    if workload == "gauss1d":
        cfg = adc.LaunchConfig(n // 256 + 1, 256, n)
        bufs = adc.BufferSet(arrays={"x": x, "p": p, "dx": dx, "dp": dp}, scalars={"sigma": 1.3})
        return lambda: adc.launch("compute", cfg, bufs)
    return lambda: adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, dx, dp)


def points_parity(workload, x, p, dx, dp, step_fn_factory, stride):
    """One fresh launch on zeroed slots (outside any timed region), then every
    `stride`-th point against the oracle."""
    import torch
    dx.zero_()
    dp.zero_()
    step_fn_factory()()
    torch.cuda.synchronize()
    n = x.shape[-1]
    idx = torch.arange(0, n, stride, device=x.device)
    dim = WORKLOADS[workload][0]
    take = (lambda t: t[idx]) if dim == 1 else (lambda t: t[:, idx])
    h = [take(t).cpu().numpy() for t in (x, p, dx, dp)]
    return parity_points(dim, *h, stride, f"every {stride}th of {n} points "
                                          f"({h[0].shape[-1]} points x {max(dim, 1)} dims), one "
                                          "fresh launch on zeroed slots")


def bench_points(a, world, rank, local, dist):
    """Headline per-point config: device-resident timing, parity, e2e."""
    import torch

    dim, npts, desc = WORKLOADS[a.workload]
    dev = torch.device("cuda", local)
    x, p = make_points(a.workload, rank, dev)
    dx, dp = torch.zeros_like(x), torch.zeros_like(x)
    stream = torch.cuda.current_stream(dev)
    step = point_step(a.workload, x, p, dx, dp)
    for _ in range(a.warmup):
        step()
    barrier_sync(dist)
    evs = []
    with ClockSampler(local) as clocks:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for _ in range(a.steps):
            evs.append(event_time(step, stream))
        t_end.record(stream)
        barrier_sync(dist)
    elapsed_ms = max_over_ranks(dist, t_start.elapsed_time(t_end))
    kernel_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    units = npts * 2 * max(dim, 1)
    value = world * units * a.steps / (elapsed_ms * 1e-3)
    roof = hbm_roofline(48 * npts * max(dim, 1), statistics.mean(kernel_ms), a.workload)
    roof["kernel_ms_min"] = min(kernel_ms)
    parity = None
    if not a.no_parity:
        parity = points_parity(a.workload, x, p, dx, dp,
                               lambda: point_step(a.workload, x, p, dx, dp), 997)
    del dx, dp
    e2e = None if a.no_e2e else bench_points_e2e(a, world, dist, x, p, units)
    return {"value": value, "ms_per_step": elapsed_ms / a.steps, "roofline": roof,
            "parity": parity, "e2e": e2e, "clocks": clocks.summary(), "desc": desc,
            "dim": dim, "npts": npts}


def bench_points_e2e(a, world, dist, x, p, units):
    """The public API with pinned HOST buffers: H2D of the step's inputs and
    slots, the kernel, D2H of the slots, all inside the timing."""
    import torch
    import paper_2203_06139_b200 as adc
    dim, npts, _ = WORKLOADS[a.workload]
    need = 4 * 8 * npts * max(dim, 1)
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = None
    if avail is not None and avail < 1.25 * need * world:
        return {"value": None, "unit": "pt*param/s",
                "skipped": f"host RAM {avail / 1e9:.0f} GB < {1.25 * need * world / 1e9:.0f} GB "
                           f"needed to pin {world} x {need / 1e9:.0f} GB"}
    hx = torch.empty(x.shape, dtype=torch.float64, pin_memory=True)
    hp = torch.empty(x.shape, dtype=torch.float64, pin_memory=True)
    hx.copy_(x)
    hp.copy_(p)
    hdx = torch.zeros(hx.shape, dtype=torch.float64, pin_memory=True)
    hdp = torch.zeros(hx.shape, dtype=torch.float64, pin_memory=True)
    nx, npp, ndx, ndp = hx.numpy(), hp.numpy(), hdx.numpy(), hdp.numpy()
    if a.workload == "gauss1d":
        cfg = adc.LaunchConfig(npts // 256 + 1, 256, npts)
        hb = adc.BufferSet(arrays={"x": nx, "p": npp, "dx": ndx, "dp": ndp},
                           scalars={"sigma": 1.3})
        hstep = lambda: adc.launch("compute", cfg, hb)  # noqa: E731
    else:
        hstep = lambda: adc.launch_batch("gaussnd_grad_0_1", nx, npp, 1.3, ndx, ndp)  # noqa
    hstep()
    e2e_steps = max(1, min(a.steps, a.e2e_steps))
    barrier_sync(dist)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        hstep()
    dt = max_over_ranks(dist, time.perf_counter() - t0)
    out = {"value": world * units * e2e_steps / dt, "unit": "pt*param/s",
           "h2d_bytes_per_step": 4 * 8 * npts * max(dim, 1),
           "d2h_bytes_per_step": 2 * 8 * npts * max(dim, 1), "steps": e2e_steps,
           "path": "launch_batch/launch with pinned numpy buffers -> adc_cuda_*_host (chunked "
                   "H2D/kernel/D2H over two streams)"}
    del hx, hp, hdx, hdp
    return out


def config_points(workload, local, steps=20, warm=3):
    """A secondary per-point config as one compact record."""
    import torch
    dim, npts, desc = WORKLOADS[workload]
    dev = torch.device("cuda", local)
    x, p = make_points(workload, 99, dev)
    dx, dp = torch.zeros_like(x), torch.zeros_like(x)
    step = point_step(workload, x, p, dx, dp)
    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    evs = [event_time(step, stream) for _ in range(steps)]
    torch.cuda.synchronize()
    ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in evs)
    units = npts * 2 * max(dim, 1)
    rec = {"workload": desc, "value": units / (ms * 1e-3), "unit": "pt*param/s", "api_ms": ms}
    kms = ms
    if workload == "gauss1d":
        # 48 MB fits in L2 and the API call's host work (validation, race
        # check, registry lookup) is longer than the kernel: the kernel alone
        # from CUDA graphs of K x [L2 flush, the call] minus K x [L2 flush]
        # (no graph-launch latency in the difference).  The flush writes
        # 512 MB and then reads another 256 MB, so every replay starts from
        # HBM with clean L2 lines (a write-only flush leaves dirty lines whose
        # write-backs would compete with the kernel).
        K = 10
        flush_w = torch.empty(64 << 20, dtype=torch.float64, device=dev)
        flush_r = torch.ones(32 << 20, dtype=torch.float64, device=dev)
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            step()
            flush_w.fill_(1.0)
            flush_r.sum()
        torch.cuda.synchronize()
        graphs = {}
        for with_call in (True, False):
            g_ = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_, stream=side):
                for _ in range(K):
                    flush_w.fill_(1.0)
                    flush_r.sum()
                    if with_call:
                        step()
            graphs[with_call] = g_
        torch.cuda.synchronize()
        tt = {True: [], False: []}
        for _ in range(steps):
            for with_call in (True, False):
                e0, e1 = event_time(graphs[with_call].replay, stream)
                torch.cuda.synchronize()
                tt[with_call].append(e0.elapsed_time(e1))
        kms = (statistics.median(tt[True]) - statistics.median(tt[False])) / K
        rec.update({"value": units / (kms * 1e-3), "api_value": units / (ms * 1e-3),
                    "note": "value: the kernel alone, from CUDA graphs of 10 x [L2 flush (512 MB "
                            "write + 256 MB read), the call] minus the same without the call; "
                            "api_*: CUDA events around each public-API call"})
        del flush_w, flush_r, graphs
    else:
        rec["note"] = f"device-resident, CUDA events around each public-API call; inputs " \
                      f"{32 * npts * dim / 1e9:.0f} GB >> L2"
    rec["kernel_ms"] = kms
    rec["roofline"] = hbm_roofline(48 * npts * max(dim, 1), kms, workload)
    rec["parity"] = points_parity(workload, x, p, dx, dp,
                                  lambda: point_step(workload, x, p, dx, dp),
                                  1 if workload == "gauss1d" else 997)
    return rec


# ---------------------------------------------------------------------------- chi2 configs
def chi2_roofline(bins, ms, device):
    """FP64-pipe roofline of the chi2 gradient pass's dominant kernel (the
    tile kernel, timed alone): executed FP64 instructions per bin (ncu,
    profiles/traffic.json chi2_1e8_fp64_per_bin) x bins / its duration, over
    the FP64 peak measured in this run (DFMA chains); beside it SURVEY.md
    §8(d)'s W = 62 for the exp-per-bin algorithm, and the kernel's HBM
    fraction (800 MB of 1/c per pass: the kernel is close to both roofs)."""
    pk = fp64_peak(device)
    peak = pk["tinstr_s"]
    w = traffic_for("chi2_1e8_fp64_per_bin") or 62.0
    achieved = w * bins / (ms * 1e-3) / 1e12
    w62 = 62.0 * bins / (ms * 1e-3) / 1e12
    hbm = 8.0 * bins / (ms * 1e-3) / 1e9
    return {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "T FP64 instr/s",
            "frac": achieved / peak, "traffic": traffic_for("chi2_1e8"),
            "hbm_frac": hbm / peaks()["hbm_gbs"],
            "work_per_bin": f"{w:g} FP64 instr executed (ncu; profiles/traffic.json)",
            "w62_equivalent": {"achieved": w62, "frac": w62 / peak},
            "peak_source": pk.get("source"), "peak_probe_sm_mhz": pk.get("sm_mhz"),
            "kernel_ms": ms}


def chi2_parity(h, q, grad, c2):
    """The 1e8-bin gradient and value against the Neumaier-compensated C
    restatement of fit.cpp:206-259 over every bin (reduction
    tolerance 1e-12 * sum_j |w_j dm_j/dq_i|)."""
    import numpy as np
    from oracle import restate_lib
    rs = restate_lib.load()
    counts = h.counts.cpu().numpy() if hasattr(h.counts, "cpu") else np.asarray(h.counts)
    ref, scale = rs.chi2_gradient_compensated("gpoly", counts, h.lo, h.hi, h.events, q)
    cref, cscale = rs.chi2_compensated("gpoly", counts, h.lo, h.hi, h.events, q)
    g = np.asarray(grad)
    norm = float(np.max(np.abs(g - ref) / scale))
    return {"max_rel": norm, "n_checked": int(counts.size), "tol": REL_TOL,
            "ok": bool(norm <= REL_TOL and abs(c2 - cref) <= REL_TOL * cscale),
            "metric": "max_i |g_i - r_i| / sum_j |w_j dm_j/dq_i| (reduction tolerance)",
            "grad_max_rel_componentwise": rel_err(g, ref),
            "chi2_rel": abs(c2 - cref) / abs(cref),
            "oracle": "oracle/restate.c rs_chi2_gradient_compensated over every bin"}


def bench_chi2(a, world, rank, local, dist, passes=20, warm=3, parity=True, clocks=None):
    """chi2 fit gradient over 1e8 bins (BASELINE configs[4]); per rank a shard
    of whole chunks, one all-gather of the chunk records per pass."""
    import torch
    import paper_2203_06139_b200 as adc
    from paper_2203_06139_b200 import synth

    dev = torch.device("cuda", local)
    bins = CHI2_BINS
    # counts ~ Poisson(E m_j / S) at the gpoly truth, sampled on the device
    # (counter-based: the same histogram on every rank), every 100th bin 0
    h = adc.sample_histogram("gpoly", synth.GPOLY_TRUTH, bins, -5.0, 5.0, bins * 100.0, seed=77,
                             zero_every=100, device=dev)
    q = list(synth.GPOLY_INIT)
    comm, transport = None, "none"
    if world > 1:
        order = [a.transport] if a.transport else (["peer", "nccl"] if BACKEND == "nccl"
                                                   else ["peer", "host"])
        for transport in order:
            try:
                comm = adc.Comm.from_torch(transport)
                plan = adc.Chi2Plan("gpoly", 6, h, comm=comm)
                break
            except Exception as ex:  # noqa: BLE001
                log(f"bench: transport {transport} unavailable: {ex!r}"[:200])
                comm = None
        if comm is None:
            raise RuntimeError("no multi-GPU transport")
    else:
        plan = adc.Chi2Plan("gpoly", 6, h)
    L = plan.layout
    R = adc.record_len(6, True)
    loc = torch.zeros(max(1, L.chunk_end - L.chunk_begin) * R, dtype=torch.float64, device=dev)
    for _ in range(warm):
        plan.gradient(q)
    barrier_sync(dist)
    t0 = time.perf_counter()
    for _ in range(passes):
        grad, c2 = plan.gradient(q)
    dt = max_over_ranks(dist, time.perf_counter() - t0) / passes
    # device time of this rank's pass kernels (tile + chunk): adc_cuda_chi2_partials
    # enqueues on the plan's user stream, torch's current stream at creation
    kt = []
    for _ in range(7):
        e0, e1 = event_time(lambda: plan.partials(q, True, loc), torch.cuda.current_stream(dev))
        torch.cuda.synchronize()
        kt.append(e0.elapsed_time(e1))
    kms = statistics.median(kt[1:])
    # the dominant kernel alone (the tile kernel; CUDA events inside the
    # library around its launch on the pass stream): the roofline's time
    tk = [plan.tile_kernel_ms(q, True, loc) for _ in range(7)]
    tms = statistics.median(tk[1:])
    # the paper's Fig. 2 comparison: the Numeric provider's pass on the same plan
    plan.set_provider(adc.GradientProvider.Numeric)
    nt = []
    for _ in range(5):
        e0, e1 = event_time(lambda: plan.partials(q, True, loc), torch.cuda.current_stream(dev))
        torch.cuda.synchronize()
        nt.append(e0.elapsed_time(e1))
    plan.set_provider(adc.GradientProvider.AdReverse)
    rec = {"workload": WORKLOADS["chi2"][2], "value": 1.0 / dt,
           "unit": "gradient passes/s", "ms_per_pass": dt * 1e3, "n_gpus": world,
           "bins": bins, "bins_per_rank": L.bin_end - L.bin_begin,
           "device_ms_per_rank_pass": kms,
           "collective": ("all-gather of chunk records inside libadc_b200 ("
                          + {"peer": "GPU-to-GPU stores into IPC-shared buffers + flags, fused "
                                     "into the chunk-reduce kernel",
                             "nccl": "ncclAllGather in the pass graph",
                             "host": "host transport over gloo"}[transport] + ")")
           if world > 1 else "none",
           "tile_kernel_ms": tms,
           "roofline": chi2_roofline(L.bin_end - L.bin_begin, tms, local),
           "numeric_provider_device_ms": statistics.median(nt[1:]),
           "ad_over_numeric_speedup": statistics.median(nt[1:]) / kms,
           "chi2": c2, "d2h_bytes_per_pass": 8 * R * L.nchunks}
    if parity and rank == 0:
        rec["parity"] = chi2_parity(h, q, grad, c2)
    plan.close()
    if comm is not None:
        comm.close()
    del h, loc
    torch.cuda.empty_cache()
    return rec


def bench_fit(local):
    """BASELINE configs[2]: chi2 fit of the Gaussian + quadratic background
    over 1e6 bins with the fit loop of fit.cpp:315-425 (GD + Armijo, and the
    Newton option), run by adc_cuda_fit as one device-resident CUDA graph."""
    import numpy as np
    import paper_2203_06139_b200 as adc
    from oracle import restate_lib
    from paper_2203_06139_b200 import synth
    counts, ev = synth.histogram(FIT_BINS, events=1e8, seed=11)
    h = adc.Histogram(FIT_BINS, -5.0, 5.0, ev, counts)
    eng = adc.FitEngine("gpoly", 6)
    q0 = list(synth.GPOLY_INIT)
    eng.chi2(h, q0)  # upload + graph capture outside the timing
    eng.chi2_gradient(h, q0)
    eng.fit(h, q0, adc.FitOptions(budget=2, use_hessian=True))
    eng.fit(h, q0, adc.FitOptions(budget=2))
    # gradient passes/s: the plan's pass (graph replay incl. the 21-double copy back)
    reps = 200
    t0 = time.perf_counter()
    for _ in range(reps):
        g = eng.chi2_gradient(h, q0)
    pass_s = (time.perf_counter() - t0) / reps
    rec = {"workload": WORKLOADS["fit"][2], "value": 1.0 / pass_s, "unit": "gradient passes/s",
           "ms_per_pass": pass_s * 1e3, "timed_passes": reps}
    # the pass's dominant kernel alone (CUDA events inside the library around
    # the tile kernel), against SURVEY.md §8(d)'s W = 62 per bin (the
    # exp-per-bin algorithm; this kernel runs 16 bins per thread per tile, one
    # wave of 245 tiles: latency- and tail-bound, not throughput-bound)
    plan = eng._plan(h)
    tk = [plan.tile_kernel_ms(q0) for _ in range(9)]
    tms = statistics.median(tk[1:])
    pk = fp64_peak(local)
    achieved = 62.0 * FIT_BINS / (tms * 1e-3) / 1e12
    rec["tile_kernel_ms"] = tms
    rec["d2h_bytes_per_pass"] = 8 * (4 + 3 * 6) * plan.layout.nchunks  # the chunk records
    rec["roofline"] = {"bound": "fp64", "achieved": achieved, "peak": pk["tinstr_s"],
                       "unit": "T FP64 instr/s", "frac": achieved / pk["tinstr_s"],
                       "hbm_frac": 8.0 * FIT_BINS / (tms * 1e-3) / 1e9 / peaks()["hbm_gbs"],
                       "traffic": None, "work_per_bin": "62 FP64 instr (SURVEY.md §8(d), the "
                       "exp-per-bin algorithm)", "bins_per_thread": plan.layout.tile_bins // 256,
                       "peak_source": pk.get("source"),
                       "kernel_ms": tms,
                       "note": "1e6 bins = 8 MB: a few-microsecond kernel, launch- and "
                               "tail-bound; the pass itself (graph replay, 21-double copy back, "
                               "host finalize) is ms_per_pass"}
    for name, hess in (("newton_numeric_hessian", True), ("gd_armijo", False)):
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            r = eng.fit(h, q0, adc.FitOptions(budget=400, use_hessian=hess))
            ts.append(time.perf_counter() - t0)
        rec[name] = {"fit_seconds": statistics.median(ts), "iterations": r.iterations,
                     "converged": r.converged, "gradient_evals": r.gradient_evals,
                     "chi2_evals": r.chi2_evals, "chi2": r.chi2,
                     "mu_sigma": [round(r.params[1], 6), round(r.params[2], 6)]}
    rec["note"] = ("newton: time to convergence; gd_armijo: the reference's steepest descent, "
                   "which does not converge on this histogram within its 400-iteration budget "
                   "(faithful to fit.cpp:315-425)")
    # parity of the pass at the init point against the compensated oracle
    rs = restate_lib.load()
    ref, scale = rs.chi2_gradient_compensated("gpoly", counts, -5.0, 5.0, ev, q0)
    cref, cscale = rs.chi2_compensated("gpoly", counts, -5.0, 5.0, ev, q0)
    c2 = eng.chi2(h, q0)
    norm = float(np.max(np.abs(np.asarray(g) - ref) / scale))
    rec["parity"] = {"max_rel": norm, "n_checked": FIT_BINS, "tol": REL_TOL,
                     "ok": bool(norm <= REL_TOL and abs(c2 - cref) <= REL_TOL * cscale),
                     "chi2_rel": abs(c2 - cref) / abs(cref),
                     "metric": "max_i |g_i - r_i| / sum_j |w_j dm_j/dq_i|",
                     "oracle": "oracle/restate.c (compensated) over every bin"}
    # the reference on the same histogram: one chi2_gradient + one chi2 pass
    if os.path.exists(REF_TOOL):
        try:
            with tempfile.TemporaryDirectory() as td:
                cf, of = os.path.join(td, "c.bin"), os.path.join(td, "o.bin")
                counts.astype(np.float64).tofile(cf)
                out = run_ref_tool(["chi2-in", "gpoly", FIT_BINS, -5.0, 5.0, cf, of, 1, *q0])
                refv = np.fromfile(of, dtype=np.float64)
            tg, tc = out["grad_seconds"], out["chi2_seconds"]
            rn = rec["newton_numeric_hessian"]
            rec["cpu_baseline"] = {
                "value": 1.0 / tg, "unit": "gradient passes/s", "cores": 1, "kind": "reference",
                "sample": f"one chi2_gradient ({tg:.2f} s) and one chi2 ({tc:.2f} s) pass of the "
                          "reference's FitEngine formula over the same 1e6-bin histogram "
                          "(ref_tool chi2-in, single thread as fit.cpp:224-259 is)",
                "newton_fit_seconds_extrapolated": rn["gradient_evals"] * tg + rn["chi2_evals"] * tc,
                "extrapolation": "our Newton fit's gradient/chi2 pass counts x the reference's "
                                 "per-pass times (the reference fit itself would take minutes)"}
            rec["parity"]["vs_reference_grad_max_rel"] = rel_err(g, refv[1:])
            rec["parity"]["vs_reference_chi2_rel"] = abs(c2 - refv[0]) / abs(refv[0])
        except Exception as ex:  # noqa: BLE001
            rec["cpu_baseline"] = {"error": repr(ex)[:200]}
    return rec


def bench_jit(local, npts=100_000_000, steps=10, warm=3):
    """Generic lowering (DSL -> CUDA -> NVRTC sm_100a):
    the reference corpus gradients rational_grad (no tape) and looped_grad
    (n = 10: tape entries in registers, the static-tape variant) called from
    Listing-style kernels over 1e8 points; 48 / 24 B per point."""
    import numpy as np
    import torch
    import paper_2203_06139_b200 as adc
    module = str(np.load(os.path.join(ROOT, "tests", "golden", "jit_cases.npz"))["module"])
    dev = torch.device("cuda", local)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    x = torch.rand(npts, dtype=torch.float64, device=dev, generator=g) * 4 - 2
    y = torch.rand(npts, dtype=torch.float64, device=dev, generator=g) * 4 - 2
    dx, dy = torch.zeros_like(x), torch.zeros_like(x)
    cfg = adc.LaunchConfig(npts // 256 + 1, 256, npts)
    stream = torch.cuda.current_stream(dev)
    rec = {"workload": "generic JIT: corpus gradients over 1e8 points (launch incl. the per-launch "
                       "error-word check)"}
    for kern, bufs, bytes_pt, ints in (
            ("k_rational", adc.BufferSet(arrays={"x": x, "y": y, "dx": dx, "dy": dy}), 48, []),
            ("k_looped", adc.BufferSet(arrays={"x": x, "dx": dx}, integers={"n": 10}), 24, [10])):
        mod = adc.JitModule(module, kern)
        step = lambda: mod.launch(cfg, bufs)  # noqa: E731
        for _ in range(warm):
            step()
        torch.cuda.synchronize()
        evs = [event_time(step, stream) for _ in range(steps)]
        torch.cuda.synchronize()
        ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in evs)
        roof = hbm_roofline(bytes_pt * npts, ms, "jit_" + kern)
        slots = traffic_for("jit_k_looped_fp64_warp_instr_per_pt") if kern == "k_looped" else None
        if slots:
            # k_looped is bound by the FP64 pipe, not HBM (ncu: pipe active 91%,
            # HBM 60%): 10 data-dependent branches per point leave part of each
            # warp's lanes predicated off, so the pipe's work is counted in
            # lane slots (warp instructions x 32), not executed thread-instructions
            pk = fp64_peak(local)
            lanes = slots * 32 * npts / (ms * 1e-3) / 1e12
            roof = {"bound": "fp64", "achieved": lanes, "peak": pk["tinstr_s"],
                    "unit": "T FP64 lane-slots/s", "frac": lanes / pk["tinstr_s"],
                    "hbm_frac": roof["frac"], "traffic": roof["traffic"],
                    "work_per_point": f"{slots:g} FP64 warp instructions x 32 lanes; "
                                      f"{traffic_for('jit_k_looped_fp64_thread_instr_per_pt'):g} "
                                      "executed thread-instructions (ncu, profiles/traffic.json)",
                    "kernel_ms": ms, "peak_source": pk["source"]}
        rec[kern] = {"ms_per_launch": ms, "static_tape": mod.static_source(ints) is not None,
                     "roofline": roof}
    return rec


def bench_fig2b(local):
    """The paper's Fig. 2b (the reference's bench_scaling, fit.cpp:427-458) at
    B200 scale: gsum fits with K = 1, 2, 4, 8 Gaussians (3K parameters) over
    1e6 bins with each gradient provider; per gradient evaluation (wall,
    host included)."""
    import paper_2203_06139_b200 as adc
    rows = adc.bench_scaling(k_list=(1, 2, 4, 8), bins=1_000_000, events=1e8, seed=42, repeats=3)
    table = {}
    for r in rows:
        t = table.setdefault(str(r.params), {})
        t[r.provider] = round(r.median_wall_ns / 1e6 / max(1, r.grad_evals), 5)
    for t in table.values():
        if "ad-reverse" in t and "numeric" in t:
            t["numeric_over_ad"] = round(t["numeric"] / t["ad-reverse"], 3)
    return {"workload": "Fig. 2b analog: bench_scaling gsum K=1,2,4,8 over 1e6 bins, ms per "
                        "gradient evaluation by provider (keys: parameter count)", "params": table}


# ---------------------------------------------------------------------------- our arm
def ours_arm(a, world, rank, local):
    import torch
    local = device_index(local)
    torch.cuda.set_device(local)
    dist = maybe_init_pg(world, local, a.dist_backend)
    import paper_2203_06139_b200  # noqa: F401  (fails loudly without the CUDA library)

    if a.workload in ("chi2", "fit"):
        line = chi2_headline(a, world, rank, local, dist)
    else:
        line = points_headline(a, world, rank, local, dist)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist_
        dist_.barrier()
        dist_.destroy_process_group()


def common_line(a, world, value, unit, ms_step, scaling):
    return {"metric": METRIC, "value": value, "unit": unit, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64"}


def points_headline(a, world, rank, local, dist):
    r = bench_points(a, world, rank, local, dist)
    configs = {}
    if not a.no_configs:
        # the chi2 config at every world size (strong-scaled, the one with an
        # exchange step); the single-GPU configs on rank 0's GPU at N = 1
        jobs = [("cfg5_chi2_1e8", lambda: bench_chi2(a, world, rank, local, dist))]
        if world == 1:
            jobs = [("cfg1_gauss1d_1M", lambda: config_points("gauss1d", local)),
                    ("cfg3_fit_1e6", lambda: bench_fit(local)),
                    ("cfg4_gaussnd1000_1M", lambda: config_points("gaussnd1000", local))] + jobs
            jobs.append(("jit_corpus", lambda: bench_jit(local)))
            jobs.append(("fig2b_bench_scaling", lambda: bench_fig2b(local)))
        for name, job in jobs:
            try:
                configs[name] = job()
            except Exception as ex:  # a secondary record never hides the headline
                configs[name] = {"error": repr(ex)[:300]}
            log(f"bench: {name} done")
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline_for(a.workload)
        for name, wl in (("cfg1_gauss1d_1M", "gauss1d"), ("cfg4_gaussnd1000_1M", "gaussnd1000"),
                         ("cfg5_chi2_1e8", "chi2")):
            if name in configs and "error" not in configs[name]:
                configs[name]["cpu_baseline"] = cpu_baseline_for(wl)
    if rank != 0:
        return None
    line = common_line(a, world, r["value"], "pt*param/s", r["ms_per_step"], "weak")
    line.update({
        "data": "synthetic (device Philox RNG: p~U(-2,2), x=p+0.1*N(0,1), sigma=1.3)",
        "config": {"workload": r["desc"], "dim": r["dim"], "points_per_gpu": r["npts"],
                   "layout": "structure-of-arrays x[d*n+i]",
                   "l2": f"inputs {4 * 8 * r['npts'] * max(r['dim'], 1) / 1e9:.1f} GB per GPU >> "
                         "126 MB L2; no flush needed",
                   "parallelism": f"dp{world} (points sharded, no collective)"},
        "roofline": r["roofline"], "cpu_baseline": cpu, "e2e": r["e2e"], "parity": r["parity"],
        "gpu_launches": a.steps, "clocks": r["clocks"], "configs": configs})
    if "cfg5_chi2_1e8" in configs:
        c = configs["cfg5_chi2_1e8"]
        line["chi2_1e8"] = {k: c.get(k) for k in ("value", "unit", "n_gpus", "ms_per_pass")}
        if "roofline" in c:
            line["chi2_1e8"]["fp64_frac"] = c["roofline"]["frac"]
    return line


def chi2_headline(a, world, rank, local, dist):
    """--workload chi2 / fit: the chi2 pass is the line."""
    import torch
    if a.workload == "fit":
        with ClockSampler(local) as clocks:
            rec = bench_fit(local) if rank == 0 else None
        if rank != 0:
            return None
        line = common_line(a, world, rec["value"], "gradient passes/s", rec["ms_per_pass"],
                           "weak")
        line.update({"data": "synthetic (numpy Poisson histogram at the gpoly truth, every 100th "
                             "bin 0)", "config": {"workload": rec["workload"], "bins": FIT_BINS},
                     "roofline": rec.get("roofline"),
                     "cpu_baseline": rec.get("cpu_baseline"), "parity": rec.get("parity"),
                     "fit": {k: rec[k] for k in ("newton_numeric_hessian", "gd_armijo")},
                     "e2e": {"value": rec["value"], "unit": "gradient passes/s",
                             "h2d_bytes_per_step": 6 * 8,
                             "d2h_bytes_per_step": rec["d2h_bytes_per_pass"],
                             "path": "FitEngine.chi2_gradient(h, q): q H2D, graph replay, "
                                     "gradient + chi2 D2H, host wall clock"},
                     # per pass: the tile kernel, the empty-bin side pass, the chunk kernel
                     "gpu_launches": 3 * rec["timed_passes"], "clocks": clocks.summary()})
        return line
    with ClockSampler(local) as clocks:
        rec = bench_chi2(a, world, rank, local, dist, passes=max(a.steps, 1),
                         warm=max(a.warmup, 1), parity=not a.no_parity)
    cpu = cpu_baseline_for("chi2") if rank == 0 and world == 1 and not a.no_cpu_baseline else None
    if rank != 0:
        return None
    line = common_line(a, world, rec["value"], "gradient passes/s", rec["ms_per_pass"], "strong")
    line.update({
        "data": "synthetic (device Philox Poisson histogram at the gpoly truth, E=1e10, every "
                "100th bin 0)",
        "config": {"workload": rec["workload"], "bins": CHI2_BINS,
                   "l2": "counts 800 MB >> 126 MB L2; no flush needed",
                   "parallelism": f"dp{world} (bins sharded by chunk, one all-gather per pass)"},
        "roofline": rec["roofline"], "cpu_baseline": cpu, "parity": rec.get("parity"),
        "e2e": {"value": rec["value"], "unit": "gradient passes/s",
                "h2d_bytes_per_step": 6 * 8,
                "d2h_bytes_per_step": rec["d2h_bytes_per_pass"],
                "path": "Chi2Plan.gradient(q): q H2D, graph replay, gradient + chi2 D2H, host "
                        "wall clock (the histogram is resident: it is the plan's state)"},
        # per pass: the tile kernel, the empty-bin side pass, the chunk kernel
        "gpu_launches": 3 * max(a.steps, 1), "clocks": clocks.summary(), "chi2_detail": rec})
    _ = torch
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="gaussnd100", choices=sorted(WORKLOADS))
    ap.add_argument("--transport", default=None, choices=["peer", "nccl", "host"],
                    help="multi-GPU exchange of the chi2 pass (default: peer, then nccl)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="alias of --no-configs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: collectives on host copies (multi-rank path test on 1 GPU)")
    a = ap.parse_args()
    a.no_configs = a.no_configs or a.no_secondary
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        respawn_under_torchrun(a.gpus)
    world, rank, local = dist_setup()
    if world != a.gpus:
        raise SystemExit(f"bench: --gpus {a.gpus} but WORLD_SIZE={world}")
    if a.impl == "reference":
        reference_arm(a, world, rank)
        return
    ours_arm(a, world, rank, local)


if __name__ == "__main__":
    main()
