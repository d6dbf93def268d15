"""Host-side mirror of the reference histogram-fit API (proj/include/adc/fit.hpp)
over the B200 C ABI, model-parameterised (gsum of fit.cpp:125-138, or the
Gaussian + quadratic background gpoly of oracle/dsl/gpoly.dsl).

    h = Histogram(bins, lo, hi, events, counts)
    eng = FitEngine("gpoly", np=6)
    eng.chi2(h, q); eng.chi2_gradient(h, q); eng.fit(h, init, FitOptions())
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List

import numpy as np

from ._capi import (MODEL_IDS, AdcError, Chi2Layout, FitOptions as _FitOptionsC, FitResultC,
                    check, dbl_array, dptr, lib)


class GradientProvider:
    """adc::GradientProvider (fit.hpp:52): the generated reverse-mode gradient
    of the model, or central differences of the model (numdiff.cpp:38-87)."""
    AdReverse = 0
    Numeric = 1


@dataclass
class Histogram:
    """fit.hpp:23-34.  counts: numpy float64 (host) or a float64 CUDA tensor."""
    bins: int
    lo: float
    hi: float
    events: float
    counts: object

    def width(self) -> float:
        return (self.hi - self.lo) / self.bins

    def save(self, path: str) -> None:
        """The ingest format (include/adc_cuda.h: "ADCHIST1", bins, lo, hi,
        events, counts); counts from host (numpy) or device (CUDA tensor)."""
        c = self.counts
        if hasattr(c, "is_cuda"):
            c = c.contiguous()
            ptr = c.data_ptr()
        else:
            c = np.ascontiguousarray(c, dtype=np.float64)
            ptr = c.ctypes.data
        check(lib.adc_histogram_write(path.encode(), int(self.bins), float(self.lo), float(self.hi),
                                      float(self.events), ctypes.c_void_p(ptr)))

    @classmethod
    def load(cls, path: str, device=None) -> "Histogram":
        """Read a histogram file; device != None puts the counts in a CUDA
        tensor on that device (pinned pieces, H2D overlapped with the reads)."""
        b, lo, hi, ev = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        check(lib.adc_histogram_read_header(path.encode(), ctypes.byref(b), ctypes.byref(lo),
                                            ctypes.byref(hi), ctypes.byref(ev)))
        if device is None:
            counts = np.empty(b.value, dtype=np.float64)
            ptr = counts.ctypes.data
        else:
            import torch
            counts = torch.empty(b.value, dtype=torch.float64, device=device)
            ptr = counts.data_ptr()
        check(lib.adc_histogram_read_counts(path.encode(), b.value, ctypes.c_void_p(ptr)))
        return cls(b.value, lo.value, hi.value, ev.value, counts)

    def center(self, i: int) -> float:
        return self.lo + (i + 0.5) * self.width()


@dataclass
class FitOptions:
    """fit.hpp:56-65."""
    budget: int = 400
    grad_tol: float = 1e-6
    chi2_rel_tol: float = 1e-12
    sigma_min: float = 1e-3
    armijo_c1: float = 1e-4
    use_hessian: bool = False
    trace_iterates: int = 0
    host_loop: bool = False  # B200 option: host-driven loop instead of the device-resident one


@dataclass
class FitResult:
    """fit.hpp:67-78 (op counters are interpreter metadata, not part of this path)."""
    params: List[float]
    chi2: float
    iterations: int
    gradient_evals: int
    gradient_wall_ns: int
    converged: bool
    sigma_clamps: int
    chi2_evals: int = 0
    iterates: List[List[float]] = field(default_factory=list)


def sample_histogram(model: str, q, bins: int, lo: float, hi: float, events: float,
                     seed: int = 42, zero_every: int = 0, device=None) -> Histogram:
    """On-device histogram: counts[j] ~ Poisson(events m_j / sum m) at the
    parameters q (counter-based Philox, a pure function of the arguments);
    Histogram.events = sum of the counts (fit.cpp:88, 94-102)."""
    import torch
    q = np.ascontiguousarray(q, dtype=np.float64)
    counts = torch.empty(bins, dtype=torch.float64, device=device or "cuda")
    total = ctypes.c_double()
    check(lib.adc_cuda_histogram_sample(
        MODEL_IDS[model], q.size, q.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), bins,
        float(lo), float(hi), float(events), seed & 0xFFFFFFFFFFFFFFFF, zero_every, dptr(counts),
        ctypes.byref(total), ctypes.c_void_p(torch.cuda.current_stream(counts.device).cuda_stream)))
    return Histogram(bins, lo, hi, total.value, counts)


def chi2_layout(bins: int, world: int = 1, rank: int = 0) -> Chi2Layout:
    L = Chi2Layout()
    check(lib.adc_chi2_make_layout(bins, world, rank, ctypes.byref(L)))
    return L


def record_len(np_: int, want_grad: bool) -> int:
    return lib.adc_chi2_record_len(np_, 1 if want_grad else 0)


def finalize(np_: int, events: float, records: np.ndarray, want_grad: bool = True):
    """Fixed-order reduction of chunk records + closed form (host, no device)."""
    rec = np.ascontiguousarray(records, dtype=np.float64).ravel()
    R = record_len(np_, want_grad)
    nchunks = rec.size // R
    g = np.zeros(np_)
    c2 = ctypes.c_double()
    check(lib.adc_chi2_finalize(np_, float(events), rec.ctypes.data_as(ctypes.POINTER(
        ctypes.c_double)), nchunks, 1 if want_grad else 0, g.ctypes.data_as(ctypes.POINTER(
            ctypes.c_double)), ctypes.byref(c2)))
    return (g, c2.value) if want_grad else c2.value


class Chi2Plan:
    """One histogram resident on one device (or one rank's shard of it).

    With a communicator (comm.Comm) a sharded plan runs the whole pass —
    kernels, the record all-gather and the fixed-order finalize — so
    gradient/chi2/chi2_multi/fit give the same bits on every rank and for
    every world size."""

    def __init__(self, model: str, np_: int, h: Histogram, world: int = 1, rank: int = 0,
                 comm=None, _shard=None):
        import torch
        if model not in MODEL_IDS:
            raise AdcError("Arg", f"unknown model '{model}'")
        self.model, self.np, self.h = model, np_, h
        self.comm = comm  # keep alive (the plan does not own it)
        counts = h.counts if _shard is None else _shard
        if not hasattr(counts, "is_cuda"):
            counts = torch.from_numpy(np.ascontiguousarray(counts, dtype=np.float64)).cuda()
        elif not counts.is_cuda or counts.dtype != torch.float64 or not counts.is_contiguous():
            counts = counts.to(device="cuda", dtype=torch.float64).contiguous()
        self.counts = counts  # keep alive
        self._p = ctypes.c_void_p()
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        if _shard is not None:
            check(lib.adc_cuda_chi2_plan_create_sharded(
                ctypes.byref(self._p), MODEL_IDS[model], np_, h.bins, float(h.lo), float(h.hi),
                float(h.events), dptr(counts), comm._p, stream))
        else:
            if comm is not None:
                world, rank = comm.world, comm.rank
            check(lib.adc_cuda_chi2_plan_create(
                ctypes.byref(self._p), MODEL_IDS[model], np_, h.bins, float(h.lo), float(h.hi),
                float(h.events), dptr(counts), world, rank, stream))
            if comm is not None:
                check(lib.adc_cuda_chi2_plan_set_comm(self._p, comm._p))
        self.layout = Chi2Layout()
        check(lib.adc_cuda_chi2_plan_layout(self._p, ctypes.byref(self.layout)))

    @classmethod
    def sharded(cls, model: str, np_: int, h: Histogram, shard_counts, comm) -> "Chi2Plan":
        """A rank holding only counts[bin_begin:bin_end] of
        chi2_layout(h.bins, comm.world, comm.rank); h.counts is not read."""
        return cls(model, np_, h, comm=comm, _shard=shard_counts)

    def set_precision(self, mode):
        """0 / False: faithful IEEE divisions; 1: fast (reciprocal multiplies,
        table exp); 2 / True (default): fast, and every pass takes each
        thread's Gaussian factors from an anchored product recurrence."""
        mode = 2 if mode is True else 0 if mode is False else int(mode)
        check(lib.adc_cuda_chi2_set_precision(self._p, mode))

    def refresh(self):
        """Recompute what depends on the counts alone (1/c, C0, linear sums)
        after the device counts were changed in place."""
        check(lib.adc_cuda_chi2_plan_refresh(self._p))

    def set_provider(self, provider: int):
        """GradientProvider.AdReverse (default) or GradientProvider.Numeric."""
        provider = int(provider)
        if provider != getattr(self, "_provider", None):  # one C call per change
            check(lib.adc_cuda_chi2_set_provider(self._p, provider))
            self._provider = provider

    def _params(self, q):
        # a ctypes array of exactly np doubles (cheaper per call than numpy +
        # data_as on this per-pass path)
        if len(q) != self.np:
            raise AdcError("Arg", f"expected {self.np} parameters, got {len(q)}")
        return (ctypes.c_double * self.np)(*map(float, q))

    def gradient(self, q):
        qa = self._params(q)
        g = (ctypes.c_double * self.np)()
        c2 = ctypes.c_double()
        check(lib.adc_cuda_chi2_gradient(self._p, qa, g, ctypes.byref(c2)))
        return np.frombuffer(g, dtype=np.float64).copy(), c2.value

    def chi2(self, q) -> float:
        c2 = ctypes.c_double()
        check(lib.adc_cuda_chi2(self._p, self._params(q), ctypes.byref(c2)))
        return c2.value

    def chi2_multi(self, qs) -> np.ndarray:
        """chi2 of several parameter vectors in one pass (bit-identical to chi2)."""
        qs = np.ascontiguousarray(qs, dtype=np.float64).reshape(-1, self.np)
        out = np.zeros(qs.shape[0])
        dp = ctypes.POINTER(ctypes.c_double)
        check(lib.adc_cuda_chi2_multi(self._p, qs.ctypes.data_as(dp), qs.shape[0],
                                      out.ctypes.data_as(dp)))
        return out

    def gradient_multi(self, qs) -> np.ndarray:
        """Gradients of several parameter vectors, one sync (each equals gradient())."""
        qs = np.ascontiguousarray(qs, dtype=np.float64).reshape(-1, self.np)
        out = np.zeros_like(qs)
        dp = ctypes.POINTER(ctypes.c_double)
        check(lib.adc_cuda_chi2_gradient_multi(self._p, qs.ctypes.data_as(dp), qs.shape[0],
                                               out.ctypes.data_as(dp)))
        return out

    def partials(self, q, want_grad: bool, records_dev=None):
        """Enqueue this rank's pass; records land in records_dev (a float64 CUDA
        tensor of local_chunks * record_len) or the plan's own buffer."""
        check(lib.adc_cuda_chi2_partials(self._p, dbl_array(q), 1 if want_grad else 0,
                                         dptr(records_dev) if records_dev is not None else None))

    def value_mode(self):
        """(residual, kappa): whether chi2 values take the residual pass
        (high counts per bin, include/adc_cuda.h) and C0 / non-empty bins."""
        r, k = ctypes.c_int32(), ctypes.c_double()
        check(lib.adc_cuda_chi2_value_mode(self._p, ctypes.byref(r), ctypes.byref(k)))
        return bool(r.value), k.value

    def tile_kernel_ms(self, q, want_grad: bool = True, records_dev=None) -> float:
        """One pass (partials) with CUDA events around its tile kernel (the
        dominant kernel); returns that kernel's duration in ms."""
        check(lib.adc_cuda_chi2_set_kernel_timing(self._p, 1))
        self.partials(q, want_grad, records_dev)
        ms = ctypes.c_float()
        check(lib.adc_cuda_chi2_kernel_ms(self._p, ctypes.byref(ms)))
        check(lib.adc_cuda_chi2_set_kernel_timing(self._p, 0))
        return ms.value

    @property
    def stream_ptr(self):
        return None

    def close(self):
        if self._p:
            lib.adc_cuda_chi2_plan_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def default_clamp(model: str, np_: int):
    """Indices the sigma clamp applies to: every third for gsum (fit.cpp:268-278),
    only the width q[2] for gpoly."""
    return list(range(2, np_, 3)) if model == "gsum" else [2]


class FitEngine:
    """adc::FitEngine (fit.hpp:82-112), model-parameterised, B200 passes."""

    def __init__(self, model: str = "gsum", np_: int = 3, comm=None):
        """comm: a comm.Comm to shard every histogram over its ranks (each rank
        calls the same methods; results are identical on all ranks)."""
        self.model, self.np, self.comm = model, np_, comm
        self._plans = {}

    @staticmethod
    def _state(h: Histogram):
        """What a plan snapshots of a histogram: the reference's FitEngine reads
        h.counts and h.events on every call, so a change of any of them (a
        reassigned field, or an in-place write to a torch counts tensor, seen
        through its version counter) rebuilds the plan.  Host (numpy) counts
        are made read-only while a plan holds their snapshot, so an in-place
        write raises instead of being silently ignored."""
        c = h.counts
        if hasattr(c, "is_cuda"):
            cs = ("torch", c.data_ptr(), int(c._version), tuple(c.shape))
        else:
            cs = ("numpy", id(c), c.__array_interface__["data"][0], c.shape)
        return (h.bins, float(h.lo), float(h.hi), float(h.events), cs)

    def _plan(self, h: Histogram) -> Chi2Plan:
        key = id(h)
        st = self._state(h)
        ent = self._plans.get(key)
        if ent is None or ent[0].h is not h or ent[1] != st:
            if ent is not None:
                ent[0].close()
            pl = Chi2Plan(self.model, self.np, h, comm=self.comm)
            c = h.counts
            if not hasattr(c, "is_cuda") and isinstance(c, np.ndarray):
                c.flags.writeable = False
            self._plans = {key: (pl, st)}
            return pl
        return ent[0]

    def gradient_fn_name(self) -> str:
        return f"{self.model}_grad_1"

    def chi2(self, h: Histogram, q) -> float:
        return self._plan(h).chi2(q)

    def chi2_gradient(self, h: Histogram, q,
                      provider: int = GradientProvider.AdReverse) -> np.ndarray:
        """FitEngine::chi2_gradient(h, q, provider, out) (fit.cpp:224-259)."""
        pl = self._plan(h)
        pl.set_provider(provider)
        return pl.gradient(q)[0]

    def fit(self, h: Histogram, init, opts: FitOptions | None = None, clamp=None,
            provider: int = GradientProvider.AdReverse) -> FitResult:
        """FitEngine::fit(h, provider, init, opts) (fit.cpp:315-425)."""
        opts = opts or FitOptions()
        pl = self._plan(h)
        pl.set_provider(provider)
        o = _FitOptionsC(opts.budget, opts.grad_tol, opts.chi2_rel_tol, opts.sigma_min,
                         opts.armijo_c1, opts.trace_iterates, 1 if opts.use_hessian else 0,
                         1 if opts.host_loop else 0)
        idx = default_clamp(self.model, self.np) if clamp is None else list(clamp)
        cidx = (ctypes.c_int32 * max(1, len(idx)))(*idx)
        params = np.ascontiguousarray(init, dtype=np.float64).copy()
        its = np.zeros(max(1, opts.trace_iterates) * self.np)
        res = FitResultC()
        dp = ctypes.POINTER(ctypes.c_double)
        check(lib.adc_cuda_fit(pl._p, params.ctypes.data_as(dp), cidx, len(idx), ctypes.byref(o),
                               ctypes.byref(res), its.ctypes.data_as(dp)))
        n_tr = min(opts.trace_iterates, res.iterations + 1) if opts.trace_iterates else 0
        return FitResult(params=list(params), chi2=res.chi2, iterations=res.iterations,
                         gradient_evals=res.gradient_evals, gradient_wall_ns=res.gradient_ns,
                         converged=bool(res.converged), sigma_clamps=res.sigma_clamps,
                         chi2_evals=res.chi2_evals,
                         iterates=[list(its[k * self.np:(k + 1) * self.np]) for k in range(n_tr)])


def default_truth(k: int, lo: float = -5.0, hi: float = 5.0):
    """gauss_sum::default_truth (fit.cpp:46-56)."""
    sig = (1.5, 1.0, 0.75)
    q = []
    for j in range(k):
        q += [1.0, lo + (hi - lo) * (j + 1) / (k + 1), sig[j % 3]]
    return q


def perturbed_init(truth):
    """gauss_sum::perturbed_init (fit.cpp:58-66)."""
    q = list(truth)
    for j in range(0, len(q) - 2, 3):
        q[j] *= 0.8
        q[j + 1] += 0.3
        q[j + 2] *= 0.8
    return q


@dataclass
class BenchRow:
    """fit.hpp BenchRow (the reference's Fig. 2b table)."""
    k: int
    params: int
    provider: str
    median_wall_ns: int
    grad_evals: int
    converged: bool
    final_params: List[float]


def bench_scaling(k_list=(1, 2, 4, 8), bins: int = 1000, events: float = 1e5, lo: float = -5.0,
                  hi: float = 5.0, seed: int = 42, repeats: int = 1,
                  opts: FitOptions | None = None) -> List[BenchRow]:
    """bench_scaling (fit.cpp:427-458), the paper's Fig. 2b, on the B200: for each
    K a gsum histogram at default_truth (sampled on the device, seed + K), fitted
    from perturbed_init with both gradient providers; median gradient wall time."""
    if not k_list:
        raise AdcError("Eval", "empty K list")
    opts = opts or FitOptions()
    rows = []
    for k in k_list:
        truth = default_truth(k, lo, hi)
        h = sample_histogram("gsum", truth, bins, lo, hi, events, seed=seed + k)
        init = perturbed_init(truth)
        eng = FitEngine("gsum", 3 * k)
        for prov, name in ((GradientProvider.AdReverse, "ad-reverse"),
                           (GradientProvider.Numeric, "numeric")):
            walls, last = [], None
            for _ in range(max(1, repeats)):
                last = eng.fit(h, init, opts, provider=prov)
                walls.append(last.gradient_wall_ns)
            walls.sort()
            rows.append(BenchRow(k, 3 * k, name, walls[len(walls) // 2], last.gradient_evals,
                                 last.converged, last.params))
    return rows


def bench_csv(rows: List[BenchRow]) -> str:
    """bench_csv (fit.cpp:460-470); op-count columns are interpreter metadata (0 here)."""
    out = "K,params,provider,median_wall_ns,grad_evals,primal_opcount,grad_opcount,converged\n"
    for r in rows:
        out += (f"{r.k},{r.params},{r.provider},{r.median_wall_ns},{r.grad_evals},0,0,"
                f"{1 if r.converged else 0}\n")
    return out
