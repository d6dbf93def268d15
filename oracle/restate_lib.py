"""ctypes binding of oracle/restate.c (TEST INFRASTRUCTURE — the checker).

Built by `make -C oracle restate` (also run by __graft_entry__.build()); if the
.so is missing this builds it with gcc (present on the GPU box too).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_ref", "librestate.so")
MODELS = {"gsum": 0, "gpoly": 1}

_D = ctypes.POINTER(ctypes.c_double)
_lib = None


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


class Restate:
    def __init__(self, lib):
        self.lib = lib
        i64, d, i = ctypes.c_int64, ctypes.c_double, ctypes.c_int
        lib.rs_gauss_grad_batch.argtypes = [_D, _D, d, _D, _D, i64]
        lib.rs_gauss_grad_shared_batch.argtypes = [_D, _D, d, _D, _D, _D, i64]
        lib.rs_gauss_shared_dsigma_compensated.argtypes = [_D, _D, d, i64, _D, _D]
        lib.rs_gaussnd_grad_shared_p.argtypes = [_D, _D, d, i64, i64, i64, _D, _D]
        lib.rs_gaussnd_shared_p_dp_compensated.argtypes = [_D, _D, d, i64, i64, i64, _D, _D]
        lib.rs_gaussnd_grad_batch.argtypes = [_D, _D, d, i64, i64, i64, _D, _D]
        lib.rs_model.argtypes = [i, d, _D, i64]
        lib.rs_model.restype = d
        lib.rs_model_grad.argtypes = [i, d, _D, i64, _D]
        lib.rs_chi2.argtypes = [i, _D, i64, d, d, d, _D, i64]
        lib.rs_chi2.restype = d
        lib.rs_chi2_gradient.argtypes = [i, _D, i64, d, d, d, _D, i64, _D]
        lib.rs_chi2_gradient_compensated.argtypes = [i, _D, i64, d, d, d, _D, i64, _D, _D]
        lib.rs_chi2_gradient_p.argtypes = [i, i, _D, i64, d, d, d, _D, i64, _D]
        lib.rs_chi2_gradient_compensated_p.argtypes = [i, i, _D, i64, d, d, d, _D, i64, _D, _D,
                                                       _D]
        lib.rs_model_grad_numeric.argtypes = [i, d, _D, i64, _D]
        lib.rs_chi2_compensated.argtypes = [i, _D, i64, d, d, d, _D, i64, _D]
        lib.rs_chi2_compensated.restype = d

    def gauss_grad(self, x, p, sigma, dx, dp):
        """In-place accumulate, like the reference slots."""
        self.lib.rs_gauss_grad_batch(_p(x), _p(p), sigma, _p(dx), _p(dp), x.size)

    def gauss_grad_shared(self, x, p, sigma, dx, dp, dsigma):
        """compute_shared, forced sequential: accumulates into dx, dp, dsigma[0]."""
        self.lib.rs_gauss_grad_shared_batch(_p(x), _p(p), sigma, _p(dx), _p(dp), _p(dsigma),
                                            x.size)

    def gauss_shared_dsigma_compensated(self, x, p, sigma):
        """(total, sum of magnitudes) of every sigma contribution."""
        t, a = np.zeros(1), np.zeros(1)
        self.lib.rs_gauss_shared_dsigma_compensated(_p(x), _p(p), sigma, x.size, _p(t), _p(a))
        return float(t[0]), float(a[0])

    def gaussnd_grad_shared_p(self, x, p, sigma, dx, dp):
        """x, dx (dim, n) SoA; p, dp (dim,): points in order, dp shared."""
        dim, n = x.shape
        self.lib.rs_gaussnd_grad_shared_p(_p(x), _p(p), sigma, dim, n, n, _p(dx), _p(dp))

    def gaussnd_shared_p_dp_compensated(self, x, p, sigma):
        dim, n = x.shape
        tot, ab = np.zeros(dim), np.zeros(dim)
        self.lib.rs_gaussnd_shared_p_dp_compensated(_p(x), _p(p), sigma, dim, n, n, _p(tot),
                                                    _p(ab))
        return tot, ab

    def gaussnd_grad(self, x, p, sigma, dx, dp):
        dim, n = x.shape
        self.lib.rs_gaussnd_grad_batch(_p(x), _p(p), sigma, dim, n, n, _p(dx), _p(dp))

    def model(self, model, x, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        return self.lib.rs_model(MODELS[model], x, _p(q), q.size)

    def model_grad(self, model, x, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        out = np.zeros(q.size)
        self.lib.rs_model_grad(MODELS[model], x, _p(q), q.size, _p(out))
        return out

    def chi2(self, model, counts, lo, hi, events, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        return self.lib.rs_chi2(MODELS[model], _p(counts), counts.size, lo, hi, events, _p(q), q.size)

    def chi2_gradient(self, model, counts, lo, hi, events, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        out = np.zeros(q.size)
        self.lib.rs_chi2_gradient(MODELS[model], _p(counts), counts.size, lo, hi, events, _p(q),
                                  q.size, _p(out))
        return out

    def model_grad_numeric(self, model, x, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        out = np.zeros(q.size)
        self.lib.rs_model_grad_numeric(MODELS[model], x, _p(q), q.size, _p(out))
        return out

    def chi2_gradient_numeric(self, model, counts, lo, hi, events, q):
        """Sequential fit.cpp:224-259 with GradientProvider::Numeric."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        out = np.zeros(q.size)
        self.lib.rs_chi2_gradient_p(MODELS[model], 1, _p(counts), counts.size, lo, hi, events,
                                    _p(q), q.size, _p(out))
        return out

    def chi2_gradient_numeric_compensated(self, model, counts, lo, hi, events, q):
        """Returns (gradient, scale, fd_scale): the Numeric provider with compensated
        sums; tolerance 1e-12 * scale + 4 * fd_scale (one primal ulp per probe
        evaluation on each side, amplified by 1/(2h))."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        out, scale, fd = np.zeros(q.size), np.zeros(q.size), np.zeros(q.size)
        self.lib.rs_chi2_gradient_compensated_p(MODELS[model], 1, _p(counts), counts.size, lo, hi,
                                                events, _p(q), q.size, _p(out), _p(scale), _p(fd))
        return out, scale, fd

    def chi2_gradient_compensated(self, model, counts, lo, hi, events, q):
        """Returns (gradient, scale) with scale_i = sum_j |w_j dm_j/dq_i|."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        out = np.zeros(q.size)
        scale = np.zeros(q.size)
        self.lib.rs_chi2_gradient_compensated(MODELS[model], _p(counts), counts.size, lo, hi,
                                              events, _p(q), q.size, _p(out), _p(scale))
        return out, scale

    def chi2_compensated(self, model, counts, lo, hi, events, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        scale = np.zeros(1)
        v = self.lib.rs_chi2_compensated(MODELS[model], _p(counts), counts.size, lo, hi, events,
                                         _p(q), q.size, _p(scale))
        return v, float(scale[0])


def build():
    subprocess.run(["make", "-s", "-C", HERE, "restate"], check=True)


def load() -> Restate:
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            build()
        _lib = Restate(ctypes.CDLL(SO))
    return _lib


def read_histogram(path):
    """The histogram ingest format (include/adc_cuda.h), read independently of
    the product: "ADCHIST1", int64 bins, double lo, hi, events, double
    counts[bins] (little-endian).  Returns (bins, lo, hi, events, counts)."""
    with open(path, "rb") as f:
        if f.read(8) != b"ADCHIST1":
            raise ValueError(f"{path}: not an ADCHIST1 histogram file")
        bins = int(np.frombuffer(f.read(8), dtype="<i8")[0])
        lo, hi, events = (float(v) for v in np.frombuffer(f.read(24), dtype="<f8"))
        counts = np.frombuffer(f.read(8 * bins), dtype="<f8").copy()
    if counts.size != bins:
        raise ValueError(f"{path}: short file")
    return bins, lo, hi, events, counts
