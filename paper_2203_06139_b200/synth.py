"""Synthetic inputs for the hot path (host side, numpy).

Shapes and distributions follow SURVEY.md §8(d):
  * 1-D Listing-1 points: x~U(-3,3), p~U(-2,2), sigma=1.3
    (acceptance.cpp:168-174 draws them from mt19937_64 through PointSampler;
    here numpy's PCG64 is used because no bit-compatibility with the C++ RNG is
    needed: every parity check feeds the SAME arrays to both sides).
  * N-dim points, structure-of-arrays rows x[d*n + i]: p~U(-2,2),
    x = p + spread*N(0,1) (spread 0.1 at dim 100, 0.03 at dim 1000).
  * Histograms for the chi2 fit: counts_j ~ Poisson(E * m_j / sum(m)), model
    gpoly with truth [1, 0, 1.5, 0.2, -0.01, 0.003] on [-5,5), every 100th bin
    forced to 0 to exercise the c>0 branch (fit.cpp:217,241,251);
    events = sum(counts) as the reference sampler guarantees (fit.cpp:88).
"""
from __future__ import annotations

import numpy as np

GPOLY_TRUTH = (1.0, 0.0, 1.5, 0.2, -0.01, 0.003)
GPOLY_INIT = (0.8, 0.3, 1.2, 0.2, -0.01, 0.003)  # perturbed_init on the Gaussian part (fit.cpp:58-66)


def points_1d(n: int, seed: int = 0x5EED):
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.uniform(-3.0, 3.0, n)
    p = rng.uniform(-2.0, 2.0, n)
    return x, p


def points_nd(dim: int, n: int, seed: int = 42, spread: float | None = None):
    """Returns x, p of shape (dim, n) (row d holds coordinate d of all points)."""
    if spread is None:
        spread = 0.1 if dim <= 100 else 0.03
    rng = np.random.Generator(np.random.PCG64(seed))
    p = rng.uniform(-2.0, 2.0, (dim, n))
    x = p + spread * rng.standard_normal((dim, n))
    return x, p


def gpoly_np(x: np.ndarray, q) -> np.ndarray:
    z = (x - q[1]) / q[2]
    return q[0] * np.exp(-0.5 * z * z) + q[3] + q[4] * x + q[5] * x * x


def gsum_np(x: np.ndarray, q) -> np.ndarray:
    acc = np.zeros_like(x)
    for j in range(len(q) // 3):
        z = (x - q[3 * j + 1]) / q[3 * j + 2]
        acc = acc + q[3 * j] * np.exp(-0.5 * z * z)
    return acc


def centers(bins: int, lo: float, hi: float) -> np.ndarray:
    """Histogram::center (fit.hpp:30-31), bit-exact: lo + (i + 0.5) * width."""
    width = (hi - lo) / bins
    return lo + (np.arange(bins, dtype=np.float64) + 0.5) * width


def histogram(bins: int, lo: float = -5.0, hi: float = 5.0, events: float = 1e8,
              model: str = "gpoly", q=GPOLY_TRUTH, seed: int = 42, zero_every: int = 100):
    """Returns (counts float64[bins], events) with events == counts.sum()."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = centers(bins, lo, hi)
    m = gpoly_np(x, q) if model == "gpoly" else gsum_np(x, q)
    lam = events * m / m.sum()
    counts = rng.poisson(lam).astype(np.float64)
    if zero_every:
        counts[::zero_every] = 0.0
    return counts, float(counts.sum())
