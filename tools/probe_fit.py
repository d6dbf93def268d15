"""Fit-loop timing at 1e6 bins (GD + Armijo and Newton) and multi-pass timing."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402

for bins in (10**6, 10**7):
    counts, ev = synth.histogram(bins, events=100.0 * bins, seed=11)
    h = adc.Histogram(bins, -5.0, 5.0, ev, counts)
    eng = adc.FitEngine("gpoly", 6)
    eng.fit(h, synth.GPOLY_INIT, adc.FitOptions(budget=2, use_hessian=True))
    pl = eng._plan(h)
    qs = np.stack([np.array(synth.GPOLY_INIT) * (1 + 1e-3 * k) for k in range(32)])
    for n in (1, 8, 32):
        pl.chi2_multi(qs[:n])
        t0 = time.perf_counter()
        for _ in range(20):
            pl.chi2_multi(qs[:n])
        print(f"bins={bins} chi2_multi({n}): {(time.perf_counter() - t0) / 20 * 1e6:.1f} us")
    for _ in range(3):
        pl.gradient(synth.GPOLY_INIT)
    t0 = time.perf_counter()
    for _ in range(50):
        pl.gradient(synth.GPOLY_INIT)
    print(f"bins={bins} gradient: {(time.perf_counter() - t0) / 50 * 1e6:.1f} us")
    for hess in (False, True):
        t0 = time.perf_counter()
        r = eng.fit(h, synth.GPOLY_INIT, adc.FitOptions(budget=400, use_hessian=hess))
        dt = time.perf_counter() - t0
        print(f"bins={bins} fit hess={hess}: {r.iterations} it in {dt*1e3:.1f} ms "
              f"({r.iterations/dt:.0f} it/s), grads {r.gradient_evals}, trials {r.chi2_evals}, "
              f"conv {r.converged}, mu/sigma {r.params[1]:.5f} {r.params[2]:.5f}")
