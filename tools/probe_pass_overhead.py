"""Where the time of one chi2 gradient pass through the API goes at 1e6 bins:
FitEngine.chi2_gradient (Python) vs Chi2Plan.gradient vs a bare ctypes call
of adc_cuda_chi2_gradient with prebuilt arguments (wall clock, 2000 calls)."""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402
from paper_2203_06139_b200._capi import lib  # noqa: E402

bins = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
counts, ev = synth.histogram(bins, events=1e8, seed=11)
h = adc.Histogram(bins, -5.0, 5.0, ev, counts)
eng = adc.FitEngine("gpoly", 6)
q0 = list(synth.GPOLY_INIT)
eng.chi2_gradient(h, q0)
pl = eng._plan(h)
qa = (ctypes.c_double * 6)(*q0)
g = np.zeros(6)
gp = g.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
c2 = ctypes.c_double()
c2r = ctypes.byref(c2)


def run(name, fn, n=2000):
    for _ in range(50):
        fn()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    print(f"{name}: {(time.perf_counter() - t) / n * 1e6:.1f} us per pass")


run("FitEngine.chi2_gradient", lambda: eng.chi2_gradient(h, q0))
run("Chi2Plan.gradient", lambda: pl.gradient(q0))
run("bare ctypes adc_cuda_chi2_gradient", lambda: lib.adc_cuda_chi2_gradient(pl._p, qa, gp, c2r))
run("FitEngine._plan + _state", lambda: eng._plan(h), 20000)
