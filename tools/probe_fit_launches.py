"""A 20-iteration GD fit at 1e6 bins (after a warm-up fit), for an ncu launch
list: which kernels an iteration runs and how long each takes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402

counts, ev = synth.histogram(10**6, events=1e8, seed=11)
h = adc.Histogram(10**6, -5.0, 5.0, ev, counts)
eng = adc.FitEngine("gpoly", 6)
eng.fit(h, synth.GPOLY_INIT, adc.FitOptions(budget=3))
t0 = time.perf_counter()
r = eng.fit(h, synth.GPOLY_INIT, adc.FitOptions(budget=int(sys.argv[1]) if len(sys.argv) > 1 else 20))
dt = time.perf_counter() - t0
print(f"iterations {r.iterations} in {dt * 1e3:.2f} ms = {dt / r.iterations * 1e6:.1f} us/iter, "
      f"trials {r.chi2_evals}")
