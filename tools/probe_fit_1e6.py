"""BASELINE configs[2]: gpoly fit over 1e6 bins (GD + Armijo, 400 iterations),
iterations/s.  ADC_PROBE_HOST_LOOP=1 runs the host-driven loop (the kernels of
a graph with a conditional node cannot be profiled by ncu; the host loop runs
the same multi-candidate kernel)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402

host = os.environ.get("ADC_PROBE_HOST_LOOP") == "1"
counts, ev = synth.histogram(10**6, events=1e8, seed=11)
h = adc.Histogram(10**6, -5.0, 5.0, ev, counts)
eng = adc.FitEngine("gpoly", 6)
eng.fit(h, synth.GPOLY_INIT, adc.FitOptions(budget=3, host_loop=host))
t0 = time.perf_counter()
r = eng.fit(h, synth.GPOLY_INIT, adc.FitOptions(budget=400, host_loop=host))
dt = time.perf_counter() - t0
print(f"{'host' if host else 'device'} loop: {r.iterations} iterations, {r.iterations / dt:.0f}/s, "
      f"chi2 {r.chi2!r}")
