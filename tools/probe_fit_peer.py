"""Fit through a peer-transport communicator (world 1): the device loop (default)
vs the host loop (FitOptions.host_loop) — same bits, different speed."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402

counts, ev = synth.histogram(10**6, events=1e8, seed=11)
h = adc.Histogram(10**6, -5.0, 5.0, ev, counts)
comm = adc.Comm.peer(1, 0, lambda a: a.copy())
res = {}
for mode in ("1", "0", "1"):
    eng = adc.FitEngine("gpoly", 6, comm=comm)
    eng.fit(h, synth.GPOLY_INIT, adc.FitOptions(budget=3, host_loop=mode == "0"))
    t0 = time.perf_counter()
    r = eng.fit(h, synth.GPOLY_INIT, adc.FitOptions(budget=200, host_loop=mode == "0"))
    dt = time.perf_counter() - t0
    res[mode] = np.array(r.params).tobytes()
    print(f"device loop={mode}: {r.iterations / dt:.0f} iterations/s, chi2 {r.chi2!r}")
print("same bits:", res["0"] == res["1"])
