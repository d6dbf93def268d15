"""The fit's kernels under compute-sanitizer racecheck / synccheck through the
host-driven loop (the tools do not follow the device loop's CUDA-graph WHILE
node): gradient passes, the batched line search, Newton probes, the value
passes of a high-count (residual) histogram."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402

for bins, events in ((200_000, 2e7), (1000, 1e8)):
    counts, ev = synth.histogram(bins, events=events, seed=5)
    h = adc.Histogram(bins, -5.0, 5.0, ev, counts)
    for hess in (False, True):
        r = adc.FitEngine("gpoly", 6).fit(h, synth.GPOLY_INIT,
                                          adc.FitOptions(budget=12, use_hessian=hess,
                                                         host_loop=True))
        assert np.isfinite(r.chi2)
print("ok")
