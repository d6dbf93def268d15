"""AD vs numeric provider (the paper's Fig. 2 comparison) on the device pass."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402

dev = torch.device("cuda:0")
bins = int(sys.argv[1]) if len(sys.argv) > 1 else 10**8
lam = torch.full((bins,), 100.0, dtype=torch.float64, device=dev)
counts = torch.poisson(lam)
counts[::100] = 0
h = adc.Histogram(bins, -5.0, 5.0, float(counts.sum()), counts)
for model, np_, q in (("gpoly", 6, list(synth.GPOLY_INIT)), ("gsum", 3, [0.8, 0.3, 1.2]),
                      ("gsum", 12, [0.8, -2.0, 1.2, 0.5, -0.5, 0.8, 0.7, 0.5, 1.0, 0.3, 2.0, 0.6])):
    pl = adc.Chi2Plan(model, np_, h)
    for prov in (0, 1):
        pl.set_provider(prov)
        for fast in (True, False):
            pl.set_precision(fast)
            for _ in range(2):
                pl.partials(q, True)
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                pl.partials(q, True)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            print(f"{model} np={np_} provider={'numeric' if prov else 'ad'} fast={fast}: "
                  f"{np.median(ts):.4f} ms per 1e8-bin gradient pass")
    pl.close()
