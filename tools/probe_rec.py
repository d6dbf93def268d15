"""chi2 gradient pass at 1e8 bins in precision modes 1 (table exp per bin) and
2 (anchored Gaussian-factor recurrence): device time and the difference of the
two gradients relative to sum|terms| (compensated oracle scale)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402

bins = int(sys.argv[1]) if len(sys.argv) > 1 else 10**8
h = adc.sample_histogram("gpoly", synth.GPOLY_TRUTH, bins, -5.0, 5.0, 100.0 * bins, seed=7,
                         zero_every=100)
pl = adc.Chi2Plan("gpoly", 6, h)
q = list(synth.GPOLY_INIT)
res = {}
for mode in (1, 2, 1, 2):
    pl.set_precision(mode)
    for _ in range(3):
        pl.partials(q, True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        pl.partials(q, True)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    g, c2 = pl.gradient(q)
    res[mode] = np.array(g)
    print(f"mode {mode}: {np.median(ts):.4f} ms (min {min(ts):.4f}); grad {g}")
print("max |g2 - g1| / |g1|:", np.max(np.abs(res[2] - res[1]) / np.abs(res[1])))
