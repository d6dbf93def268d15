"""chi2 gradient pass over `bins` bins (default 1e8, gpoly, the bench's
histogram): device time per pass (CUDA events), for ncu -k regex:chi2_tile."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402

bins = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
h = adc.sample_histogram("gpoly", synth.GPOLY_TRUTH, bins, -5.0, 5.0, 100.0 * bins, seed=77,
                         zero_every=100)
pl = adc.Chi2Plan("gpoly", 6, h)
q = list(synth.GPOLY_INIT)
for _ in range(3):
    pl.partials(q, True)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    pl.partials(q, True)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
g, c2 = pl.gradient(q)
print(f"chi2 gradient pass, {bins} bins: {np.median(ts):.4f} ms (min {min(ts):.4f}); chi2 {c2!r}")
