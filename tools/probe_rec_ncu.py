"""One gradient pass per precision mode (1, 2) at 1e8 bins, for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402

bins = 10**8
h = adc.sample_histogram("gpoly", synth.GPOLY_TRUTH, bins, -5.0, 5.0, 100.0 * bins, seed=7,
                         zero_every=100)
pl = adc.Chi2Plan("gpoly", 6, h)
q = list(synth.GPOLY_INIT)
for mode in (2,):
    pl.set_precision(mode)
    pl.partials(q, True)
    torch.cuda.synchronize()
