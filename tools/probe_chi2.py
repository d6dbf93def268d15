"""chi2 kernel variants (ADC_CHI2_TUNE) timed with CUDA events on the device pass."""
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
pl = adc.Chi2Plan("gpoly", 6, h)
q = list(synth.GPOLY_INIT)
for tune in [int(t) for t in (sys.argv[2].split(',') if len(sys.argv) > 2 else ['0', '2'])]:
    os.environ["ADC_CHI2_TUNE"] = str(tune)
    pl.set_precision(True)
    for grad in (True, False):
        for _ in range(3):
            pl.partials(q, grad)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            pl.partials(q, grad)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"tune={tune} grad={grad}: {np.median(ts):.4f} ms (min {min(ts):.4f})  "
              f"{62e-9 * bins / (np.median(ts) * 1e-3) if grad else 0:.2f} T fp64-alg/s")

# per-rank device pass time of a W-way split (rank 0's shard, same layout)
os.environ["ADC_CHI2_TUNE"] = "0"
for world in (1, 2, 4, 8):
    pr = adc.Chi2Plan("gpoly", 6, h, world=world, rank=0)
    for _ in range(3):
        pr.partials(q, True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        pr.partials(q, True)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    L = pr.layout
    print(f"world={world}: rank-0 shard {L.bin_end - L.bin_begin} bins, "
          f"{np.median(ts):.4f} ms -> ideal-scaling ratio "
          f"{np.median(ts) * world:.4f} ms-equivalent")
    pr.close()
