"""The forced `compute_shared` (K1s: dx, dp private, the shared dsigma slot
reduced in a fixed order) against `compute` (K1) over 1e8 points, CUDA events."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
x = torch.rand(n, dtype=torch.float64, device="cuda") * 6 - 3
p = torch.rand(n, dtype=torch.float64, device="cuda") * 4 - 2
dx, dp = torch.zeros_like(x), torch.zeros_like(x)
ds = torch.zeros(1, dtype=torch.float64, device="cuda")
cfg = adc.LaunchConfig(n // 256 + 1, 256, n)
for kern, extra in (("compute", {}), ("compute_shared", {"dsigma": ds})):
    bufs = adc.BufferSet(arrays={"x": x, "p": p, "dx": dx, "dp": dp, **extra}, scalars={"sigma": 1.3})
    o = adc.LaunchOptions(unsafe=True)
    for _ in range(3):
        adc.launch(kern, cfg, bufs, o)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        adc.launch(kern, cfg, bufs, o)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    print(f"{kern}: {ms:.3f} ms per {n} points, {48 * n / ms / 1e6:.0f} GB/s of 48 B/pt")
