"""Shared-mean gaussnd (K2sr / TMA form / K2s) throughput at 10M points x 100 dims:
per-launch CUDA events, median and min of `reps` launches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 9
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 100
n = int(sys.argv[3]) if len(sys.argv) > 3 else 10_000_000
p = torch.rand(dim, dtype=torch.float64, device="cuda")
x = p[:, None] + 0.1 * torch.randn((dim, n), dtype=torch.float64, device="cuda")
dx = torch.zeros_like(x)
dp = torch.zeros(dim, dtype=torch.float64, device="cuda")
o = adc.LaunchOptions(unsafe=True)
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith(("ADC_SHAREDP", "ADC_SPV")))
for dxx, name in ((dx, "with dx"), (None, "dp only")):
    for _ in range(3):
        adc.launch_batch_shared_p("gaussnd_grad_0_1", x, p, 1.3, dxx, dp, o)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        adc.launch_batch_shared_p("gaussnd_grad_0_1", x, p, 1.3, dxx, dp, o)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    byt = (8 + (16 if dxx is not None else 0)) * dim * n
    print(f"{tag} {name}: median {ms:.3f} ms (min {min(ts):.3f}), {byt / ms / 1e6:.0f} GB/s", " ".join(f"{v:.2f}" for v in ts))
