"""Shared-mean gaussnd on an odd-offset view (rows not 16-byte aligned: the
K2s form) and on the aligned layout, per-launch CUDA events (median)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402

dim = int(sys.argv[1]) if len(sys.argv) > 1 else 60
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
p = torch.rand(dim, dtype=torch.float64, device="cuda")
wide = torch.randn((dim, n + 1), dtype=torch.float64, device="cuda") * 0.1 + p[:, None]
dxw = torch.zeros_like(wide)
dp = torch.zeros(dim, dtype=torch.float64, device="cuda")
o = adc.LaunchOptions(unsafe=True)
for name, x, dx in (("odd view", wide[:, 1:], dxw[:, 1:]), ("aligned", torch.randn((dim, n), dtype=torch.float64, device="cuda") * 0.1 + p[:, None], torch.zeros((dim, n), dtype=torch.float64, device="cuda"))):
    for dxx, what in ((dx, "with dx"), (None, "dp only")):
        for _ in range(3):
            adc.launch_batch_shared_p("gaussnd_grad_0_1", x, p, 1.3, dxx, dp, o)
        torch.cuda.synchronize()
        ts = []
        for _ in range(7):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            adc.launch_batch_shared_p("gaussnd_grad_0_1", x, p, 1.3, dxx, dp, o)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        byt = (8 + (16 if dxx is not None else 0)) * dim * x.shape[1]
        print(f"dim {dim} {name} {what}: {ms:.3f} ms, {byt / ms / 1e6:.0f} GB/s")
