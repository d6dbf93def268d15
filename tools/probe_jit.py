"""JIT-lowered corpus gradient (k_rational) over 1e8 points, for ncu."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
module = str(np.load(os.path.join(ROOT, "tests", "golden", "jit_cases.npz"))["module"])
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
x = torch.rand(n, dtype=torch.float64, device="cuda") * 4 - 2
y = torch.rand(n, dtype=torch.float64, device="cuda") * 4 - 2
dx, dy = torch.zeros_like(x), torch.zeros_like(x)
mod = adc.JitModule(module, "k_rational")
cfg = adc.LaunchConfig(n // 256 + 1, 256, n)
bufs = adc.BufferSet(arrays={"x": x, "y": y, "dx": dx, "dy": dy})
for _ in range(4):
    mod.launch(cfg, bufs)
torch.cuda.synchronize()
print("ok")
ts = []
for _ in range(10):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    mod.launch(cfg, bufs)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = float(np.median(ts))
print(f"k_rational n={n}: {ms:.3f} ms per launch, {48 * n / ms / 1e6:.0f} GB/s")
