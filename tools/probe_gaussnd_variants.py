"""gaussnd dim 100 x 10M (the headline) per kernel variant, CUDA events, plus a
bitwise check of every variant against variant 0."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200.launch import set_gaussnd_variant  # noqa: E402

dim = int(sys.argv[1]) if len(sys.argv) > 1 else 100
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
variants = [int(v) for v in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "10", "11"])]
g = torch.Generator(device="cuda")
g.manual_seed(3)
p = torch.rand((dim, n), dtype=torch.float64, device="cuda", generator=g) * 4 - 2
x = p + 0.1 * torch.randn((dim, n), dtype=torch.float64, device="cuda", generator=g)
ref = None
for v in variants:
    set_gaussnd_variant(v)
    dx = torch.zeros_like(x)
    dp = torch.zeros_like(x)
    adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, dx, dp)
    torch.cuda.synchronize()
    sig = (dx[:, :1000].cpu().numpy().tobytes(), dx[:, -1000:].cpu().numpy().tobytes())
    if ref is None:
        ref = sig
    same = sig == ref
    for _ in range(2):
        adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, dx, dp)
    torch.cuda.synchronize()
    ts = []
    for _ in range(8):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, dx, dp)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    print(f"variant {v}: {ms:.3f} ms, {48 * dim * n / ms / 1e6:.0f} GB/s, bits equal to v{variants[0]}: {same}")
    del dx, dp
set_gaussnd_variant(0)
