"""gaussnd dim 1000 x 1M (BASELINE configs[3]): the auto kernel vs the
cluster form (variant 15), CUDA events, and the cluster form's outputs
within 1e-12 relative of the auto kernel's (which the parity tests pin)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200.launch import set_gaussnd_variant  # noqa: E402

dim = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
variants = [int(v) for v in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "15"])]
g = torch.Generator(device="cuda")
g.manual_seed(3)
p = torch.rand((dim, n), dtype=torch.float64, device="cuda", generator=g) * 4 - 2
x = p + 0.03 * torch.randn((dim, n), dtype=torch.float64, device="cuda", generator=g)
ref = None
for v in variants:
    set_gaussnd_variant(v)
    dx = torch.zeros_like(x)
    dp = torch.zeros_like(x)
    adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, dx, dp)
    torch.cuda.synchronize()
    out = dx.cpu().numpy()
    if ref is None:
        ref = out
    rel = np.abs(out - ref) / np.maximum(np.maximum(np.abs(out), np.abs(ref)), 1e-300)
    same = bool(np.array_equal(out, ref))
    del out
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
    print(f"variant {v}: {ms:.3f} ms, {48 * dim * n / ms / 1e6:.0f} GB/s, "
          f"bitwise v{variants[0]}: {same}, max rel vs v{variants[0]}: {rel.max():.3e}", flush=True)
    del dx, dp
set_gaussnd_variant(0)
