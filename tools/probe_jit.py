"""JIT-lowered corpus gradients over 1e8 points (CUDA events per launch, incl.
the per-launch error-word check): k_rational (no tape) and k_looped (n = 10:
the static-tape variant, tape entries in registers) — and, for ncu, the
kernel named on the command line."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
module = str(np.load(os.path.join(ROOT, "tests", "golden", "jit_cases.npz"))["module"])
n = 100_000_000
only = sys.argv[1] if len(sys.argv) > 1 else None
g = torch.Generator(device="cuda")
g.manual_seed(5)
x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 4 - 2
y = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 4 - 2
dx, dy = torch.zeros_like(x), torch.zeros_like(x)
cfg = adc.LaunchConfig(n // 256 + 1, 256, n)
for kern, bufs, bytes_pt, npar in (
        ("k_rational", adc.BufferSet(arrays={"x": x, "y": y, "dx": dx, "dy": dy}), 48, 2),
        ("k_looped", adc.BufferSet(arrays={"x": x, "dx": dx}, integers={"n": 10}), 24, 1)):
    if only and kern != only:
        continue
    mod = adc.JitModule(module, kern)
    static = mod.static_source([10] if kern == "k_looped" else []) is not None
    for _ in range(3):
        mod.launch(cfg, bufs)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        mod.launch(cfg, bufs)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    print(f"{kern}: {ms:.4f} ms per 1e8 points, {bytes_pt * n / ms / 1e6:.0f} GB/s, "
          f"{npar * n / ms / 1e-3:.3e} pt*param/s, static tape: {static}")
