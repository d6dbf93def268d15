"""Shared-mean gaussnd (K2s) throughput at 10M points x 100 dims."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402

dim, n = 100, 10_000_000
p = torch.rand(dim, dtype=torch.float64, device="cuda")
x = p[:, None] + 0.1 * torch.randn((dim, n), dtype=torch.float64, device="cuda")
dx = torch.zeros_like(x)
dp = torch.zeros(dim, dtype=torch.float64, device="cuda")
o = adc.LaunchOptions(unsafe=True)
for dxx, name in ((dx, "with dx"), (None, "dp only")):
    for _ in range(3):
        adc.launch_batch_shared_p("gaussnd_grad_0_1", x, p, 1.3, dxx, dp, o)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        adc.launch_batch_shared_p("gaussnd_grad_0_1", x, p, 1.3, dxx, dp, o)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    byt = (8 + (16 if dxx is not None else 0)) * dim * n
    print(f"stage={os.environ.get('ADC_SHAREDP_STAGE', 'default')} {name}: {ms:.3f} ms, "
          f"{byt / ms / 1e6:.0f} GB/s")
