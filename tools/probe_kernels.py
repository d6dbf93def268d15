"""Quick kernel timings (CUDA events) for development; not the bench."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06139_b200 as adc  # noqa: E402
from paper_2203_06139_b200.launch import set_gaussnd_variant  # noqa: E402
from paper_2203_06139_b200 import synth  # noqa: E402

dev = torch.device("cuda:0")
print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0).multi_processor_count)
os.system("free -g | head -2; nproc")


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), float(np.min(ts))


# K1 1e6 and 1e8
for n in (10**6, 10**8):
    x = torch.rand(n, dtype=torch.float64, device=dev)
    p = torch.rand(n, dtype=torch.float64, device=dev)
    dx = torch.zeros(n, dtype=torch.float64, device=dev)
    dp = torch.zeros(n, dtype=torch.float64, device=dev)
    b = adc.BufferSet(arrays={"x": x, "p": p, "dx": dx, "dp": dp}, scalars={"sigma": 1.3})
    cfg = adc.LaunchConfig(n // 256 + 1, 256, n)
    med, mn = timeit(lambda: adc.launch("compute", cfg, b))
    print(f"gauss1d n={n}: {med:.4f} ms  {48*n/med/1e6:.1f} GB/s (min {48*n/mn/1e6:.1f})")
    del x, p, dx, dp, b

for dim, n in ((100, 10**7), (1000, 10**6)):
    p = torch.rand((dim, n), dtype=torch.float64, device=dev) * 4 - 2
    x = p + 0.1 * torch.randn((dim, n), dtype=torch.float64, device=dev)
    dx = torch.zeros_like(x)
    dp = torch.zeros_like(x)
    for v in ((3, 8, 9) if dim == 100 else (2,)):
        set_gaussnd_variant(v)
        med, mn = timeit(lambda: adc.launch_batch("gaussnd_grad_0_1", x, p, 1.3, dx, dp), reps=5)
        print(f"gaussnd dim={dim} n={n} variant={v}: {med:.3f} ms  {48*dim*n/med/1e6:.1f} GB/s "
              f"(min {48*dim*n/mn/1e6:.1f})  {2*dim*n/med/1e-3:.3e} pt*param/s")
    set_gaussnd_variant(0)
    del x, p, dx, dp
    torch.cuda.empty_cache()

for bins in (10**6, 10**8):
    lam = torch.full((bins,), 100.0, dtype=torch.float64, device=dev)
    counts = torch.poisson(lam)
    counts[::100] = 0
    ev = float(counts.sum())
    h = adc.Histogram(bins, -5.0, 5.0, ev, counts)
    pl = adc.Chi2Plan("gpoly", 6, h)
    q = list(synth.GPOLY_INIT)
    for fast in (False, True):
        pl.set_precision(fast)
        for _ in range(3):
            pl.gradient(q)
        t0 = time.perf_counter()
        for _ in range(20):
            pl.gradient(q)
        dt = (time.perf_counter() - t0) / 20
        t0 = time.perf_counter()
        for _ in range(20):
            pl.chi2(q)
        dv = (time.perf_counter() - t0) / 20
        print(f"chi2 bins={bins} fast={fast}: gradient API {dt*1e3:.4f} ms/pass, value {dv*1e3:.4f} ms")
    del pl, counts
