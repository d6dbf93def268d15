"""Host<->device copy bandwidth on the box (pinned buffers): H2D alone, D2H
alone, both directions at once — the ceiling of the e2e (host-buffer) path."""
import time

import torch

n = 2 << 30  # 2 GiB per buffer
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    return reps * n / (time.perf_counter() - t0) / 1e9


for _ in range(2):
    print(f"H2D {run(True, False):.1f} GB/s, D2H {run(False, True):.1f} GB/s, "
          f"both: {run(True, True):.1f} GB/s each direction")
