"""Row alignment on the B200's HBM, independent of our kernels: torch's own
copy and read-only reduction over [rows, n] views whose rows start 8 B into a
128 B line (leading dimension n + 1) vs 128 B aligned (n + 16).  Separates the
read and write sides of the K2 slowdown on 16-byte-aligned rows."""
import torch

rows, n = 100, 10_000_000


def ms(fn, reps=8):
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
    ts.sort()
    return ts[len(ts) // 2]


for name, ld in (("aligned (ld = n + 16)", n + 16), ("odd (ld = n + 1)", n + 1)):
    src = torch.rand(rows, ld, dtype=torch.float64, device="cuda")[:, :n]
    dst = torch.empty(rows, ld, dtype=torch.float64, device="cuda")[:, :n]
    nbytes = rows * n * 8
    t_copy = ms(lambda: dst.copy_(src))
    t_read = ms(lambda: src.sum(dim=1))
    t_write = ms(lambda: dst.fill_(1.0))
    print(f"{name}: copy {2 * nbytes / t_copy / 1e6:.0f} GB/s, read-only {nbytes / t_read / 1e6:.0f} GB/s, "
          f"write-only {nbytes / t_write / 1e6:.0f} GB/s", flush=True)
    del src, dst
