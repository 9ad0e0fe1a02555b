"""Pinned host <-> device copy bandwidth on this box (the e2e bound): H2D and
D2H alone and concurrently (two streams), 134 MB buffers. Not a test."""
import torch

n = 16777216
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
h3 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
d3 = torch.empty(n, dtype=torch.float64, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
B = n * 8


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t = timed(lambda: d1.copy_(h1, non_blocking=True))
print(f"H2D alone {B / t / 1e6:.1f} GB/s")
t = timed(lambda: h1.copy_(d1, non_blocking=True))
print(f"D2H alone {B / t / 1e6:.1f} GB/s")


def both():
    with torch.cuda.stream(s_in):
        d1.copy_(h1, non_blocking=True)
        d2.copy_(h2, non_blocking=True)
    with torch.cuda.stream(s_out):
        h3.copy_(d3, non_blocking=True)


t = timed(both)
print(f"2 x H2D + 1 x D2H concurrently: {t:.2f} ms per set -> H2D {2 * B / t / 1e6:.1f} GB/s, "
      f"e2e bound for a 28.47 GB step = {28.47e9 / (t * 1e-3) / 1e9:.0f} GB/s")
