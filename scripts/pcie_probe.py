"""Host<->device copy bandwidth from pinned memory: H2D alone, D2H alone, both at
once on two streams (what the e2e streaming mode overlaps)."""
import time

import torch

n = 1 << 27  # 1 GiB of doubles
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


gb = n * 8 / 1e9
print(f"H2D {gb / timed(h2d):.1f} GB/s  D2H {gb / timed(d2h):.1f} GB/s  both at once {2 * gb / timed(both):.1f} GB/s total")
