"""Host<->device copy ceilings with pinned memory: H2D alone, D2H alone, both at once (two streams)."""
import torch
n = 4 << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        torch.cuda.synchronize()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    s1.synchronize()


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    s2.synchronize()


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    s1.synchronize()
    s2.synchronize()


for name, fn, nb in (("h2d", h2d, n), ("d2h", d2h, n), ("both", both, 2 * n)):
    ms = t(fn)
    print(f"{name}: {nb / ms / 1e6:.1f} GB/s ({ms:.1f} ms)")
