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

# the e2e pipeline's per-field volumes at c5: 16 GiB in; x' (16 GiB) + the compressed stream (3.47 GB) out
import sys
if "--e2e" in sys.argv:
    del h1, h2, d1, d2
    torch.cuda.empty_cache()
    gib = 1 << 30
    hx = torch.empty(16 * gib, dtype=torch.uint8, pin_memory=True)
    ho = torch.empty(16 * gib, dtype=torch.uint8, pin_memory=True)
    hc = torch.empty(3_470_000_000, dtype=torch.uint8, pin_memory=True)
    dx = torch.empty(16 * gib, dtype=torch.uint8, device="cuda")
    do = torch.empty(16 * gib, dtype=torch.uint8, device="cuda")
    dc = torch.empty(3_470_000_000, dtype=torch.uint8, device="cuda")

    def e2e_copies():
        with torch.cuda.stream(s1):
            dx.copy_(hx, non_blocking=True)
        with torch.cuda.stream(s2):
            hc.copy_(dc, non_blocking=True)
            ho.copy_(do, non_blocking=True)
        s1.synchronize()
        s2.synchronize()

    ms = t(e2e_copies, reps=2)
    print(f"e2e volumes (16 GiB in || 3.47 GB + 16 GiB out): {ms:.1f} ms, "
          f"{(16 * gib) / ms / 1e6:.1f} GB/s of input")
