"""Achievable DRAM bandwidth for the traffic mixes of the hot kernels, measured with plain streaming
kernels (torch casts) at the c5 size: u16 -> f32 (read 2 B, write 4 B per element: the decompressor's
mix) and f32 -> u16 (read 4 B, write 2 B: the quantiser's mix), plus a f32 copy (1:1, the
MEASURED_PEAKS.json recipe).  CUDA events, median of --reps after a warm-up; prints one JSON line."""
import argparse
import json
import statistics

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024 * 2048 * 2048)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
n = a.n
f = torch.empty(n, dtype=torch.float32, device="cuda").uniform_(0, 60000)
u = torch.empty(n, dtype=torch.int16, device="cuda")
g = torch.empty_like(f)


def timed(fn, nbytes):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    return {"ms": ms, "gbs": nbytes / ms / 1e6}


out = {
    "copy_f32 (1:1)": timed(lambda: g.copy_(f), 8 * n),
    "f32->i16 (2:1, quantise mix)": timed(lambda: u.copy_(f), 6 * n),
    "i16->f32 (1:2, decompress mix)": timed(lambda: g.copy_(u), 6 * n),
}
print(json.dumps({"n": n, "mixes": out}))
