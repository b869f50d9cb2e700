"""Why is the quantise kernel slower inside the bench step than back to back?  Times k_compress_tma
(c5, two-pass) (a) back to back, (b) inside RoundTrip steps, (c) inside steps with an L2 flush before
it, (d) after a 2 ms idle gap (a spin kernel), (e) inside steps without the decompress."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2111_02925_b200 import sz3g  # noqa: E402
from paper_2111_02925_b200.roundtrip import RoundTrip  # noqa: E402
from synth import config_by_name, make_field  # noqa: E402

cfg = config_by_name("c5")
sz3g.load()
x = make_field(cfg, device="cuda")
rt = RoundTrip(x, cfg.eb, cfg.eb_mode, cfg.radius)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
st = rt.stream
for _ in range(3):
    rt.step()
res = {}


def q_only(n=10):
    ts = []
    for _ in range(n):
        a, b = E(), E()
        rt._range_reset(st)
        a.record(st)
        rt._quantize(st)
        b.record(st)
        ts.append((a, b))
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ts)[n // 2]


def in_step(n=10, pre=None, skip_dec=False):
    ts = []
    for _ in range(n):
        a, b = E(), E()
        rt._analyze(st)
        rt._range_reset(st)
        if pre:
            pre()
        a.record(st)
        rt._quantize(st)
        b.record(st)
        if not skip_dec:
            rt._decompress(st)
        ts.append((a, b))
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ts)[n // 2]


res["back_to_back"] = q_only()
res["in_step"] = in_step()
res["in_step_flush_before"] = in_step(pre=lambda: flush.fill_(1))
res["in_step_idle_2ms"] = in_step(pre=lambda: torch.cuda._sleep(2_000_000))
res["in_step_no_decompress"] = in_step(skip_dec=True)
res["back_to_back_again"] = q_only()
print(json.dumps(res))
