#!/usr/bin/env python
"""A/B of library builds in the bench's own regime: each variant runs in its own process, generates
the config once, replays RoundTrip steps from CUDA graphs for --warm-steps untimed steps (the GPU
reaches its sustained power / clock state) then --steps timed steps, and reports the median analyze /
quantise / decompress / step times.  Variants alternate over --rounds.

  python tools/ab_step.py --config c5 --rounds 3 A=paper_2111_02925_b200/lib/ab/A.so B=...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(a):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2111_02925_b200 import sz3g
    from paper_2111_02925_b200.roundtrip import RoundTrip
    from synth import config_by_name, make_field
    cfg = config_by_name(a.config)
    sz3g.load()
    x = make_field(cfg, device="cuda")
    rt = RoundTrip(x, cfg.eb, cfg.eb_mode, cfg.radius).capture()
    for _ in range(a.warm_steps):
        rt.step()
    recs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(a.steps)]
    for r in recs:
        rt.step(r)
    torch.cuda.synchronize()
    med = lambda i, j: statistics.median(r[i].elapsed_time(r[j]) for r in recs)   # noqa: E731
    print(json.dumps({"analyze_ms": med(4, 5), "quantize_ms": med(0, 1), "decompress_ms": med(2, 3),
                      "step_ms": med(4, 3)}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--warm-steps", type=int, default=40)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--worker", action="store_true")
    ap.add_argument("variants", nargs="*")
    a = ap.parse_args()
    if a.worker:
        worker(a)
        return
    vs = [v.split("=", 1) for v in a.variants]
    res = {n: [] for n, _ in vs}
    for r in range(a.rounds):
        for n, path in vs:
            env = dict(os.environ, SZ3G_LIB=path if os.path.isabs(path) else os.path.join(ROOT, path))
            out = subprocess.run([sys.executable, __file__, "--worker", "--config", a.config, "--warm-steps",
                                  str(a.warm_steps), "--steps", str(a.steps)], env=env, capture_output=True, text=True)
            line = [l for l in out.stdout.splitlines() if l.startswith("{")]
            if not line:
                print(n, "FAILED", out.stderr[-2000:], flush=True)
                continue
            d = json.loads(line[-1])
            res[n].append(d)
            print(json.dumps({"round": r, "variant": n, **d}), flush=True)
    for n, ds in res.items():
        if ds:
            print(json.dumps({"variant": n, **{k: round(statistics.median(d[k] for d in ds), 4) for k in ds[0]}}))


if __name__ == "__main__":
    main()
