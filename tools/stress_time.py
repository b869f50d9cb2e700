"""Time the bench step (RoundTrip from CUDA graphs) on a config at another radius (the labelled stress
variants, e.g. c5 at R = 16): median analyze / quantise / decompress / step ms over --steps after
--warm-steps.  One JSON line."""
import argparse
import json
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2111_02925_b200 import sz3g  # noqa: E402
from paper_2111_02925_b200.roundtrip import RoundTrip  # noqa: E402
from synth import config_by_name, make_field  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--radius", type=int, default=16)
ap.add_argument("--warm-steps", type=int, default=3)
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
cfg = config_by_name(a.config)
sz3g.load()
x = make_field(cfg, device="cuda")
rt = RoundTrip(x, cfg.eb, cfg.eb_mode, a.radius, outlier_cap=x.numel()).capture()
for _ in range(a.warm_steps):
    rt.step()
recs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(a.steps)]
for r in recs:
    rt.step(r)
torch.cuda.synchronize()
res = rt.result()
st = sz3g.error_stats(x, rt.out, res.eb_abs).cpu().tolist()
med = lambda i, j: statistics.median(r[i].elapsed_time(r[j]) for r in recs)   # noqa: E731
print(json.dumps({"config": a.config, "radius": a.radius, "outliers": res.n_outliers, "analyze_ms": med(4, 5),
                  "quantize_ms": med(0, 1), "decompress_ms": med(2, 3), "step_ms": med(4, 3),
                  "max_err_ok": st[2] == 0 and st[0] <= res.eb_abs}))
