"""Time sz3g_regression_analyze on one config (CUDA events, median of --reps); prints tune.py's JSON
format (compress_ms = analyze, decompress_ms = 0) so tools/ab.py --tool analyze_time.py can A/B builds."""
import argparse
import json
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_02925_b200 import sz3g
from synth import make_field, config_by_name

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--reps", type=int, default=7)
a, _ = ap.parse_known_args()
cfg = config_by_name(a.config)
x = make_field(cfg, device="cuda")
mm = torch.empty(2, dtype=torch.float64, device="cuda")
beta = torch.empty((sz3g.num_blocks(x.shape), 4), dtype=torch.float64, device="cuda")
sz3g.regression_analyze(x, mm, beta)
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sz3g.regression_analyze(x, mm, beta)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(json.dumps({"compress_ms": [statistics.median(ts)], "decompress_ms": [0.0]}))
