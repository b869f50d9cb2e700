"""Time SZ3-Interp compress / decompress on one config (CUDA events, median of --reps)."""
import argparse
import json
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2111_02925_b200 import sz3g  # noqa: E402
from synth import config_by_name, make_field  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--reps", type=int, default=3)
a, _ = ap.parse_known_args()
cfg = config_by_name(a.config)
sz3g.load()
x = make_field(cfg, device="cuda")
mm = sz3g.value_range(x)
res = sz3g.interp_compress(x, cfg.eb, cfg.eb_mode, cfg.radius, d_minmax=mm, outlier_cap=max(1 << 20, x.numel() // 64))
res.finalize()
out = torch.empty_like(x)
tc, td = [], []
for _ in range(a.reps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    sz3g.interp_compress(x, cfg.eb, cfg.eb_mode, cfg.radius, d_minmax=mm, out=res)
    e[1].record()
    sz3g.interp_decompress(res.codes, res.outlier_idx, res.outlier_val, res.outlier_idx.numel(), cfg.eb, cfg.radius,
                           x.dtype, out=out, d_outlier_count=res.outlier_count, eb_mode=cfg.eb_mode, d_minmax=mm)
    e[2].record()
    torch.cuda.synchronize()
    tc.append(e[0].elapsed_time(e[1]))
    td.append(e[1].elapsed_time(e[2]))
res.finalize()
st = sz3g.error_stats(x, out, res.eb_abs).cpu().tolist()
h = res.hist.cpu().double()
p = h[h > 0] / h.sum()
print(json.dumps({"config": a.config, "compress_ms": statistics.median(tc), "decompress_ms": statistics.median(td),
                  "outliers": res.n_outliers, "max_err": st[0], "eb_abs": res.eb_abs, "above": st[2],
                  "entropy_bits": float(-(p * p.log2()).sum())}))
