"""Small fixed workload for ncu captures: compress + decompress of one config, 3 times.
  python tools/ncu_target.py <config> [two-pass|fused]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_02925_b200 import sz3g
from synth import make_field, config_by_name
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
path = sys.argv[2] if len(sys.argv) > 2 else "two-pass"
cfg = config_by_name(name)
x = make_field(cfg, device="cuda")
bufs = sz3g.CompressBuffers(x.shape, x.dtype, cfg.radius, device=x.device)
out = torch.empty_like(x)
for it in range(3):
    if path == "two-pass" and cfg.eb_mode == "rel":
        res = sz3g.compress_two_pass(x, cfg.eb, cfg.eb_mode, cfg.radius, bufs=bufs).finalize()
    else:
        res = sz3g.regression_compress(x, cfg.eb, cfg.eb_mode, cfg.radius, bufs=bufs).finalize()
    sz3g.regression_decompress(res.codes, res.coef_codes, res.outlier_idx, res.outlier_val, res.n_outliers,
                               res.eb_abs, res.radius, x.dtype, out=out)
torch.cuda.synchronize()
print("ok", name, path, res.n_outliers, res.eb_abs)
