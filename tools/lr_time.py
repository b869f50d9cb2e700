"""Time SZ3-LR on one config (CUDA events, median of --reps): lr_quantize and lr_decompress, the share of
Lorenzo blocks, and Huffman bits per code against the regression-only path.  Prints one JSON line in
tools/tune.py's format (compress_ms = lr_quantize, decompress_ms = lr_decompress) plus extra keys."""
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
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--flags", type=int, default=int(os.environ.get("LR_FLAGS", "0")))
ap.add_argument("--no-hist", action="store_true")
ap.add_argument("rest", nargs="*")
a, _ = ap.parse_known_args()
cfg = config_by_name(a.config)
x = make_field(cfg, device="cuda")
bufs = sz3g.CompressBuffers(x.shape, x.dtype, cfg.radius, None, x.device)
minmax, beta = sz3g.regression_analyze(x, bufs.minmax, bufs.beta_buffer())
res = sz3g.lr_quantize(x, cfg.eb, cfg.eb_mode, cfg.radius, minmax, beta, bufs, flags=a.flags).finalize()
out = torch.empty_like(x)
qs, ds = [], []
for _ in range(a.reps):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    sz3g.lr_quantize(x, cfg.eb, cfg.eb_mode, cfg.radius, minmax, beta, bufs, flags=a.flags, hist=not a.no_hist)
    e1.record()
    sz3g.lr_decompress(res.codes, res.coef_codes, res.lr_flags, res.outlier_idx, res.outlier_val,
                       res.outlier_idx.numel(), cfg.eb, cfg.radius, x.dtype, out=out, d_outlier_count=res.outlier_count,
                       eb_mode=cfg.eb_mode, d_minmax=minmax)
    e2.record()
    torch.cuda.synchronize()
    qs.append(e0.elapsed_time(e1))
    ds.append(e1.elapsed_time(e2))
res = sz3g.lr_quantize(x, cfg.eb, cfg.eb_mode, cfg.radius, minmax, beta, bufs, flags=a.flags).finalize()
t = sz3g.huffman_codebook(res.hist)
hs = sz3g.huffman_encode(res.codes.view(-1), t)
lr_bits = hs.words() * 32 / x.numel()
frac = float(res.lr_flags.float().mean())
reg = sz3g.compress(x, cfg.eb, cfg.eb_mode, cfg.radius)
t2 = sz3g.huffman_codebook(reg.hist)
reg_bits = sz3g.huffman_encode(reg.codes.view(-1), t2).words() * 32 / x.numel()
err = float((out.double() - x.double()).abs().max())
print(json.dumps({"compress_ms": [statistics.median(qs)], "decompress_ms": [statistics.median(ds)],
                  "lorenzo_fraction": frac, "bits_per_code_lr": lr_bits, "bits_per_code_regression": reg_bits,
                  "max_abs_err": err, "eb_abs": res.eb_abs}))
