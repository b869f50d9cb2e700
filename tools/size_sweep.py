"""Kernel efficiency against field size (GPU): one config's recipe at several dim-0 extents, the bench
leg's measurement (RoundTrip from CUDA graphs, L2 flushed before every step, SURVEY 8(d) bytes).
  python tools/size_sweep.py c4 64 256 1024"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2111_02925_b200 import sz3g  # noqa: E402
from synth import config_by_name, make_field  # noqa: E402

name = sys.argv[1]
cfg = config_by_name(name)
sz3g.load()
peaks = bench.measured_peaks()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n0 in (int(v) for v in sys.argv[2:]):
    shape = (n0,) + tuple(cfg.shape[1:])
    x = make_field(cfg, device="cuda", shape=shape)
    d = bench.config_leg(sz3g, name, peaks, 10, 3, flush, x=x)
    print(json.dumps({"shape": shape, "MB": round(x.numel() * x.element_size() / 1e6, 1),
                      **{k: round(d[k + "_roofline"]["frac"], 3) for k in ("analyze", "quantize", "decompress")},
                      **{k + "_us": round(1e3 * d[k + "_roofline"]["ms_per_launch"], 1)
                         for k in ("analyze", "quantize", "decompress")}}), flush=True)
    del x
    torch.cuda.empty_cache()
