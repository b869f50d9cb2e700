"""ncu target for the encoder stage: compress one config, then codebook / encode / decode twice.
  python tools/huff_target.py [config]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_02925_b200 import sz3g
from synth import make_field, config_by_name
cfg = config_by_name(sys.argv[1] if len(sys.argv) > 1 else "c3")
x = make_field(cfg, device="cuda")
res = sz3g.compress(x, cfg.eb, cfg.eb_mode, cfg.radius)
codes = res.codes.view(-1)
for it in range(2):
    t = sz3g.huffman_codebook(res.hist)
    hs = sz3g.huffman_encode(codes, t)
    out = sz3g.huffman_decode(hs, t)
torch.cuda.synchronize()
assert torch.equal(out, codes)
print("ok", cfg.name, hs.words() * 32 / codes.numel(), "bits/code")
