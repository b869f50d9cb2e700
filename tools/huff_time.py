"""Time the Huffman encode / decode of one config's codes (CUDA events, median of --reps); prints one
JSON line in tools/tune.py's format (compress_ms = encode, decompress_ms = decode) so that
tools/ab.py --tool huff_time.py can A/B library variants."""
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
ap.add_argument("--reps", type=int, default=6)
ap.add_argument("--max-len", type=int, default=16)
ap.add_argument("rest", nargs="*")
a, _ = ap.parse_known_args()
cfg = config_by_name(a.config)
x = make_field(cfg, device="cuda")
res = sz3g.compress(x, cfg.eb, cfg.eb_mode, cfg.radius)
del x
codes = res.codes.view(-1)
t = sz3g.huffman_codebook(res.hist, max_len=a.max_len).check()
hs = sz3g.huffman_encode(codes, t)
out = sz3g.huffman_decode(hs, t)
torch.cuda.synchronize()
assert torch.equal(out, codes), "round trip failed"
enc, dec = [], []
for _ in range(a.reps):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    sz3g.huffman_encode(codes, t, payload=hs.payload, offsets=hs.offsets)
    e1.record()
    sz3g.huffman_decode(hs, t, out=out)
    e2.record()
    torch.cuda.synchronize()
    enc.append(e0.elapsed_time(e1))
    dec.append(e1.elapsed_time(e2))
lens = t.lengths.cpu().double()
h = res.hist.cpu().double()
print(json.dumps({"compress_ms": [statistics.median(enc)], "decompress_ms": [statistics.median(dec)],
                  "max_len": a.max_len, "bits_per_code": float((lens * h).sum() / h.sum()),
                  "frac_codes_over_12_bits": float(h[lens > 12].sum() / h.sum()),
                  "lut2_entries": int(65536 - sum(int((lens == L).sum()) << (16 - L) for L in range(1, 13)))}))
