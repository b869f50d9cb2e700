#!/bin/bash
# (needs tools/experiments/huffman_fused_encoder.patch applied: the fused encoder is not in the tree, DESIGN 10)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/ef; mkdir -p $O
cat > /tmp/ef_time.py <<'PY'
import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
from paper_2111_02925_b200 import sz3g
from synth import make_field, config_by_name
cfg = config_by_name("c5")
x = make_field(cfg, device="cuda")
res = sz3g.compress(x, cfg.eb, cfg.eb_mode, cfg.radius); del x
codes = res.codes.view(-1)
t = sz3g.huffman_codebook(res.hist).check()
hs = sz3g.huffman_encode(codes, t)
enc = []
for _ in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sz3g.huffman_encode(codes, t, payload=hs.payload, offsets=hs.offsets); e1.record()
    torch.cuda.synchronize(); enc.append(e0.elapsed_time(e1))
print("encode_ms", statistics.median(enc))
PY
for v in "SZ3G_HUFF_FUSED=0" "SZ3G_HUFF_FUSED=1" "SZ3G_HUFF_FUSED=1 SZ3G_EF_FAKE=1"; do echo "== $v"; env $v timeout 300 python /tmp/ef_time.py 2>&1 | tail -1; done
