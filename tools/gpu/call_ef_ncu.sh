#!/bin/bash
# (needs tools/experiments/huffman_fused_encoder.patch applied: the fused encoder is not in the tree, DESIGN 10)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/ef; mkdir -p $O
SZ3G_HUFF_FUSED=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_huff_encode_fused' --launch-skip 2 -c 1 -o $O/fused_c5 -f python tools/huff_time.py --config c5 > $O/ncu_fused.log 2>&1; echo "ncu rc=$?"
