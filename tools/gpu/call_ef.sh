#!/bin/bash
# (needs tools/experiments/huffman_fused_encoder.patch applied: the fused encoder is not in the tree, DESIGN 10)
# fused Huffman encoder (SZ3G_HUFF_FUSED=1): Huffman / stream / pipeline tests, then encode timing off vs on
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/ef; mkdir -p $O
SZ3G_HUFF_FUSED=1 timeout 600 python -m pytest tests/test_gpu_huffman.py tests/test_gpu_stream.py tests/test_gpu_pipeline.py -x -q -p no:cacheprovider > $O/tests_fused.log 2>&1; echo "fused tests rc=$?" | tee -a $O/rc.txt
tail -15 $O/tests_fused.log
for c in c5 c3 c2 c4; do
  for f in 0 1; do
    echo "== $c fused=$f" | tee -a $O/time.log
    SZ3G_HUFF_FUSED=$f timeout 300 python tools/huff_time.py --config $c 2>&1 | tail -1 | tee -a $O/time.log
  done
done
