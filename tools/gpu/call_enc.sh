#!/bin/bash
# Huffman / stream / pipeline tests, then encode / decode timing per config
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/enc; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_huffman.py tests/test_gpu_stream.py tests/test_gpu_pipeline.py -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"
tail -2 $O/tests.log
for c in c5 c3 c2 c4; do echo "== $c"; timeout 300 python tools/huff_time.py --config $c 2>&1 | tail -1 | cut -c1-100; done | tee $O/time.log
