#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/c5
timeout 900 python -m pytest tests/test_gpu_huffman.py tests/test_gpu_stream.py -q -x > gpurun_out/c5/huff_tests.log 2>&1; echo "huff tests rc=$?"; tail -2 gpurun_out/c5/huff_tests.log
timeout 900 python tools/ab.py --tool huff_time.py --config c5 --rounds 3 --reps 5 H0=paper_2111_02925_b200/lib/ab/H0.so H1=paper_2111_02925_b200/lib/libsz3g.so > gpurun_out/c5/ab_huff.log 2>&1
tail -3 gpurun_out/c5/ab_huff.log
