#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/c8
timeout 900 python -m pytest tests/test_gpu_huffman.py tests/test_gpu_stream.py -q -x > gpurun_out/c8/tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/c8/tests.log
for c in c5 c2; do python tools/huff_time.py --config $c; done
timeout 900 python tools/ab.py --tool huff_time.py --config c5 --rounds 3 --reps 5 H2=paper_2111_02925_b200/lib/ab/H2.so N=paper_2111_02925_b200/lib/libsz3g.so 2>&1 | tail -2
timeout 900 python tools/ab.py --tool huff_time.py --config c2 --rounds 3 --reps 5 H2=paper_2111_02925_b200/lib/ab/H2.so N=paper_2111_02925_b200/lib/libsz3g.so 2>&1 | tail -2
