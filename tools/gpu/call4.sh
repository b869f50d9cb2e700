#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/c4
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x -s -k graph > gpurun_out/c4/test_graph.log 2>&1; echo "graph test rc=$?"
timeout 900 python tools/ab.py --config c4 --path two-pass --flush --graphs --rounds 4 --reps 10 V0=paper_2111_02925_b200/lib/libsz3g.so V1=paper_2111_02925_b200/lib/ab/V1.so V2=paper_2111_02925_b200/lib/ab/V2.so V3=paper_2111_02925_b200/lib/ab/V3.so V4=paper_2111_02925_b200/lib/ab/V4.so > gpurun_out/c4/ab_c4.log 2>&1
tail -5 gpurun_out/c4/ab_c4.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-huffman --no-truncation --no-lr --no-e2e --no-cpu-baseline > gpurun_out/c4/bench.json 2> gpurun_out/c4/bench.err; echo "bench rc=$?"
