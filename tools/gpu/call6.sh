#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/c6
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_chaos.py -q -x -k "two_pass or graph or chaos or value_range" > gpurun_out/c6/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/c6/tests.log
for c in c4 c3; do
timeout 600 python tools/ab.py --config $c --path two-pass --flush --graphs --rounds 3 --reps 10 H1=paper_2111_02925_b200/lib/ab/H1.so N=paper_2111_02925_b200/lib/libsz3g.so > gpurun_out/c6/ab_$c.log 2>&1
tail -2 gpurun_out/c6/ab_$c.log
done
