#!/bin/bash
# f64 decompress kernel shapes on c4 (A/B, alternating processes)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/ab64; mkdir -p $O
L=paper_2111_02925_b200/lib
timeout 900 python tools/ab.py --config c4 --path two-pass --flush --graphs --rounds 3 --reps 10 N=$L/libsz3g.so V1=$L/ab/V1.so V3=$L/ab/V3.so V4=$L/ab/V4.so V5=$L/ab/V5.so > $O/ab_c4.log 2>&1
tail -8 $O/ab_c4.log
