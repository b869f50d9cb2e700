#!/bin/bash
# timing experiment: outlier counter spread over 128 addresses (wrong results) vs the single counter;
# lib/ab/SPREAD.so = the tree with tools/experiments/outlier_counter_spread.patch applied, built with -DSZ3G_EXP_SPREAD=1
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/row; mkdir -p $O
L=paper_2111_02925_b200/lib
for cr in "c3 4" "c5 16" "c5 64"; do set -- $cr
for v in libsz3g.so ab/SPREAD.so; do
echo "== $1 R=$2 $v"; SZ3G_LIB=$L/$v timeout 300 python tools/stress_time.py --config $1 --radius $2 --steps 5 2>&1 | tail -1 | cut -c1-300
done; done | tee $O/spread.log
