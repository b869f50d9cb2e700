#!/bin/bash
# rare-path instance (row-ordered vs per-lane outlier append) on the low-outlier small-radius leg c3 at R = 4, and on c3 at R = 64 / 1024
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/row; mkdir -p $O
L=paper_2111_02925_b200/lib
for R in 4 64 1024; do
for v in libsz3g.so ab/LANES.so; do
echo "== c3 R=$R $v"; SZ3G_LIB=$L/$v timeout 300 python tools/stress_time.py --config c3 --radius $R --steps 10 2>&1 | tail -1 | cut -c1-300
done; done | tee $O/row.log
