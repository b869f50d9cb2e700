#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/c2p; mkdir -p $O
python tools/ncu_target.py c2 > $O/run.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:'k_compress_tma|k_decompress_plain' --launch-skip 2 -c 2 -o $O/c2 -f python tools/ncu_target.py c2 > $O/ncu.log 2>&1; echo "ncu rc=$?"
