#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/c7
timeout 900 python -m pytest tests/test_gpu_chaos.py tests/test_gpu_huffman.py -q -x > gpurun_out/c7/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/c7/tests.log
python tools/ncu_target.py c5 two-pass > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:'k_compress_tma' --launch-skip 2 -c 1 -o gpurun_out/c7/q_c5 -f python tools/ncu_target.py c5 two-pass > gpurun_out/c7/ncu.log 2>&1; echo "ncu rc=$?"
