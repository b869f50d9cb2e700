#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/c3
timeout 2400 python -m pytest tests -m gpu -q -x -s -p no:cacheprovider > gpurun_out/c3/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/c3/rc.txt
cat gpurun_out/c3/rc.txt
