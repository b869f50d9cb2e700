#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/c9
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c9/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/c9/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/c9/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/c9/tests.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/c9/bench.json 2> gpurun_out/c9/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/c9/bench.err
