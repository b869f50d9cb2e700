#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/c2
timeout 1200 python -m pytest tests/test_gpu_ties.py tests/test_gpu_stream.py tests/test_gpu_pipeline.py tests/test_gpu_dist.py -x -q -s > gpurun_out/c2/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/c2/rc.txt
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/c2/bench.json 2> gpurun_out/c2/bench.err; echo "bench rc=$?" >> gpurun_out/c2/rc.txt
cat gpurun_out/c2/rc.txt
