#!/bin/bash
# r02 session 3: full GPU suite, default bench, launch list of the bench step, ncu of the new decoder
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 420 python -m pytest tests -m gpu -x -q > gpurun_out/s3_gpu_tests.log 2>&1
timeout 420 python bench.py > gpurun_out/s3_bench_final.json 2> gpurun_out/s3_bench_final.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/s3_launch.csv python bench.py --steps 2 --warmup 3 --configs '' > gpurun_out/s3_ncu_launch.log 2>&1
