#!/bin/bash
# c5 bench-path parity + compute-sanitizer sweep (one gpurun call)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/san
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/san/smi.txt
timeout 1500 python -m pytest tests/test_gpu_c5.py -x -q -s > gpurun_out/san/c5_test.log 2>&1; echo "c5 rc=$?" >> gpurun_out/san/rc.txt
for tool in memcheck synccheck initcheck racecheck; do
  for fam in regression lr huffman truncation stream; do
    timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_cases.py --only $fam > gpurun_out/san/${tool}_${fam}.log 2>&1
    echo "$tool $fam rc=$?" >> gpurun_out/san/rc.txt
  done
done
cat gpurun_out/san/rc.txt
