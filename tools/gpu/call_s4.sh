#!/bin/bash
# r02 session 4: smoke, full GPU suite, default bench, launch list of the bench step, ncu of the Huffman kernels
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/s4; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/rc.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launch.csv python bench.py --steps 2 --warmup 3 --configs '' > $O/ncu_launch.log 2>&1; echo "launch rc=$?" >> $O/rc.txt
python tools/huff_time.py --config c5 > $O/huff_time.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_huff' --launch-skip 6 -c 8 -o $O/huff_c5 -f python tools/huff_time.py --config c5 > $O/ncu_huff.log 2>&1; echo "ncu huff rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -3 $O/gpu_tests.log; cat $O/huff_time.log | tail -5
