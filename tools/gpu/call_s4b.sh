#!/bin/bash
# r02 session 4, final state: smoke, full GPU suite, default bench, launch lists (bench step, c2), ncu of the c2 kernels
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/s4b; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/rc.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launch.csv python bench.py --steps 2 --warmup 3 --configs '' > $O/ncu_launch.log 2>&1; echo "launch rc=$?" >> $O/rc.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c2.csv python tools/ncu_target.py c2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:'k_compress_tma|k_decompress_staged' --launch-skip 2 -c 2 -o $O/c2 -f python tools/ncu_target.py c2 > $O/ncu_c2.log 2>&1; echo "ncu c2 rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -2 $O/gpu_tests.log
