#!/bin/bash
# launch lists of c3/c4 round trips + full captures of the analyze / decompress kernels (c3, c4)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/ncu_cfg; mkdir -p $O
for c in c3 c4 c2; do
  python tools/ncu_target.py $c > $O/run_$c.log 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_$c.csv python tools/ncu_target.py $c > /dev/null 2>&1
done
for c in c4 c3; do
  ncu --set full --import-source on --clock-control none -k regex:'k_analyze_tma|k_decompress_tma|k_compress_tma' --launch-skip 3 -c 3 -o $O/full_$c -f python tools/ncu_target.py $c > $O/full_$c.log 2>&1
done
ls -la $O
