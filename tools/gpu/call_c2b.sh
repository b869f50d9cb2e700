#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/c2p; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_memsafety.py tests/test_gpu_chaos.py tests/test_gpu_dist.py -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for c in c2 c3; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_$c.csv python tools/ncu_target.py $c > /dev/null 2>&1
python tools/launch_table.py $O/launches_$c.csv "# $c" | tail -7
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-huffman --no-truncation --no-lr --no-e2e --no-cpu-baseline --no-interp --configs c2 > $O/bench_c2.json 2>$O/bench_c2.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/c2p/bench_c2.json').read().strip().splitlines()[-1])
c=d['configs']['c2']
print({k:(round(v['ms_per_launch'],4), round(v['frac'],3), round(v.get('frac_of_stream') or 0,3)) for k,v in c.items() if k.endswith('_roofline')}, c['ms_per_step'])
PY
