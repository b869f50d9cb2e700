#!/bin/bash
# Build libsz3g with -Xptxas -v and print registers / spills / smem per kernel (short names).
cd "$(dirname "$0")/.." && python -m paper_2111_02925_b200.build --force -v 2>&1 | python3 -c '
import sys,re
name=None
for line in sys.stdin:
    m=re.search(r"Compiling entry function .(\S+).", line)
    if m: name=m.group(1); continue
    m=re.search(r"(\d+) bytes spill stores", line)
    if m: spill=m.group(1); continue
    m=re.search(r"Used (\d+) registers", line)
    if m and name:
        short=re.sub(r"_ZN\d+_GLOBAL__N__\w+?_\d+_sz3g_cu_\w{8}\d+","",name)[:60]
        print(f"{short:62s} regs={m.group(1):>4s} spill={spill}")
    if "error" in line: print(line.rstrip())
'
