"""Attribute an ncu source page (SASS, --page source --csv) to CUDA source lines through the line table of
the cubin (nvdisasm -g): instructions executed per element and stall samples per file:line.
  python tools/ncu_lines.py page.csv kernel.cubin mangled_kernel_name n_elements [top]"""
import collections
import csv
import re
import subprocess
import sys

page, cubin, kname, n = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
lines = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(lines) if l.startswith(".text." + kname)][0]
cur, off2loc = None, {}
for l in lines[start + 1:]:
    if l.startswith(".text.") or (l.startswith("//---------------------") and off2loc):
        break
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = m.group(1).split("/")[-1] + ":" + m.group(2)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        off2loc[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(page)))
h, data = None, []
for r in rows:
    if r and r[0] == "Address":
        h = r
        continue
    if h and r and r[0] != "Kernel Name":
        data.append(r)
ia, iex, iss = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
num = lambda v: int(v) if v and v.isdigit() else 0   # noqa: E731
base = int(data[0][ia], 16)
ex, ss = collections.Counter(), collections.Counter()
for r in data:
    loc = off2loc.get(int(r[ia], 16) - base, "?")
    ex[loc] += num(r[iex])
    ss[loc] += num(r[iss])
print(f"instructions per element {sum(ex.values()) * 32 / n:.2f}")
print("instr/elem  stall-samples  file:line")
for k, v in sorted(ex.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v * 32 / n:9.2f}  {ss[k]:13d}  {k}")
