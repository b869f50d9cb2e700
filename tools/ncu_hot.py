"""Top SASS lines of an ncu source page CSV by one stall reason (default long_sb), with 3 lines of
context: python tools/ncu_hot.py page.csv [stall_name] [n]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
key = "stall_" + (sys.argv[2] if len(sys.argv) > 2 else "long_sb")
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 10
h, data = None, []
for r in rows:
    if r and r[0] == 'Address':
        h = r
        continue
    if r and r[0] == 'Kernel Name' and data:
        break
    if h and r:
        data.append(r)
li, isrc = h.index(key), h.index('Source')
n = lambda v: int(v) if v and v.isdigit() else 0   # noqa: E731
tot = sum(n(r[li]) for r in data)
print(key, "total samples", tot)
for i in sorted(range(len(data)), key=lambda i: -n(data[i][li]))[:ntop]:
    print(f"{i:5d} {n(data[i][li]):6d}  {data[i][isrc][:90]}")
    for j in range(max(0, i - 3), i):
        print("            ", data[j][isrc][:90])
