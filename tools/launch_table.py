"""ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv log -> the
launch table kept under profiles/ (kernel | us | DRAM read GB | DRAM write GB), libsz3g kernels only.
  python tools/launch_table.py gpurun_out/launch.csv "# header line" > profiles/rNN_launches.txt"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
launches = {}
order = []
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h is None or len(r) != len(h):
        continue
    d = dict(zip(h, r))
    key = d["ID"]
    if key not in launches:
        launches[key] = {"name": d["Kernel Name"]}
        order.append(key)
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    m = d["Metric Name"]
    if m == "gpu__time_duration.sum":
        launches[key]["us"] = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                                   "msecond": 1e3}.get(unit, 1.0)
    else:
        scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}.get(unit, 1e-9)
        launches[key][m] = v * scale
for line in sys.argv[2:]:
    print(line)
print("# kernel | gpu__time_duration.sum (us) | dram read GB | dram write GB")
for k in order:
    d = launches[k]
    name = d["name"]
    if not re.search(r"k_[a-z]", name) or "at::" in name:
        continue
    name = re.sub(r"^(void )?<unnamed>::", "", name)
    name = re.sub(r"\(.*$", "", name)
    print(f"{name[:52]:52s} {d.get('us', 0):9.1f} {d.get('dram__bytes_read.sum', 0):8.3f} {d.get('dram__bytes_write.sum', 0):8.3f}")
