import sys, json, torch
sys.path.insert(0, '.')
import bench
from paper_2111_02925_b200 import sz3g
peaks = bench.measured_peaks()
fb = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for spec in ["c3", "c4", "c2"]:
    o = bench.config_leg(sz3g, spec, peaks, 10, 3, fb)
    print(spec, json.dumps({k: o[k] for k in ("analyze_roofline", "quantize_roofline", "decompress_roofline", "stream_ceiling")}))
