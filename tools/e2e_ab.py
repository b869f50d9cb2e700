"""e2e A/B: the PipelinedCodec of round 1 (tools/_pipeline_r01.py) against the current one on c5,
alternating, same box.  Prints ms per field for each."""
import importlib.util
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2111_02925_b200 import sz3g  # noqa: E402
from paper_2111_02925_b200 import pipeline as cur  # noqa: E402
from synth import config_by_name, make_field  # noqa: E402

spec = importlib.util.spec_from_file_location("p_old", os.path.join(ROOT, "tools", "_pipeline_r01.py"))
old = importlib.util.module_from_spec(spec)
sys.modules["p_old"] = old
spec.loader.exec_module(old)
cfg = config_by_name("c5")
sz3g.load()
x = make_field(cfg, device="cuda")
h_x = torch.empty_like(x, device="cpu").pin_memory()
h_x.copy_(x)
h_out = torch.empty_like(x, device="cpu").pin_memory()
del x
torch.cuda.empty_cache()
res = {}
for rnd in range(2):
    for name, mod in (("r01", old), ("cur", cur)):
        codec = mod.PipelinedCodec(tuple(h_x.shape), h_x.dtype, cfg.eb, cfg.eb_mode, cfg.radius)
        codec.run([h_x, h_x], h_out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(codec.s_in)
        codec.run([h_x] * 6, h_out)
        e1.record(codec.s_out)
        e1.synchronize()
        res.setdefault(name, []).append(e0.elapsed_time(e1) / 6)
        print(name, rnd, res[name][-1], flush=True)
        del codec
        torch.cuda.empty_cache()
print(json.dumps(res))
