"""Quick throughput probe of the kernels (CUDA events, L2-flushed); not the bench contract."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_02925_b200 import sz3g
from synth import make_field, config_by_name

def tm(fn, reps=10, flush=None):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    fn(); torch.cuda.synchronize()
    ts = []
    for a, b in ev:
        if flush is not None: flush.zero_()
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[reps // 2]

names = sys.argv[1:] or ["c2", "c3", "c4"]
flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
for name in names:
    cfg = config_by_name(name)
    x = make_field(cfg, device="cuda")
    N = x.numel(); s = x.element_size()
    for flags in (0, 1):
        bufs = sz3g.CompressBuffers(x.shape, x.dtype, cfg.radius, device=x.device)
        mm = sz3g.value_range(x)
        t_r = tm(lambda: sz3g.value_range(x, bufs.minmax), flush=flush)
        def comp():
            bufs.reset()
            sz3g.regression_compress(x, cfg.eb, cfg.eb_mode, cfg.radius, d_minmax=mm, bufs=bufs, reset=False, flags=flags)
        t_c = tm(comp, flush=flush)
        res = sz3g.regression_compress(x, cfg.eb, cfg.eb_mode, cfg.radius, d_minmax=mm, bufs=bufs, flags=flags).finalize()
        out = torch.empty_like(x)
        t_d = tm(lambda: sz3g.regression_decompress(res.codes, res.coef_codes, res.outlier_idx, res.outlier_val, res.n_outliers, res.eb_abs, res.radius, x.dtype, out=out, flags=flags), flush=flush)
        cb = N * (s + 2) + 16 * sz3g.num_blocks(x.shape)
        print(f"{name} flags={flags} N={N} range {t_r:.3f} ms ({N*s/t_r/1e6:.0f} GB/s) | compress {t_c:.3f} ms "
              f"in {N*s/t_c/1e6:.0f} GB/s alg {cb/t_c/1e6:.0f} GB/s | decompress {t_d:.3f} ms alg {cb/t_d/1e6:.0f} GB/s | outliers {res.n_outliers}", flush=True)
