#!/usr/bin/env python
"""Kernel tuning sweep (GPU): generate one workload once, then time the compress / decompress kernels
under each tuning setting (sz3g_set_tuning) with CUDA events.  Tuning knobs never change a result;
the codes of every setting are compared with the first one as a sanity check.

  python tools/tune.py --config c5 --reps 10 "WAIT=0,PWAIT=0" "WAIT=1,PWAIT=1" ...
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=2, help="passes over the settings (interleaved)")
    ap.add_argument("--path", default="fused", choices=["fused", "two-pass"])
    ap.add_argument("--flush", action="store_true", help="write 256 MB before every timed launch (evict L2)")
    ap.add_argument("--graphs", action="store_true", help="replay each timed call from a CUDA graph (no host gaps)")
    ap.add_argument("settings", nargs="+")
    args = ap.parse_args()
    import torch
    from paper_2111_02925_b200 import sz3g
    from synth import config_by_name, make_field
    torch.cuda.set_device(0)
    cfg = config_by_name(args.config)
    sz3g.load()
    x = make_field(cfg, device="cuda")
    cap = max(1 << 20, x.numel() // 256)
    bufs = sz3g.CompressBuffers(x.shape, x.dtype, cfg.radius, outlier_cap=cap, device=x.device)
    out = torch.empty_like(x)
    sz3g.value_range(x, bufs.minmax)
    stream = torch.cuda.current_stream()

    beta = None
    if args.path == "two-pass":
        _, beta = sz3g.regression_analyze(x, bufs.minmax, bufs.beta_buffer())

    def comp():
        bufs.reset()
        if beta is not None:
            sz3g.regression_quantize(x, cfg.eb, cfg.eb_mode, cfg.radius, bufs.minmax, beta, bufs=bufs, reset=False)
        else:
            sz3g.regression_compress(x, cfg.eb, cfg.eb_mode, cfg.radius, d_minmax=bufs.minmax, bufs=bufs,
                                     reset=False)

    def dec():
        sz3g.regression_decompress(bufs.codes, bufs.coef_codes, bufs.outlier_idx, bufs.outlier_val, cap, cfg.eb,
                                   cfg.radius, x.dtype, out=out, d_outlier_count=bufs.outlier_count,
                                   eb_mode=cfg.eb_mode, d_minmax=bufs.minmax)

    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if args.flush else None

    def ana():
        sz3g.regression_analyze(x, bufs.minmax, bufs.beta_buffer())

    def timeit(fn):
        for _ in range(2):
            fn()
        if args.graphs:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn_ = fn
                fn_()
            fn = g.replay
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
        for a, b in evs:
            bufs.reset()
            if flush_buf is not None:
                flush_buf.fill_(1)
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        ts = sorted(a.elapsed_time(b) for a, b in evs)
        return ts[len(ts) // 2]

    ref_codes = None
    res = {}
    for rnd in range(args.rounds):
        for st in args.settings:
            kv = dict(p.split("=") for p in st.split(",") if p)
            for k, v in kv.items():
                try:
                    sz3g.set_tuning(k, int(v))
                except Exception as e:   # older A/B builds: defaults only
                    print("set_tuning skipped:", e, file=sys.stderr)
            tc = timeit(comp)
            comp()
            torch.cuda.synchronize()
            h = int(bufs.codes.view(torch.int16).to(torch.int64).sum())
            if ref_codes is None:
                ref_codes = h
            td = timeit(dec)
            ta = timeit(ana) if beta is not None else 0.0
            res.setdefault(st, []).append((tc, td, h == ref_codes, ta))
            # restore defaults for keys not in the next setting: every setting lists its keys explicitly
    for st, v in res.items():
        print(json.dumps({"setting": st, "compress_ms": [round(a, 4) for a, _, _, _ in v],
                          "decompress_ms": [round(b, 4) for _, b, _, _ in v],
                          "analyze_ms": [round(t, 4) for *_, t in v], "codes_match": all(c for _, _, c, _ in v)}))


if __name__ == "__main__":
    main()
