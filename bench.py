#!/usr/bin/env python
"""Benchmark of the B200 block-regression compressor hot path (SZ3, arxiv 2111.02925).

Metric (BASELINE.json): regression compress & decompress GB/s per GPU and at N GPUs, % of HBM roofline.
Workload: config c5 -- 1024 x 2048 x 2048 fp32 (16 GiB) k^-3 Gaussian random field (seed 4), eb = 1e-3 x
value range, R = 32768, 6^3 blocks, sharded as block-aligned slabs over the N GPUs (strong scaling).

One step = the whole hot path over the field.  Default (--path two-pass): analyze = a0 value range + a2-a3
block coefficients in one read of x (+ MAX all-reduce of the range when N > 1), quantize = a4-a7 from those
coefficients (+ SUM all-reduce of the histogram when N > 1), a8 decompress + outlier scatter.  --path fused:
value range, then the single-pass a1-a7 kernel.
value = input bytes of the whole field / step time (max over ranks), i.e. round-trip GB/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sz3g|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU, NCCL)

Prints ONE JSON line on rank 0.  Inputs (16 GiB) are larger than the 126 MB L2, so no flush is needed
between steps.  `--impl reference` times the CPU oracle (oracle/, the test checker) on a bounded sample
of the same workload: the only other place bench.py runs oracle/ is the cpu_baseline leg.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NOMINAL_HBM_GBS = 8000.0   # B200 nominal HBM3e bandwidth (north_star's ~8 TB/s): the second denominator of SURVEY 8(d)
METRIC = "regression compress & decompress GB/s per GPU and 8-GPU, % of HBM roofline"
UNIT = "GB/s"
CONFIG = "c5"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="sz3g", choices=["sz3g", "reference"])
    ap.add_argument("--config", default=CONFIG)
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-planes", type=int, default=24)
    ap.add_argument("--no-huffman", action="store_true", help="skip the encoder-stage (NEXT-1) measurement")
    ap.add_argument("--huffman-reps", type=int, default=5)
    ap.add_argument("--no-truncation", action="store_true", help="skip the SZ3-Truncation (NEXT-2) measurement")
    ap.add_argument("--trunc-k", type=int, default=2)
    ap.add_argument("--no-lr", action="store_true", help="skip the SZ3-LR (NEXT-4) measurement")
    ap.add_argument("--path", default="two-pass", choices=["two-pass", "fused"],
                    help="REL compression: analyze (range + beta) -> quantize, or value_range -> fused compress")
    return ap.parse_args()


# ----------------------------------------------------------------------------------------- helpers
def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def profiled_traffic(kernel: str, config: str):
    """DRAM bytes per launch of `kernel` from the committed ncu capture summary, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(f"{config}:{kernel}")


REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int, period_ms: int = 50):
        self.index, self.period_ms = index, period_ms
        self.proc, self.lines, self.thread = None, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
                bits = int(parts[2], 16)
            except ValueError:
                continue
            for b, n in REASON_BITS.items():
                if bits & b:
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def max_over_ranks(v: float, world: int) -> float:
    import torch
    import torch.distributed as dist
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def make_slab(cfg, world, rank):
    """Generate the global field on this GPU (deterministic: seed 4) and keep this rank's slab."""
    import torch
    from paper_2111_02925_b200.dist import slab_bounds
    from synth import make_field
    full = make_field(cfg, device="cuda")
    a, b = slab_bounds(cfg.shape[0], world, rank)
    x = full[a:b].clone()
    del full
    torch.cuda.empty_cache()
    return x, a


# ----------------------------------------------------------------------------------------- CPU oracle
def oracle_round_trip(xs_np, cfg, lo, hi, dim0_offset):
    import oracle
    t0 = time.perf_counter()
    c = oracle.compress(xs_np, cfg.eb, cfg.eb_mode, radius=cfg.radius, dim0_offset=dim0_offset,
                        value_range_override=(lo, hi))
    oracle.decompress(c)
    return time.perf_counter() - t0


def run_reference(args):
    """--impl reference: the CPU oracle (oracle/, plain single-threaded C++) timed on the host, on a
    bounded sample of the workload (one 6-plane block row of the c5 field, with the global range)."""
    import numpy as np
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth import config_by_name, make_field
    cfg = config_by_name(args.config)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    shape = cfg.shape if dev == "cuda" else (48, 256, 256)
    full = make_field(cfg, device=dev, shape=shape)
    lo, hi = float(full.min()), float(full.max())
    a = (shape[0] // 12) * 6
    xs = full[a:a + 6].cpu().numpy()
    del full
    sample_bytes = xs.nbytes
    import oracle
    oracle.build()
    for _ in range(args.warmup):
        oracle_round_trip(xs, cfg, lo, hi, a)
    times = [oracle_round_trip(xs, cfg, lo, hi, a) for _ in range(args.steps)]
    t = sum(times)
    value = sample_bytes * args.steps / t / 1e9
    sample = f"planes [{a},{a + 6}) of {cfg.name} {shape} (one block row, {xs.size} elements, global range)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 (f32 data)",
            "data": "synthetic", "config": {"workload": f"{cfg.name}: {cfg.desc}", "shape": list(shape),
                                            "eb_rel": cfg.eb, "radius": cfg.radius, "block": 6},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------- encoder stage
def huffman_leg(sz3g, bufs, res, N_local, NB_local, s, args, world, peaks, stream):
    """NEXT-1 measured on this rank's codes with the merged histogram: codebook (1 CTA), encode,
    decode, timed with CUDA events (median of --huffman-reps), decode checked against the codes."""
    import torch
    codes = bufs.codes.view(-1)
    n = codes.numel()
    table = sz3g.huffman_codebook(bufs.hist).check()
    hs = sz3g.huffman_encode(codes, table).check()
    out = torch.empty_like(codes)
    sz3g.huffman_decode(hs, table, out=out)
    torch.cuda.synchronize()
    if int(hs.status.item()) or not torch.equal(out, codes):
        raise RuntimeError("Huffman round trip failed")
    ev = lambda: torch.cuda.Event(enable_timing=True)   # noqa: E731
    t_cb, t_en, t_de = [], [], []
    for _ in range(args.huffman_reps):
        e = [ev() for _ in range(4)]
        e[0].record(stream)
        table = sz3g.huffman_codebook(bufs.hist)
        e[1].record(stream)
        sz3g.huffman_encode(codes, table, payload=hs.payload, offsets=hs.offsets, scratch=hs._scratch)
        e[2].record(stream)
        sz3g.huffman_decode(hs, table, out=out)
        e[3].record(stream)
        torch.cuda.synchronize()
        t_cb.append(e[0].elapsed_time(e[1]))
        t_en.append(e[1].elapsed_time(e[2]))
        t_de.append(e[2].elapsed_time(e[3]))
    med = lambda v: sorted(v)[len(v) // 2]   # noqa: E731
    cb_ms = max_over_ranks(med(t_cb), world)
    en_ms = max_over_ranks(med(t_en), world)
    de_ms = max_over_ranks(med(t_de), world)
    words = hs.words()
    nch = hs.offsets.numel() - 1
    pay_b = 4 * words
    # algorithmic bytes: encode reads the codes once, writes payload + chunk offsets;
    # decode reads payload + offsets, writes the codes
    enc_bytes = 2 * n + pay_b + 8 * (nch + 1)
    dec_bytes = pay_b + 8 * (nch + 1) + 2 * n
    n_out = res.n_outliers
    cstream = sz3g.encode_coefficients(bufs.coef_codes)
    coef_b = cstream.nbytes()
    stored = pay_b + 8 * (nch + 1) + coef_b + (8 + s) * n_out + table.stored_bytes()
    return {
        "bits_per_code": 8 * pay_b / n, "payload_bytes": pay_b, "chunk": hs.chunk, "max_len": table.max_len,
        "compression_ratio": N_local * s / stored,
        "coefficient_bytes": coef_b, "coefficient_bytes_raw": 16 * NB_local,
        "ratio_note": "input bytes / (payload + chunk offsets + delta+Huffman-coded coefficient codes + outliers + "
                      "canonical codebook)",
        "codebook_ms": cb_ms, "encode_ms": en_ms, "decode_ms": de_ms,
        "encode_gbs_input": N_local * s / (en_ms * 1e-3) / 1e9,
        "encode_roofline": {"achieved": enc_bytes / (en_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                            "frac": enc_bytes / (en_ms * 1e-3) / 1e9 / peaks["hbm_gbs"], "alg_bytes": enc_bytes},
        "decode_roofline": {"achieved": dec_bytes / (de_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                            "frac": dec_bytes / (de_ms * 1e-3) / 1e9 / peaks["hbm_gbs"], "alg_bytes": dec_bytes},
    }


def truncation_leg(sz3g, x, out, args, world, peaks, stream):
    """NEXT-2: keep k most-significant bytes per value, timed with CUDA events (median of 5),
    reconstruction checked against the zero-filled definition on a sample."""
    import torch
    k, n, s = args.trunc_k, x.numel(), x.element_size()
    xf = x.view(-1)
    b = sz3g.truncation_compress(xf, k)
    y = out.view(-1)
    sz3g.truncation_decompress(b, n, k, x.dtype, out=y)
    torch.cuda.synchronize()
    mask = -(1 << (8 * (s - k))) if s == 4 else None
    if s == 4:   # spot check: y == x with the low bytes cleared
        xi = xf[:1 << 20].view(torch.int32)
        if not torch.equal(y[:1 << 20].view(torch.int32), xi & mask):
            raise RuntimeError("truncation round trip failed")
    tc, td = [], []
    for _ in range(5):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        sz3g.truncation_compress(xf, k, out=b)
        e[1].record(stream)
        sz3g.truncation_decompress(b, n, k, x.dtype, out=y)
        e[2].record(stream)
        torch.cuda.synchronize()
        tc.append(e[0].elapsed_time(e[1]))
        td.append(e[1].elapsed_time(e[2]))
    c_ms = max_over_ranks(sorted(tc)[2], world)
    d_ms = max_over_ranks(sorted(td)[2], world)
    nb = n * (s + k)   # algorithmic bytes of either direction
    return {"k": k, "compression_ratio": s / k, "compress_ms": c_ms, "decompress_ms": d_ms,
            "compress_gbs_input": n * s / (c_ms * 1e-3) / 1e9,
            "compress_roofline": {"achieved": nb / (c_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                                  "frac": nb / (c_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]},
            "decompress_roofline": {"achieved": nb / (d_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                                    "frac": nb / (d_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]}}


def lr_leg(sz3g, x, out, bufs, cfg, a0, N_local, NB_local, s, args, world, peaks, stream):
    """NEXT-4: SZ3-LR on the same field, from the analyze pass's range and beta (bufs.minmax /
    bufs.beta of the timed steps): lr_quantize and lr_decompress timed with CUDA events (median of 3),
    the reconstruction checked against the bound, the codes Huffman-coded for the ratio (not timed)."""
    import torch
    ev = lambda: torch.cuda.Event(enable_timing=True)   # noqa: E731
    if bufs.beta is None:   # the fused path ran no analyze pass: the range stays the timed steps'
        sz3g.regression_analyze(x, torch.empty_like(bufs.minmax), bufs.beta_buffer(), stream)
    tq, td = [], []
    for _ in range(3):
        e = [ev() for _ in range(3)]
        e[0].record(stream)
        res = sz3g.lr_quantize(x, cfg.eb, cfg.eb_mode, cfg.radius, bufs.minmax, bufs.beta, bufs, dim0_offset=a0,
                               stream=stream)
        e[1].record(stream)
        sz3g.lr_decompress(res.codes, res.coef_codes, res.lr_flags, res.outlier_idx, res.outlier_val,
                           res.outlier_idx.numel(), cfg.eb, cfg.radius, x.dtype, a0, out, stream=stream,
                           d_outlier_count=res.outlier_count, eb_mode=cfg.eb_mode, d_minmax=bufs.minmax)
        e[2].record(stream)
        torch.cuda.synchronize()
        tq.append(e[0].elapsed_time(e[1]))
        td.append(e[1].elapsed_time(e[2]))
    res.finalize()
    q_ms = max_over_ranks(sorted(tq)[1], world)
    d_ms = max_over_ranks(sorted(td)[1], world)
    st = sz3g.error_stats(x, out, res.eb_abs).cpu().tolist()
    if st[2] != 0 or not st[0] <= res.eb_abs:
        raise RuntimeError(f"SZ3-LR error bound violated: {st}")
    n_out = res.n_outliers
    nl = int(res.lr_flags.sum())
    table = sz3g.huffman_codebook(res.hist).check()
    hs = sz3g.huffman_encode(bufs.codes.view(-1), table).check()
    pay_b = 4 * hs.words()
    coef_b = sz3g.encode_coefficients(bufs.coef_codes).nbytes()
    stored = pay_b + 8 * hs.offsets.numel() + coef_b + (NB_local + 7) // 8 + (8 + s) * n_out + table.stored_bytes()
    # algorithmic bytes: quantize reads x and beta, writes codes, coefficient codes, flags,
    # outliers; decompress reads codes, coefficient codes, flags, outliers, writes x'
    q_bytes = N_local * (s + 2) + NB_local * (32 + 16 + 1) + n_out * (8 + s)
    d_bytes = N_local * (2 + s) + NB_local * (16 + 1) + n_out * (8 + s)
    lo, hi = (float(v) for v in bufs.minmax.cpu())
    return {"lorenzo_blocks": nl, "blocks": NB_local, "lorenzo_fraction": nl / max(1, NB_local),
            "bits_per_code": 8 * pay_b / N_local, "compression_ratio": N_local * s / stored,
            "psnr_db": sz3g.psnr(hi - lo, st[1] / N_local), "max_abs_err": st[0], "outliers": n_out,
            "quantize_ms": q_ms, "decompress_ms": d_ms,
            "quantize_roofline": {"achieved": q_bytes / (q_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                                  "frac": q_bytes / (q_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]},
            "decompress_roofline": {"achieved": d_bytes / (d_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                                    "frac": d_bytes / (d_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]},
            "note": "compression = analyze pass (shared with the regression path) + lr_quantize; ratio counts the "
                    "predictor flags as a bitmap (1 bit per block)"}


# ----------------------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    from paper_2111_02925_b200 import dist as pdist
    from paper_2111_02925_b200 import sz3g
    from synth import config_by_name

    world, rank, local = dist_setup(args)
    cfg = config_by_name(args.config)
    sz3g.load()
    x, a0 = make_slab(cfg, world, rank)
    N_local, N_global = x.numel(), math.prod(cfg.shape)
    s = x.element_size()
    NB_local = sz3g.num_blocks(x.shape)
    cap = max(1 << 20, N_local // 256)
    bufs = sz3g.CompressBuffers(x.shape, x.dtype, cfg.radius, outlier_cap=cap, device=x.device)
    out = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    ev = {}

    two_pass = args.path == "two-pass"
    beta = bufs.beta_buffer() if two_pass else None

    def step(record=None):
        if record is not None:
            record[4].record(stream)
        if two_pass:
            sz3g.regression_analyze(x, bufs.minmax, beta)
        else:
            sz3g.value_range(x, bufs.minmax)
        if record is not None:
            record[5].record(stream)
        pdist.allreduce_range_(bufs.minmax)
        bufs.reset()
        if record is not None:
            record[0].record(stream)
        if two_pass:
            sz3g.regression_quantize(x, cfg.eb, cfg.eb_mode, cfg.radius, bufs.minmax, beta, bufs=bufs, reset=False,
                                     dim0_offset=a0)
        else:
            sz3g.regression_compress(x, cfg.eb, cfg.eb_mode, cfg.radius, d_minmax=bufs.minmax, bufs=bufs,
                                     reset=False, dim0_offset=a0)
        if record is not None:
            record[1].record(stream)
        pdist.allreduce_hist_(bufs.hist)
        if record is not None:
            record[2].record(stream)
        sz3g.regression_decompress(bufs.codes, bufs.coef_codes, bufs.outlier_idx, bufs.outlier_val, cap, cfg.eb,
                                   cfg.radius, x.dtype, dim0_offset=a0, out=out, d_outlier_count=bufs.outlier_count,
                                   eb_mode=cfg.eb_mode, d_minmax=bufs.minmax)
        if record is not None:
            record[3].record(stream)

    for _ in range(args.warmup):
        step()
    barrier(world)
    recs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = sz3g.launch_count()
    with ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ else local) as clk:
        barrier(world)
        t_start.record(stream)
        for k in range(args.steps):
            step(recs[k])
        t_end.record(stream)
        barrier(world)
    launches = sz3g.launch_count() - l0
    ms_total = max_over_ranks(t_start.elapsed_time(t_end), world)
    ms_step = ms_total / args.steps
    comp_ms = sum(r[0].elapsed_time(r[1]) for r in recs) / args.steps
    dec_ms = sum(r[2].elapsed_time(r[3]) for r in recs) / args.steps
    ana_ms = sum(r[4].elapsed_time(r[5]) for r in recs) / args.steps
    comp_ms_max = max_over_ranks(comp_ms, world)
    dec_ms_max = max_over_ranks(dec_ms, world)

    res = sz3g.Compressed(tuple(x.shape), x.dtype, cfg.radius, a0, bufs.codes, bufs.coef_codes, None, bufs.outlier_idx,
                          bufs.outlier_val, bufs.outlier_count, bufs.hist, bufs.eb_abs, bufs.status).finalize()
    n_out = res.n_outliers
    # algorithmic bytes per launch: compress reads x, writes codes, coefficient codes, outliers
    # (two-pass quantize also reads the analyze pass's beta, 32 B per block); analyze reads x, writes beta
    comp_bytes = N_local * (s + 2) + NB_local * 16 + n_out * (8 + s) + (NB_local * 32 if two_pass else 0)
    ana_bytes = N_local * s + (NB_local * 32 if two_pass else 0)
    dec_bytes = N_local * (2 + s) + NB_local * 16 + n_out * (8 + s)
    peaks = measured_peaks()
    comp_gbs = comp_bytes / (comp_ms * 1e-3) / 1e9
    value = N_global * s / (ms_step * 1e-3) / 1e9

    # ---------------- reconstruction quality (NEXT-3 metrics): bound check, max error, PSNR
    st = sz3g.error_stats(x, out, res.eb_abs).cpu().tolist()
    lo, hi = (float(v) for v in bufs.minmax.cpu())
    quality = {"max_abs_err": st[0], "eb_abs": res.eb_abs, "above_eb": int(st[2]),
               "psnr_db": sz3g.psnr(hi - lo, st[1] / N_local)}
    if st[2] != 0 or not st[0] <= res.eb_abs:
        raise RuntimeError(f"error bound violated: {quality}")

    # ---------------- encoder stage (NEXT-1): codebook from the merged histogram, encode, decode
    huff = None
    if not args.no_huffman:
        huff = huffman_leg(sz3g, bufs, res, N_local, NB_local, s, args, world, peaks, stream)
        quality["bit_rate"] = sz3g.bit_rate(8 * s, huff["compression_ratio"])
        quality["compression_ratio"] = huff["compression_ratio"]

    # ---------------- SZ3-Truncation (NEXT-2) on the same field
    trunc = None
    if not args.no_truncation:
        trunc = truncation_leg(sz3g, x, out, args, world, peaks, stream)

    # ---------------- SZ3-LR (NEXT-4) on the same field (reuses bufs: runs after the other legs)
    lr = None
    if not args.no_lr:
        lr = lr_leg(sz3g, x, out, bufs, cfg, a0, N_local, NB_local, s, args, world, peaks, stream)

    # ---------------- CPU oracle beside it (rank 0, N = 1 only; bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        lo, hi = (float(v) for v in bufs.minmax.cpu())
        p = min(args.cpu_sample_planes, x.shape[0] - 504)
        xs = x[504:504 + p].cpu().numpy()
        t = oracle_round_trip(xs, cfg, lo, hi, 504)
        cpu = {"value": xs.nbytes / t / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"planes [504,{504 + p}) of {cfg.name} ({xs.size} elements, global range), "
                         f"compress + decompress, one host core, {t:.1f} s"}

    # ---------------- end to end through the public API with HOST buffers (pinned), copies timed:
    # paper_2111_02925_b200.pipeline.PipelinedCodec round-trips a sequence of fields from pinned host
    # memory (here: the same field, e2e_steps times) -- host->device copy, analyze, quantise, Huffman
    # coding of codes and coefficients, decompression, device->host copy of the compressed stream and of
    # x' -- with consecutive fields' copies overlapped on the two copy engines.
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        from paper_2111_02925_b200.pipeline import PipelinedCodec
        del bufs
        torch.cuda.empty_cache()
        h_x = torch.empty_like(x, device="cpu").pin_memory()
        h_x.copy_(x)
        h_out = torch.empty_like(x, device="cpu").pin_memory()
        codec = PipelinedCodec(tuple(x.shape), x.dtype, cfg.eb, cfg.eb_mode, cfg.radius, device=x.device,
                               dim0_offset=a0)
        del x, out
        torch.cuda.empty_cache()
        codec.run([h_x], h_out)                      # warm-up (one field)
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(codec.s_in)
        results = codec.run([h_x] * args.e2e_steps, h_out)
        e1.record(codec.s_out)
        barrier(world)
        e1.synchronize()
        e_ms = max_over_ranks(e0.elapsed_time(e1), world) / args.e2e_steps
        bi = h_x.numel() * s
        bo = int(sum(r.nbytes() for r in results) / len(results)) + h_out.numel() * s
        e2e = {"value": N_global * s / (e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": bi,
               "d2h_bytes_per_step": bo, "ms_per_step": e_ms, "fields": args.e2e_steps,
               "note": "PipelinedCodec: pinned host field -> device, analyze + quantise + Huffman (codes, "
                       "coefficients) + decompress, compressed stream + x' -> pinned host; copies of consecutive "
                       "fields overlapped (3 streams, double-buffered)"}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 data, f64 arithmetic", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.desc}", "shape": list(cfg.shape), "eb_rel": cfg.eb,
                       "radius": cfg.radius, "block": 6, "parallelism": f"slabs{world}",
                       "l2": "inputs (16 GiB) larger than L2; no flush"},
            "roofline": {"bound": "hbm", "kernel": "k_compress_tma" + ("<beta in>" if two_pass else ""),
                         "achieved": comp_gbs, "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": comp_gbs / peaks["hbm_gbs"],
                         "traffic": profiled_traffic("k_compress_tma" + ("_beta" if two_pass else ""), cfg.name),
                         "peak_source": peaks["source"],
                         "frac_nominal": comp_gbs / NOMINAL_HBM_GBS, "peak_nominal": NOMINAL_HBM_GBS,
                         "alg_bytes_per_launch": comp_bytes, "ms_per_launch": comp_ms},
            "compress_gbs": N_global * s / (comp_ms_max * 1e-3) / 1e9,
            "decompress_gbs": N_global * s / (dec_ms_max * 1e-3) / 1e9,
            "decompress_roofline": {"achieved": dec_bytes / (dec_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                                    "frac": dec_bytes / (dec_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                                    "frac_nominal": dec_bytes / (dec_ms * 1e-3) / 1e9 / NOMINAL_HBM_GBS,
                                    "ms_per_launch": dec_ms},
            "analyze_roofline": {"kernel": "k_analyze_tma" if two_pass else "k_value_range",
                                 "achieved": ana_bytes / (ana_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                                 "frac": ana_bytes / (ana_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                                 "frac_nominal": ana_bytes / (ana_ms * 1e-3) / 1e9 / NOMINAL_HBM_GBS,
                                 "ms_per_step": ana_ms},
            "path": args.path,
            "quality": quality, "huffman": huff, "truncation": trunc, "lr": lr,
            "outliers": n_out, "eb_abs": res.eb_abs,
            "clocks": clocks, "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
