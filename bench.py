#!/usr/bin/env python
"""Benchmark of the B200 block-regression compressor hot path (SZ3, arxiv 2111.02925).

Metric (BASELINE.json): regression compress & decompress GB/s per GPU and at N GPUs, % of HBM roofline.
Workload: config c5 -- 1024 x 2048 x 2048 fp32 (16 GiB) k^-3 Gaussian random field (seed 4), eb = 1e-3 x
value range, R = 32768, 6^3 blocks, sharded as block-aligned slabs over the N GPUs (strong scaling).

One step = the whole hot path over the field, ``RoundTrip.step`` (paper_2111_02925_b200/roundtrip.py, the
object tests/test_gpu_c5.py checks against the oracle).  Default (--path two-pass): analyze = a0 value
range + a2-a3 block coefficients in one read of x (+ MAX all-reduce of the range when N > 1), quantize =
a4-a7 from those coefficients (+ SUM all-reduce of the histogram when N > 1), a8 decompress + outlier
scatter.  --path fused: value range, then the single-pass a1-a7 kernel.
value = input bytes of the whole field / step time (max over ranks), i.e. round-trip GB/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sz3g|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU, NCCL)
  torchrun --nproc-per-node 2 bench.py --gpus 2 --dist-backend gloo --shape 96,2048,2048 ...
                                                            (multi-rank rehearsal on ONE GPU, gloo)

Prints ONE JSON line on rank 0.  c5's inputs (16 GiB) are larger than the 126 MB L2, so no flush is
needed between its steps; the per-config legs (`configs`) flush L2 before every step.  `--impl
reference` times the CPU oracle (oracle/, the test checker) on a bounded sample of the same workload:
the only other place bench.py runs oracle/ is the cpu_baseline leg.
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
    ap.add_argument("--no-interp", action="store_true", help="skip the SZ3-Interp (NEXT-4) measurement")
    ap.add_argument("--path", default="two-pass", choices=["two-pass", "fused"],
                    help="REL compression: analyze (range + beta) -> quantize, or value_range -> fused compress")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend at N > 1 (gloo: rehearse the multi-rank path on one GPU)")
    ap.add_argument("--shape", default=None, help="n0,n1,n2: the config's recipe at another shape (rehearsals)")
    ap.add_argument("--configs", default="c2,c3,c4,c5r16,c3r4",
                    help="per-config legs after the main line (N = 1 only): config names, cNrR = config N at "
                         "radius R (stress variant); '' for none")
    ap.add_argument("--config-steps", type=int, default=10)
    ap.add_argument("--no-ties", action="store_true", help="skip the reported-counter pass (sz3g_tie_counts)")
    ap.add_argument("--graphs", default="auto", choices=["auto", "on", "off"],
                    help="replay the step from CUDA graphs (auto: at N = 1; NCCL collectives can be captured, gloo not)")
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
    """One process per GPU.  NCCL by default; gloo (CUDA tensors staged through the host) rehearses the
    same code path with every rank on one GPU (device = LOCAL_RANK mod the visible GPUs)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    return world, rank, dev


def max_over_ranks(v: float, world: int) -> float:
    import torch
    import torch.distributed as dist
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(v: int, world: int) -> int:
    import torch
    import torch.distributed as dist
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.int64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())


def host_cpu() -> dict:
    """Host CPU of this box (the cpu_baseline's machine): model name and logical cores."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def entropy_bits(hist) -> float:
    """Shannon entropy (bits per code) of the merged code histogram (zeroth-order, P:418's Huffman input)."""
    import numpy as np
    h = hist.cpu().numpy().astype(np.float64)
    n = h.sum()
    p = h[h > 0] / n
    return float(-(p * np.log2(p)).sum())


# The paper's own CPU numbers: context only -- other hardware, whole pipelines
PAPER_CONTEXT = {
    "hardware": "Bebop (ANL): 2x Intel Xeon E5-2695v4 Broadwell, 36 cores/node, 128 GB DDR4 (P:522); "
                "thread count not stated",
    "sz3_truncation_compress_gbs": 1.0,
    "second_best_compress_gbs": 0.25,
    "sz3_interp_compress_gbs": "> 0.1",
    "source": "P:891 (SZ3-Truncation 1 GB/s, 4x the second best = SZ2.1 / SZ3-LR-s, both containing the "
              "regression predictor; SZ3-Interp > 100 MB/s); the paper has no number for the regression "
              "path alone and no GPU results (P:900)",
}


def barrier(world):
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def make_slab(cfg, world, rank, shape):
    """Generate the global field (deterministic: the config's seed) and keep only this rank's
    block-aligned slab on its GPU (the generator needs the whole spectrum; the rest is freed)."""
    import torch
    from paper_2111_02925_b200.dist import slab_bounds
    from synth import make_field
    full = make_field(cfg, device="cuda", shape=shape)
    a, b = slab_bounds(shape[0], world, rank)
    x = full[a:b].clone()
    del full
    torch.cuda.empty_cache()
    return x, a


def flush_l2(buf):
    """Evict L2 (126 MB) by writing a buffer twice its size (SURVEY 8(d) "Flush L2")."""
    buf.fill_(1)


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
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             **host_cpu()},
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


def interp_leg(sz3g, x, out, minmax, cfg, N_local, s, args, world, peaks, stream):
    """NEXT-4 SZ3-Interp (DEFINITION.md I1-I6) on the same field with the timed steps' range:
    compress (level passes + histogram) and decompress timed with CUDA events (median of 3), the
    reconstruction checked against the bound, the codes Huffman-coded for the ratio (not timed).  Level
    passes cross every slab boundary, so at N > 1 every rank compresses its own slab as a separate field."""
    import torch
    ev = lambda: torch.cuda.Event(enable_timing=True)   # noqa: E731
    res = sz3g.interp_compress(x, cfg.eb, cfg.eb_mode, cfg.radius, d_minmax=minmax,
                               outlier_cap=max(1 << 20, N_local // 64), stream=stream)
    tc, td = [], []
    for _ in range(3):
        e = [ev() for _ in range(3)]
        e[0].record(stream)
        sz3g.interp_compress(x, cfg.eb, cfg.eb_mode, cfg.radius, d_minmax=minmax, out=res, stream=stream)
        e[1].record(stream)
        sz3g.interp_decompress(res.codes, res.outlier_idx, res.outlier_val, res.outlier_idx.numel(), cfg.eb,
                               cfg.radius, x.dtype, out=out, d_outlier_count=res.outlier_count, eb_mode=cfg.eb_mode,
                               d_minmax=minmax, stream=stream)
        e[2].record(stream)
        torch.cuda.synchronize()
        tc.append(e[0].elapsed_time(e[1]))
        td.append(e[1].elapsed_time(e[2]))
    res.finalize()
    c_ms = max_over_ranks(sorted(tc)[1], world)
    d_ms = max_over_ranks(sorted(td)[1], world)
    st = sz3g.error_stats(x, out, res.eb_abs).cpu().tolist()
    if st[2] != 0 or not st[0] <= res.eb_abs:
        raise RuntimeError(f"SZ3-Interp error bound violated: {st}")
    n_out = res.n_outliers
    table = sz3g.huffman_codebook(res.hist).check()
    hs = sz3g.huffman_encode(res.codes.view(-1), table).check()
    pay_b = 4 * hs.words()
    stored = pay_b + 8 * hs.offsets.numel() + (8 + s) * n_out + table.stored_bytes()
    # algorithmic bytes: compress reads x, writes codes and the reconstruction x' (its
    # working buffer); decompress reads codes, writes x'; the donors' re-reads are the method's own
    c_bytes = N_local * (s + 2 + s) + n_out * (8 + s)
    d_bytes = N_local * (2 + s) + n_out * (8 + s)
    lo, hi = (float(v) for v in minmax.cpu())
    del res, hs
    return {"outliers": n_out, "bits_per_code": 8 * pay_b / N_local, "compression_ratio": N_local * s / stored,
            "psnr_db": sz3g.psnr(hi - lo, st[1] / N_local), "max_abs_err": st[0],
            "compress_ms": c_ms, "decompress_ms": d_ms,
            "compress_roofline": {"achieved": c_bytes / (c_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                                  "frac": c_bytes / (c_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]},
            "decompress_roofline": {"achieved": d_bytes / (d_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                                    "frac": d_bytes / (d_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]},
            "note": "level-serial: one launch per pass (3 per level); compression = value range (shared) + passes "
                    "+ histogram"}


# ----------------------------------------------------------------------------------------- per-config legs
def alg_bytes(N, NB, s, n_out):
    """SURVEY 8(d) algorithmic bytes per launch of each kernel: the quantise kernel reads
    x and writes codes, coefficient codes (16 B / block) and outliers (index + value); the analyze
    kernel reads x (its 32 B / block of beta is the two-pass split's own traffic, reported apart);
    decompress reads codes, coefficient codes and outliers and writes x'."""
    return {"quantize": N * (s + 2) + 16 * NB + n_out * (8 + s), "analyze": N * s,
            "decompress": N * (2 + s) + 16 * NB + n_out * (8 + s), "beta": 32 * NB}


def roof(bytes_, ms, peak):
    gbs = bytes_ / (ms * 1e-3) / 1e9
    return {"achieved": gbs, "frac": gbs / peak, "frac_nominal": gbs / NOMINAL_HBM_GBS, "ms_per_launch": ms,
            "alg_bytes": bytes_}


def stream_ceilings(x, steps, flush_buf):
    """Size-matched ceilings for a per-config leg: plain torch streaming ops on the same field, each
    replayed from a CUDA graph after the same L2 flush -- a read of x (`torch.sum`, N s bytes: the
    analyze kernel's traffic) and an elementwise copy of x (`torch.neg`: N 2s bytes, the MEASURED_PEAKS.json recipe at this size, as an SM
    kernel -- `copy_` of a contiguous tensor may go to the copy engines:
    the ceiling quoted for quantise and decompress, whose 2:1 / 1:2 mixes torch has no plain streamer
    for -- its dtype casts run well below it at these sizes).  Fixed per-launch costs and ramp / tail
    at this size are in them as they are in the kernels: the part of the gap to MEASURED_PEAKS.json
    that no kernel closes."""
    import statistics
    import torch
    N, s = x.numel(), x.element_size()
    y = torch.empty_like(x)
    acc = torch.empty((), dtype=x.dtype, device=x.device)
    ops = {"read": ("torch.sum(x)", lambda: torch.sum(x.view(-1), 0, out=acc), N * s),
           "copy": ("torch.neg(x, out=y)", lambda: torch.neg(x, out=y), 2 * N * s)}
    out = {}
    stream = torch.cuda.Stream()   # graph capture needs a non-default stream
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        for k, (name, fn, nbytes) in ops.items():
            fn()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                fn()
            ts = []
            for _ in range(steps):
                flush_l2(flush_buf)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                g.replay()
                e1.record(stream)
                stream.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            out[k] = {"op": name, "ms": ms, "gbs": nbytes / (ms * 1e-3) / 1e9}
            del g
    del y
    return out


def config_leg(sz3g, spec, peaks, steps, warmup, flush_buf, x=None):
    """One per-config measurement: `spec` = config name, or cNrR = config N at radius R (labelled
    stress variant, SURVEY 8(d) point 3).  The same RoundTrip step as the main line (two-pass), L2
    flushed before every step, per-kernel CUDA events, §8(d) bytes, bound checked, counters reported."""
    import torch
    from paper_2111_02925_b200.roundtrip import RoundTrip, bench_outlier_cap
    from synth import config_by_name, make_field
    name, R = (spec.split("r")[0], int(spec.split("r")[1])) if "r" in spec else (spec, None)
    cfg = config_by_name(name)
    R = R or cfg.radius
    if x is None:
        x = make_field(cfg, device="cuda")
    N, s = x.numel(), x.element_size()
    NB = sz3g.num_blocks(x.shape)
    cap = bench_outlier_cap(N) if R >= 1024 else N
    rt = RoundTrip(x, cfg.eb, cfg.eb_mode, R, outlier_cap=cap)
    launch = "each segment of the step replayed from a CUDA graph (RoundTrip.capture)"
    try:
        rt.capture()   # CUDA graphs: no host gaps between the small configs' kernels
    except Exception as e:
        print(f"bench: CUDA graph capture failed for {spec} ({e}); eager", file=sys.stderr)
        torch.cuda.synchronize()
        rt.graphs = None
        launch = "eager (graph capture failed)"
    stream = rt.stream
    for _ in range(warmup):
        rt.step()
    recs = []
    timed = None
    try:   # the whole step as one graph with its timing events as graph nodes (no launch gaps)
        timed = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(6)]
        rt.capture_timed(timed)
        launch = "the whole step replayed from ONE CUDA graph, timing events as graph nodes"
    except Exception as e:
        print(f"bench: single-graph capture failed for {spec} ({e}); per-segment graphs", file=sys.stderr)
        torch.cuda.synchronize()
        timed = None
    spans = ((4, 5), (0, 1), (2, 3), (4, 3))   # analyze, quantise, decompress, step (event indices)
    for _ in range(steps):
        flush_l2(flush_buf)
        if timed is not None:
            rt.replay_timed()
            torch.cuda.synchronize()
            recs.append([timed[i].elapsed_time(timed[j]) for i, j in spans])
        else:
            r = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            rt.step(r)
            recs.append(r)
    torch.cuda.synchronize()
    if timed is None:
        recs = [[r[i].elapsed_time(r[j]) for i, j in spans] for r in recs]
    res = rt.result()
    ana, qua, dec, step = (sum(r[k] for r in recs) / steps for k in range(4))
    b = alg_bytes(N, NB, s, res.n_outliers)
    st = sz3g.error_stats(x, rt.out, res.eb_abs).cpu().tolist()
    if st[2] != 0 or not st[0] <= res.eb_abs:
        raise RuntimeError(f"{spec}: error bound violated {st}")
    ties = sz3g.tie_counts(x, cfg.eb, cfg.eb_mode, R, rt.bufs.minmax, res.coef_codes, rt.beta).cpu().tolist()
    out = {"shape": list(x.shape), "dtype": str(x.dtype).replace("torch.", ""), "eb_rel": cfg.eb, "radius": R,
           "stress_variant": R != cfg.radius, "outliers": res.n_outliers, "outlier_frac": res.n_outliers / N,
           "entropy_bits": entropy_bits(res.hist), "max_abs_err": st[0], "eb_abs": res.eb_abs,
           "ties": dict(zip(sz3g.TIE_COUNTER_NAMES, ties)),
           "compress_gbs": N * s / ((ana + qua) * 1e-3) / 1e9, "decompress_gbs": N * s / (dec * 1e-3) / 1e9,
           "round_trip_gbs": N * s / (step * 1e-3) / 1e9, "ms_per_step": step,
           "quantize_roofline": roof(b["quantize"], qua, peaks["hbm_gbs"]),
           "analyze_roofline": roof(b["analyze"], ana, peaks["hbm_gbs"]),
           "decompress_roofline": roof(b["decompress"], dec, peaks["hbm_gbs"]),
           "l2": "flushed (2x L2 write) before every step", "steps": steps, "warmup": warmup, "launch": launch}
    try:
        if N * s > (1 << 30):   # the c5-sized stress legs: the main line's peak applies
            raise RuntimeError("not measured above 1 GiB (MEASURED_PEAKS.json is the ceiling there)")
        ceil = stream_ceilings(x, max(steps, 5), flush_buf)
        for k, c in (("analyze", "read"), ("quantize", "copy"), ("decompress", "copy")):
            out[f"{k}_roofline"]["frac_of_stream"] = out[f"{k}_roofline"]["achieved"] / ceil[c]["gbs"]
        out["stream_ceiling"] = ceil
    except Exception as e:   # a measurement aid: never fail the leg on it
        out["stream_ceiling"] = {"error": str(e)[:200]}
    del rt
    torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    from paper_2111_02925_b200 import sz3g
    from paper_2111_02925_b200.roundtrip import RoundTrip
    from synth import config_by_name

    world, rank, dev = dist_setup(args)
    cfg = config_by_name(args.config)
    shape = tuple(int(v) for v in args.shape.split(",")) if args.shape else tuple(cfg.shape)
    sz3g.load()
    x, a0 = make_slab(cfg, world, rank, shape)
    N_local, N_global = x.numel(), math.prod(shape)
    s = x.element_size()
    NB_local = sz3g.num_blocks(x.shape)
    two_pass = args.path == "two-pass"
    rt = RoundTrip(x, cfg.eb, cfg.eb_mode, cfg.radius, dim0_offset=a0, path=args.path)
    graphs = args.graphs == "on" or (args.graphs == "auto" and world == 1)
    if graphs:
        try:
            rt.capture()      # each segment of the step replayed from a CUDA graph (no host gaps)
        except Exception as e:   # keep measuring (eagerly) rather than fail the run; say so in the line
            print(f"bench: CUDA graph capture failed ({e}); timing the eager step", file=sys.stderr)
            torch.cuda.synchronize()
            rt.graphs = None
            graphs = False
    bufs, out, stream = rt.bufs, rt.out, rt.stream

    for _ in range(max(3, args.warmup)):
        rt.step()
    barrier(world)
    recs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = sz3g.launch_count()
    with ClockSampler(dev) as clk:
        barrier(world)
        t_start.record(stream)
        for k in range(args.steps):
            rt.step(recs[k])
        rt.finish()                     # the last step's histogram all-reduce is part of the step
        t_end.record(stream)
        barrier(world)
    launches = sz3g.launch_count() - l0 if not graphs else rt.launches_per_step * args.steps
    launches = sum_over_ranks(launches, world)
    ms_total = max_over_ranks(t_start.elapsed_time(t_end), world)
    ms_step = ms_total / args.steps
    # per-kernel times: mean over the timed steps on this rank, then the max over ranks
    comp_ms = max_over_ranks(sum(r[0].elapsed_time(r[1]) for r in recs) / args.steps, world)
    dec_ms = max_over_ranks(sum(r[2].elapsed_time(r[3]) for r in recs) / args.steps, world)
    ana_ms = max_over_ranks(sum(r[4].elapsed_time(r[5]) for r in recs) / args.steps, world)
    hist_ar_ms = max_over_ranks(sum(r[1].elapsed_time(r[2]) for r in recs) / args.steps, world)   # on-stream part

    res = rt.result()
    n_out_local = res.n_outliers
    n_out = sum_over_ranks(n_out_local, world)
    peaks = measured_peaks()
    # algorithmic bytes, per rank; the roofline rows use the max-over-ranks times with
    # the largest rank's bytes (rank 0 holds the largest slab: slab_bounds gives the extra block rows
    # to the first ranks)
    b = alg_bytes(N_local, NB_local, s, n_out_local)
    b = {k: max_over_ranks(float(v), world) for k, v in b.items()}
    value = N_global * s / (ms_step * 1e-3) / 1e9
    step_bytes = b["analyze"] + b["quantize"] + b["decompress"]

    # ---------------- reconstruction quality (NEXT-3 metrics): bound check, max error, PSNR
    st = sz3g.error_stats(x, out, res.eb_abs).cpu().tolist()
    lo, hi = (float(v) for v in bufs.minmax.cpu())
    quality = {"max_abs_err": max_over_ranks(st[0], world), "eb_abs": res.eb_abs,
               "above_eb": sum_over_ranks(int(st[2]), world),
               "psnr_db": sz3g.psnr(hi - lo, (st[1] if world == 1 else _sum_f(st[1], world)) / N_global),
               "entropy_bits": entropy_bits(bufs.hist)}
    if quality["above_eb"] != 0 or not quality["max_abs_err"] <= res.eb_abs:
        raise RuntimeError(f"error bound violated: {quality}")

    # ---------------- reported counters (north_star parity rule): near-ties etc. on the whole field
    ties = None
    if not args.no_ties:
        cnt = sz3g.tie_counts(x, cfg.eb, cfg.eb_mode, cfg.radius, bufs.minmax, bufs.coef_codes, rt.beta)
        ties = {k: sum_over_ranks(int(v), world) for k, v in zip(sz3g.TIE_COUNTER_NAMES, cnt.cpu().tolist())}
        ties["note"] = ("(i) elements within 1e-9 of a half-integer (t by true division), (ii) rint(division) != "
                        "rint(reciprocal product), (iii) coefficients in the parity tie window, blocks holding one; "
                        "sz3g_tie_counts, equal to the oracle's counters on c1-c4 (tests/test_gpu_ties.py)")

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

    # ---------------- SZ3-Interp (NEXT-4) on the same field
    interp = None
    if not args.no_interp:
        interp = interp_leg(sz3g, x, out, bufs.minmax, cfg, N_local, s, args, world, peaks, stream)

    # ---------------- CPU oracle beside it (rank 0, N = 1 only; bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        pa = min(504, max(0, (x.shape[0] // 2 // 6) * 6))
        p = min(args.cpu_sample_planes, x.shape[0] - pa)
        xs = x[pa:pa + p].cpu().numpy()
        t = oracle_round_trip(xs, cfg, lo, hi, pa)
        cpu = {"value": xs.nbytes / t / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"planes [{pa},{pa + p}) of {cfg.name} ({xs.size} elements, global range), "
                         f"compress + decompress, one host core, {t:.1f} s", **host_cpu()}

    # ---------------- per-config legs on the same GPU (N = 1): stress variants of this field first
    legs = {}
    specs = [v for v in args.configs.split(",") if v] if world == 1 else []
    eb_abs_used = res.eb_abs
    del rt, bufs, res, out
    torch.cuda.empty_cache()
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if specs else None
    for spec in [v for v in specs if v.split("r")[0] == cfg.name and shape == tuple(cfg.shape)]:
        legs[spec] = config_leg(sz3g, spec, peaks, args.config_steps, 3, flush_buf, x=x)

    # ---------------- end to end through the public API with HOST buffers (pinned), copies timed:
    # paper_2111_02925_b200.pipeline.PipelinedCodec round-trips a sequence of fields from pinned host
    # memory (here: the same field, e2e_steps times) -- host->device copy, analyze, quantise, Huffman
    # coding of codes and coefficients, decompression, device->host copy of the compressed stream and of
    # x' -- with consecutive fields' copies overlapped on the two copy engines.
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        from paper_2111_02925_b200.pipeline import PipelinedCodec
        h_x = torch.empty_like(x, device="cpu").pin_memory()
        h_x.copy_(x)
        h_out = torch.empty_like(x, device="cpu").pin_memory()
        codec = PipelinedCodec(tuple(x.shape), x.dtype, cfg.eb, cfg.eb_mode, cfg.radius, device=x.device,
                               dim0_offset=a0)
        del x
        torch.cuda.empty_cache()
        codec.run([h_x, h_x], h_out)                 # warm-up: both slots (their pinned payload buffers)
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(codec.s_in)
        sizes = codec.run([h_x] * args.e2e_steps, h_out)
        e1.record(codec.s_out)
        barrier(world)
        e1.synchronize()
        e_ms = max_over_ranks(e0.elapsed_time(e1), world) / args.e2e_steps
        bi = sum_over_ranks(h_x.numel() * s, world)
        bo = sum_over_ranks(int(sum(sizes) / len(sizes)) + h_out.numel() * s, world)
        e2e = {"value": N_global * s / (e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": bi,
               "d2h_bytes_per_step": bo, "ms_per_step": e_ms, "fields": args.e2e_steps,
               "note": "PipelinedCodec: pinned host field -> device, analyze + quantise + Huffman (codes, "
                       "coefficients) + decompress, compressed stream + x' -> pinned host; copies of consecutive "
                       "fields overlapped (3 streams, double-buffered)"}
        del codec, h_x, h_out
    else:
        del x
    torch.cuda.empty_cache()

    for spec in specs:
        if spec not in legs:
            legs[spec] = config_leg(sz3g, spec, peaks, args.config_steps, 3, flush_buf)

    if rank == 0:
        clocks = clk.summary()
        qroof = roof(b["quantize"], comp_ms, peaks["hbm_gbs"])
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 data, f64 arithmetic", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.desc}", "shape": list(shape), "eb_rel": cfg.eb,
                       "radius": cfg.radius, "block": 6, "parallelism": f"slabs{world}",
                       "dist_backend": args.dist_backend if world > 1 else None,
                       "launch": "CUDA graph per step segment" if graphs else "eager (one host call per kernel)",
                       "l2": "inputs (16 GiB) larger than L2; no flush" if N_global * s > (1 << 30)
                       else "input smaller than 1 GiB: NOT flushed between steps (rehearsal shape)"},
            "roofline": {"bound": "hbm", "kernel": "k_compress_tma" + ("<beta in>" if two_pass else ""),
                         "achieved": qroof["achieved"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": qroof["frac"],
                         "traffic": profiled_traffic("k_compress_tma" + ("_beta" if two_pass else ""), cfg.name),
                         "peak_source": peaks["source"], "frac_nominal": qroof["frac_nominal"],
                         "peak_nominal": NOMINAL_HBM_GBS, "alg_bytes_per_launch": b["quantize"],
                         "bytes_rule": "SURVEY 8(d): N (s + 2) + 16 NB + outliers (8 + s)",
                         "beta_reread_bytes": b["beta"] if two_pass else 0,
                         "frac_incl_beta_reread": (b["quantize"] + (b["beta"] if two_pass else 0)) /
                         (comp_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                         "ms_per_launch": comp_ms, "ranks": "max over ranks"},
            "step_roofline": {"alg_bytes": step_bytes, "frac": step_bytes / (ms_step * 1e-3) / 1e9 / peaks["hbm_gbs"],
                              "frac_nominal": step_bytes / (ms_step * 1e-3) / 1e9 / NOMINAL_HBM_GBS,
                              "note": "analyze (N s) + quantize + decompress algorithmic bytes / step time"},
            "compress_gbs": N_global * s / ((ana_ms + comp_ms) * 1e-3) / 1e9,
            "compress_note": "input bytes / (analyze + quantise) time: REL compression needs both passes (P:833)",
            "decompress_gbs": N_global * s / (dec_ms * 1e-3) / 1e9,
            "decompress_roofline": roof(b["decompress"], dec_ms, peaks["hbm_gbs"]),
            "analyze_roofline": {"kernel": "k_analyze_tma" if two_pass else "k_value_range",
                                 **roof(b["analyze"], ana_ms, peaks["hbm_gbs"])},
            "hist_allreduce_ms": hist_ar_ms if world > 1 else 0.0,
            "hist_allreduce_note": "N > 1: the histogram all-reduce runs on a side stream overlapped with the "
                                   "decompression (the codebook needs it, decompression does not); the timed region "
                                   "ends after the last one",
            "path": args.path,
            "quality": quality, "ties": ties, "huffman": huff, "truncation": trunc, "lr": lr, "interp": interp,
            "configs": legs or None, "outliers": n_out, "eb_abs": eb_abs_used,
            "clocks": clocks, "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu,
            "paper_context": PAPER_CONTEXT,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def _sum_f(v: float, world: int) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


if __name__ == "__main__":
    main()
