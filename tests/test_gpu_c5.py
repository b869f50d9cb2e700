"""Config c5 (1024 x 2048 x 2048 f32, 16 GiB) in the launch configuration bench.py times, against the
oracle element by element on sampled block-aligned slabs (the oracle cannot finish the whole field in
seconds), plus every property that holds at any size on the whole output.

The measured step is ``RoundTrip(path="two-pass")`` -- the same object bench.py drives:
k_analyze_tma (range + beta) -> k_compress_tma<BETA> -> k_decompress_tma + k_outlier_scatter, with the
REL decompression reading the device range and the device outlier counter.  Definition: oracle/DEFINITION.md
O1-O11 + D; Algorithm 1's predict / quantize loop P:447-450; value-range eb P:833.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from tests.parity_util import compare  # noqa: E402

pytestmark = pytest.mark.gpu

# (first plane, planes): the first block row, two in the upper half (global indices > 2^31), and the
# ragged last block row (planes 1020-1023, edge extent 4, indices up to 2^32 - 1)
SLABS = [(0, 12), (504, 12), (768, 6), (1020, 4)]


@pytest.fixture(scope="module")
def c5():
    from paper_2111_02925_b200 import sz3g
    from paper_2111_02925_b200.roundtrip import RoundTrip
    from synth import config_by_name, make_field
    sz3g.load()
    cfg = config_by_name("c5")
    x = make_field(cfg, device="cuda")
    rt = RoundTrip(x, cfg.eb, cfg.eb_mode, cfg.radius)
    for _ in range(2):      # the bench runs warm-up steps into the same buffers first
        rt.step()
    res = rt.result()
    torch.cuda.synchronize()
    yield cfg, x, rt, res
    del rt, x
    torch.cuda.empty_cache()


def slab_gpu(res, rt, a0, rows, n1, n2):
    NB1, NB2 = math.ceil(n1 / 6), math.ceil(n2 / 6)
    b0, b1 = (a0 // 6) * NB1 * NB2, ((a0 + rows + 5) // 6) * NB1 * NB2
    n = res.n_outliers
    oidx = res.outlier_idx[:n].cpu().numpy().view(np.uint64)
    oval = res.outlier_val[:n].cpu().numpy()
    sel = (oidx >= a0 * n1 * n2) & (oidx < (a0 + rows) * n1 * n2)
    return dict(codes=res.codes[a0:a0 + rows].cpu().numpy(), coef_codes=res.coef_codes[b0:b1].cpu().numpy(),
                coef_raw=res.coef_raw[b0:b1].cpu().numpy() if res.coef_raw is not None else None,
                outlier_idx=oidx[sel], outlier_val=oval[sel], eb_abs=res.eb_abs)


def test_c5_bench_path_whole_field_properties(c5):
    """Global invariants of the bench step on all 4.3 G elements (P3): range = numpy-free device
    min/max of sz3g_value_range, eb_abs = eb * (max - min), sum(hist) = N, hist[0] = #outliers,
    |x - x'| <= eb_abs everywhere, outliers reproduced exactly."""
    from paper_2111_02925_b200 import sz3g
    cfg, x, rt, res = c5
    lo, hi = (float(v) for v in sz3g.value_range(x).cpu())
    mm = rt.bufs.minmax.cpu().tolist()
    assert mm == [lo, hi]
    assert res.eb_abs == cfg.eb * (hi - lo)
    N = x.numel()
    assert int(res.hist.sum()) == N and int(res.hist[0]) == res.n_outliers
    assert res.n_outliers <= rt.cap
    st = sz3g.error_stats(x, rt.out, res.eb_abs).cpu().tolist()
    assert st[2] == 0 and st[0] <= res.eb_abs
    n = res.n_outliers
    if n:
        idx = res.outlier_idx[:n]
        assert torch.equal(rt.out.view(-1)[idx].view(torch.int32), res.outlier_val[:n].view(torch.int32))


@pytest.mark.parametrize("a0,rows", SLABS, ids=[f"planes{a}-{a + r}" for a, r in SLABS])
def test_c5_bench_path_slab_parity(c5, a0, rows):
    """Codes, coefficient codes, beta (1e-12 block scale), outlier set (global indices) and x' of one
    block-aligned slab of the bench step's output == the oracle on that slab with the global range."""
    cfg, x, rt, res = c5
    n0, n1, n2 = x.shape
    lo, hi = (float(v) for v in rt.bufs.minmax.cpu())
    xs = x[a0:a0 + rows].cpu().numpy()
    orc = oracle.compress(xs, cfg.eb, "rel", radius=cfg.radius, dim0_offset=a0, value_range_override=(lo, hi))
    gpu = slab_gpu(res, rt, a0, rows, n1, n2)
    rep = compare(xs, gpu, orc, xdec_gpu=rt.out[a0:a0 + rows].cpu().numpy())
    assert rep["exempt_blocks"] <= 4
    print(a0, rows, rep)


def test_c5_fused_path_slab_parity(c5):
    """The fused kernel (value range -> k_compress_tma<fused>) on the same field, one slab vs the oracle."""
    from paper_2111_02925_b200 import sz3g
    cfg, x, rt, _ = c5
    rt.out.zero_()   # reuse the bench buffers' output tensor for the fused path's x'
    mm = sz3g.value_range(x)
    res = sz3g.regression_compress(x, cfg.eb, cfg.eb_mode, cfg.radius, d_minmax=mm, coef_raw=True,
                                   outlier_cap=rt.cap).finalize()
    xo = sz3g.decompress(res, out=rt.out)
    torch.cuda.synchronize()
    lo, hi = (float(v) for v in mm.cpu())
    n0, n1, n2 = x.shape
    a0, rows = 510, 6
    xs = x[a0:a0 + rows].cpu().numpy()
    orc = oracle.compress(xs, cfg.eb, "rel", radius=cfg.radius, dim0_offset=a0, value_range_override=(lo, hi))
    compare(xs, slab_gpu(res, rt, a0, rows, n1, n2), orc, xdec_gpu=xo[a0:a0 + rows].cpu().numpy())
    # and the two kernels agree bit for bit on the whole field
    assert torch.equal(res.codes, rt.bufs.codes) and torch.equal(res.coef_codes, rt.bufs.coef_codes)
    del res
    torch.cuda.empty_cache()


def test_c5_slab_outlier_indices_above_2_32(c5):
    """Global outlier indices beyond 2^32: a c5 slab compressed as if it were planes [6000, 6006) of a
    taller field (dim0_offset = 6000, indices ~ 2.5e10), R = 64 so that ~2% of the elements are radius
    outliers, through the bench's two-pass kernels; vs the oracle with the same offset."""
    from paper_2111_02925_b200.roundtrip import RoundTrip
    cfg, x, rt0, _ = c5
    lo, hi = (float(v) for v in rt0.bufs.minmax.cpu())
    xs_d = x[1014:1020].contiguous()
    rt = RoundTrip(xs_d, cfg.eb, cfg.eb_mode, 64, dim0_offset=6000, outlier_cap=xs_d.numel())
    rt.step()
    # REL with the GLOBAL range: overwrite the slab range and rerun quantise + decompress (as the
    # sharded bench does after its MAX all-reduce)
    from paper_2111_02925_b200 import sz3g
    b = rt.bufs
    b.minmax.copy_(torch.tensor([lo, hi], dtype=torch.float64))
    b.reset()
    sz3g.regression_quantize(xs_d, cfg.eb, cfg.eb_mode, 64, b.minmax, rt.beta, bufs=b, reset=False, dim0_offset=6000)
    sz3g.regression_decompress(b.codes, b.coef_codes, b.outlier_idx, b.outlier_val, rt.cap, cfg.eb, 64, xs_d.dtype,
                               dim0_offset=6000, out=rt.out, d_outlier_count=b.outlier_count, eb_mode="rel",
                               d_minmax=b.minmax)
    res = rt.result()
    xs = xs_d.cpu().numpy()
    orc = oracle.compress(xs, cfg.eb, "rel", radius=64, dim0_offset=6000, value_range_override=(lo, hi))
    n = res.n_outliers
    assert n > 10000 and n == orc.outlier_idx.size
    gpu = dict(codes=res.codes.cpu().numpy(), coef_codes=res.coef_codes.cpu().numpy(),
               coef_raw=res.coef_raw.cpu().numpy(), outlier_idx=res.outlier_idx[:n].cpu().numpy().view(np.uint64),
               outlier_val=res.outlier_val[:n].cpu().numpy(), hist=res.hist.cpu().numpy(), eb_abs=res.eb_abs)
    assert int(gpu["outlier_idx"].min()) >= 6000 * 2048 * 2048 > 2 ** 32
    compare(xs, gpu, orc, xdec_gpu=rt.out.cpu().numpy())


def test_c5_stress_r16_slab_parity(c5):
    """The bench's c5 stress leg (R = 16: 38.6% of the elements are radius outliers) on a slab, through
    the bench's two-pass kernels with the global range, element by element against the oracle: the
    outlier-heavy rare path at the measured configuration."""
    from paper_2111_02925_b200.roundtrip import RoundTrip
    cfg, x, rt0, _ = c5
    lo, hi = (float(v) for v in rt0.bufs.minmax.cpu())
    a0, rows = 504, 6
    xs_d = x[a0:a0 + rows].contiguous()
    rt = RoundTrip(xs_d, cfg.eb, cfg.eb_mode, 16, dim0_offset=a0, outlier_cap=xs_d.numel())
    rt.bufs.minmax.copy_(torch.tensor([lo, hi], dtype=torch.float64))
    from paper_2111_02925_b200 import sz3g
    b = rt.bufs
    sz3g.regression_analyze(xs_d, torch.empty_like(b.minmax), rt.beta)      # beta of the slab's blocks
    b.reset()
    sz3g.regression_quantize(xs_d, cfg.eb, cfg.eb_mode, 16, b.minmax, rt.beta, bufs=b, reset=False, dim0_offset=a0)
    sz3g.regression_decompress(b.codes, b.coef_codes, b.outlier_idx, b.outlier_val, rt.cap, cfg.eb, 16, xs_d.dtype,
                               dim0_offset=a0, out=rt.out, d_outlier_count=b.outlier_count, eb_mode="rel",
                               d_minmax=b.minmax)
    res = rt.result()
    xs = xs_d.cpu().numpy()
    orc = oracle.compress(xs, cfg.eb, "rel", radius=16, dim0_offset=a0, value_range_override=(lo, hi))
    n = res.n_outliers
    assert n == orc.outlier_idx.size and n > 0.3 * xs.size
    gpu = dict(codes=res.codes.cpu().numpy(), coef_codes=res.coef_codes.cpu().numpy(),
               coef_raw=res.coef_raw.cpu().numpy(), outlier_idx=res.outlier_idx[:n].cpu().numpy().view(np.uint64),
               outlier_val=res.outlier_val[:n].cpu().numpy(), hist=res.hist.cpu().numpy(), eb_abs=res.eb_abs)
    compare(xs, gpu, orc, xdec_gpu=rt.out.cpu().numpy())


def test_c5_lr_slab_parity(c5):
    """SZ3-LR (NEXT-4) as the bench's lr leg runs it -- lr_quantize from the analyze pass's range and beta
    of the whole field -- on a slab of c5, against the LR oracle on that slab with the global range."""
    from paper_2111_02925_b200 import sz3g
    cfg, x, rt0, _ = c5
    lo, hi = (float(v) for v in rt0.bufs.minmax.cpu())
    n0, n1, n2 = x.shape
    NB1, NB2 = math.ceil(n1 / 6), math.ceil(n2 / 6)
    a0, rows = 1014, 6
    xs_d = x[a0:a0 + rows].contiguous()
    b0 = (a0 // 6) * NB1 * NB2
    beta = rt0.beta[b0:b0 + NB1 * NB2].contiguous()       # the timed step's beta of these blocks
    res = sz3g.lr_quantize(xs_d, cfg.eb, cfg.eb_mode, cfg.radius, rt0.bufs.minmax, beta,
                           outlier_cap=xs_d.numel(), dim0_offset=a0).finalize()
    xo = sz3g.lr_decompress(res.codes, res.coef_codes, res.lr_flags, res.outlier_idx, res.outlier_val,
                            res.outlier_idx.numel(), cfg.eb, cfg.radius, xs_d.dtype, a0,
                            d_outlier_count=res.outlier_count, eb_mode=cfg.eb_mode, d_minmax=rt0.bufs.minmax)
    torch.cuda.synchronize()
    xs = xs_d.cpu().numpy()
    orc = oracle.lr_compress(xs, cfg.eb, "rel", radius=cfg.radius, dim0_offset=a0, value_range_override=(lo, hi))
    n = res.n_outliers
    gflags = res.lr_flags.cpu().numpy()
    ex = orc.block_exempt.astype(bool)
    assert np.array_equal(gflags[~ex], orc.flags[~ex]) and int(gflags.sum()) > 0
    gpu = dict(codes=res.codes.cpu().numpy(), coef_codes=res.coef_codes.cpu().numpy(),
               coef_raw=res.coef_raw.cpu().numpy(), outlier_idx=res.outlier_idx[:n].cpu().numpy().view(np.uint64),
               outlier_val=res.outlier_val[:n].cpu().numpy(), hist=res.hist.cpu().numpy(), eb_abs=res.eb_abs)
    compare(xs, gpu, orc, xdec_gpu=xo.cpu().numpy())
