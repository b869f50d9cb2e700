"""GPU parity of SZ3-LR (NEXT-4: sz3g_lr_quantize / sz3g_lr_decompress) against the LR oracle
(oracle/DEFINITION.md L1-L7), on the same seeded input bytes.  Rules of tests/parity_util.py, plus the
per-block predictor flags (bit-exact outside the oracle's coefficient near-tie blocks).  Covers the TMA
and the plain kernels, f32 / f64, ABS / REL, ragged shapes, small radii, non-finite and huge values, the
closed-form fields of tests/test_lr_oracle.py and the configs at full size."""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from tests.parity_util import block_ids, compare  # noqa: E402
from tests.test_gpu_parity import fuzz_case  # noqa: E402

pytestmark = pytest.mark.gpu

GEN = 0x1  # FLAG_FORCE_GENERIC


def sz():
    from paper_2111_02925_b200 import sz3g
    sz3g.load()
    return sz3g


def check_lr(xh: np.ndarray, eb, mode, R, flags=0):
    s = sz()
    x = torch.from_numpy(np.ascontiguousarray(xh)).cuda()
    res = s.lr_compress(x, eb, mode, R, outlier_cap=x.numel(), flags=flags)
    xo = s.decompress(res, flags=flags)
    torch.cuda.synchronize()
    n = res.n_outliers
    gpu = dict(codes=res.codes.cpu().numpy(), coef_codes=res.coef_codes.cpu().numpy(),
               coef_raw=res.coef_raw.cpu().numpy(), outlier_idx=res.outlier_idx[:n].cpu().numpy().view(np.uint64),
               outlier_val=res.outlier_val[:n].cpu().numpy(), hist=res.hist.cpu().numpy(), eb_abs=res.eb_abs)
    gflags = res.lr_flags.cpu().numpy()
    orc = oracle.lr_compress(xh, eb, mode, radius=R)
    exempt = orc.block_exempt.astype(bool)
    bad = np.flatnonzero(~exempt & (gflags != orc.flags))
    assert bad.size == 0, f"predictor flags differ in {bad.size} non-exempt blocks, e.g. {bad[:5]}"
    dec_of_gpu = oracle.lr_decompress(dims=orc.dims, dtype=xh.dtype, radius=R, eb_abs=orc.eb_abs, codes=gpu["codes"],
                                      coef_codes=gpu["coef_codes"], flags=gflags, outlier_idx=gpu["outlier_idx"],
                                      outlier_val=gpu["outlier_val"])
    rep = compare(xh, gpu, orc, xdec_gpu=xo.cpu().numpy(), xdec_orc_of_gpu=dec_of_gpu)
    rep["lorenzo_blocks"] = int(gflags.sum())
    rep["blocks"] = int(gflags.size)
    return rep


@pytest.mark.parametrize("flags", [0, GEN], ids=["tma", "plain"])
@pytest.mark.parametrize("t", list(range(0, 40, 2)))
def test_lr_fuzz_parity(t, flags):
    xh, eb, mode, R = fuzz_case(t)
    check_lr(xh.reshape((1,) * (3 - xh.ndim) + xh.shape), eb, mode, R, flags)


def tiled(shape, f, dtype):
    i, j, k = np.meshgrid(*(np.arange(n) % 6 for n in shape), indexing="ij")
    return np.ascontiguousarray(f(i, j, k).astype(dtype))


@pytest.mark.parametrize("flags", [0, GEN], ids=["tma", "plain"])
@pytest.mark.parametrize("shape,dtype", [((12, 12, 96), np.float32), ((14, 13, 100), np.float64),
                                         ((6, 6, 6), np.float32), ((30, 31, 200), np.float32)])
def test_lr_closed_form_fields(shape, dtype, flags):
    # f = i + 2j + 3k + 5ijk per block with 2eb = 1: Lorenzo residuals 0/1/2/3/5, exact reconstruction
    rep = check_lr(tiled(shape, lambda i, j, k: i + 2 * j + 3 * k + 5 * i * j * k, dtype), 0.5, "abs", 32768, flags)
    assert rep["lorenzo_blocks"] > 0
    # a step inside every block: Lorenzo, one residual of 1000 (a radius outlier for R = 64)
    for R in (32768, 64):
        rep = check_lr(tiled(shape, lambda i, j, k: 1000.0 * (k >= 3), dtype), 0.5, "abs", R, flags)
        assert rep["lorenzo_blocks"] == rep["blocks"] or shape[2] % 6 != 0


@pytest.mark.parametrize("flags", [0, GEN], ids=["tma", "plain"])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("mode", ["abs", "rel"])
def test_lr_mixed_field_with_specials(dtype, mode, flags):
    rng = np.random.default_rng(7)
    shape = (37, 45, 130)
    i, j, k = np.meshgrid(*(np.arange(n, dtype=np.float64) for n in shape), indexing="ij")
    curved = np.sin(i / 3.0) * np.cos(j / 5.0) + 0.01 * (k - 60) ** 2 / 100
    noisy = 0.1 * i - 0.05 * j + 0.02 * k + 1e-3 * rng.standard_normal(shape)
    xh = np.where(i < 18, curved, noisy).astype(dtype)
    flat = xh.reshape(-1)
    pos = rng.choice(flat.size, 200, replace=False)
    if mode == "abs":   # REL with non-finite values has no finite range
        flat[pos[:50]] = np.nan
        flat[pos[50:100]] = np.inf
        flat[pos[100:150]] = -np.inf
    flat[pos[150:]] = 1e30 if dtype == np.float32 else 1e300
    eb = 1e-4 if mode == "abs" else 1e-6
    rep = check_lr(xh, eb, mode, 4096, flags)
    assert 0 < rep["lorenzo_blocks"] < rep["blocks"]


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_lr_config_full_size(name):
    from synth import config_by_name, make_field
    cfg = config_by_name(name)
    xh = make_field(cfg, device="cuda").cpu().numpy()
    rep = check_lr(xh, cfg.eb, cfg.eb_mode, cfg.radius)
    print(name, rep)
    assert rep["exempt_blocks"] <= max(4, oracle.num_blocks(xh.shape) // 10000)


def test_lr_matches_regression_when_all_regression():
    # a linear field: every block keeps regression, and the outputs equal sz3g_regression_quantize's
    s = sz()
    shape = (25, 31, 97)
    i, j, k = np.meshgrid(*(np.arange(n, dtype=np.float64) for n in shape), indexing="ij")
    x = torch.from_numpy((3.0 + 0.25 * i - 0.5 * j + 0.125 * k).astype(np.float32)).cuda()
    lr = s.lr_compress(x, 1e-3, "abs", 1024, outlier_cap=x.numel())
    codes, coef, hist = lr.codes.clone(), lr.coef_codes.clone(), lr.hist.clone()
    assert int(lr.lr_flags.sum()) == 0
    reg = s.compress(x, 1e-3, "abs", 1024, two_pass=False, outlier_cap=x.numel())
    assert torch.equal(codes, reg.codes) and torch.equal(coef, reg.coef_codes) and torch.equal(hist, reg.hist)


def test_lr_invalid_arguments():
    s = sz()
    lib = s.load()
    x = torch.zeros((6, 6, 6), device="cuda")
    g = s.make_grid(x.shape, x.dtype)
    p = s.make_params(1e-3, "abs", 1024)
    import ctypes
    rc = lib.sz3g_lr_quantize(ctypes.byref(g), ctypes.byref(p), s._ptr(x), None, None, None, None, None, None, None,
                              0, None, None, None, None, None)
    assert rc == -1
    rc = lib.sz3g_lr_decompress(ctypes.byref(g), ctypes.byref(p), None, None, None, None, None, None, 0, None, None,
                                None)
    assert rc == -1


@pytest.mark.parametrize("flags", [0, GEN], ids=["tma", "plain"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_lr_large_q_tiles(dtype, flags):
    """|x / 2eb| beyond 2^26: those tiles leave the int32 fast routine for the exact int64 one (f64: the
    Lorenzo codes stay usable; f32: the prequantised grid is coarser than the data, mostly outliers)."""
    rng = np.random.default_rng(3)
    shape = (13, 14, 100)
    i, j, k = np.meshgrid(*(np.arange(n, dtype=np.float64) for n in shape), indexing="ij")
    x = 1e9 + 1e3 * np.sin(i / 4.0) * np.cos(j / 3.0) + 50.0 * k + rng.uniform(-0.2, 0.2, shape)
    x[i < 6] -= 1e9          # first block row small: the fast routine, the rest large
    rep = check_lr(x.astype(dtype), 1.0, "abs", 32768, flags)
    assert rep["lorenzo_blocks"] > 0


def test_lr_slab_invariance():
    """Block-aligned slabs (dim0_offset, the global range) reproduce the whole-field SZ3-LR output: codes,
    flags, coefficient codes, histogram, and outliers with global indices; each slab decompresses to the
    matching planes of the whole field's reconstruction."""
    s = sz()
    from synth import make_field
    x = make_field("c2", device="cuda", shape=(48, 64, 96))
    x.view(-1)[12345] = float("inf")      # an outlier in the second slab (global index)
    x.view(-1)[250000] = 1e30
    whole = s.lr_compress(x, 1e-4, "abs", 4096, outlier_cap=x.numel())
    wcodes, wflags, wcoef, whist = (whole.codes.clone(), whole.lr_flags.clone(), whole.coef_codes.clone(),
                                    whole.hist.clone())
    widx = set(whole.outlier_idx[:whole.n_outliers].cpu().tolist())
    xw = s.decompress(whole).clone()
    codes, flags, coef, idx, hist = [], [], [], set(), torch.zeros_like(whist)
    for a, b in [(0, 12), (12, 30), (30, 48)]:
        xs = x[a:b].contiguous()
        mm, beta = s.regression_analyze(xs)
        part = s.lr_quantize(xs, 1e-4, "abs", 4096, mm, beta, outlier_cap=xs.numel(), dim0_offset=a)
        part.finalize()
        codes.append(part.codes.clone())
        flags.append(part.lr_flags.clone())
        coef.append(part.coef_codes.clone())
        idx |= set(part.outlier_idx[:part.n_outliers].cpu().tolist())
        hist += part.hist
        xo = s.lr_decompress(part.codes, part.coef_codes, part.lr_flags, part.outlier_idx, part.outlier_val,
                             part.n_outliers, part.eb_abs, 4096, xs.dtype, dim0_offset=a)
        assert torch.equal(xo.view(torch.int32), xw[a:b].view(torch.int32))
    assert torch.equal(torch.cat(codes), wcodes)
    assert torch.equal(torch.cat(flags), wflags) and torch.equal(torch.cat(coef), wcoef)
    assert torch.equal(hist, whist)
    assert idx == widx and len(widx) >= 2


@pytest.mark.parametrize("flags", [0, GEN], ids=["tma", "plain"])
@pytest.mark.parametrize("R", [32768, 3000])
def test_lr_codes_outside_histogram_window(R, flags):
    """Residuals spread over thousands of bins: many codes fall outside the kernels' 4096-bin shared
    histogram window (global atomics in the second walk), with a curved region where Lorenzo wins; at
    R = 3000 the wide residuals are also radius outliers."""
    rng = np.random.default_rng(11)
    shape = (18, 24, 200)
    i, j, k = np.meshgrid(*(np.arange(n, dtype=np.float64) for n in shape), indexing="ij")
    eb = 1e-3
    noisy = rng.uniform(-1.0, 1.0, shape) * 6000 * 2 * eb
    curved = 40.0 * np.sin(i / 2.0) * np.cos(k / 3.0) + 0.5 * j * j
    x = np.where(j < 12, noisy, curved).astype(np.float32)
    rep = check_lr(x, eb, "abs", R, flags)
    assert 0 < rep["lorenzo_blocks"] < rep["blocks"]
    res = sz().lr_compress(torch.from_numpy(x).cuda(), eb, "abs", R, outlier_cap=x.size, flags=flags)
    codes = res.codes.cpu().numpy().astype(np.int64)
    inside = (codes >= R - 2048) & (codes < R + 2048)
    assert (codes != 0).sum() > 0 and (~inside & (codes != 0)).sum() > 1000
