"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element, on the same
seeded input bytes.  Rules in tests/parity_util.py.  Needs a B200 (marked gpu)."""
from __future__ import annotations

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from tests.parity_util import compare  # noqa: E402

pytestmark = pytest.mark.gpu

GEN = 0x1  # FLAG_FORCE_GENERIC


def sz():
    from paper_2111_02925_b200 import sz3g
    sz3g.load()
    return sz3g


def run_gpu(x: torch.Tensor, eb, mode, R, flags=0, dim0_offset=0, d_minmax=None, cap=None, two_pass=False):
    s = sz()
    cap = cap if cap is not None else x.numel()
    if two_pass:   # analyze (range + beta) -> quantize; REL uses the analyze pass's own range
        minmax, beta = s.regression_analyze(x)
        res = s.regression_quantize(x, eb, mode, R, d_minmax if d_minmax is not None else minmax, beta,
                                    outlier_cap=cap, flags=flags, dim0_offset=dim0_offset)
    else:
        res = s.regression_compress(x, eb, mode, R, d_minmax=d_minmax, coef_raw=True, flags=flags,
                                    dim0_offset=dim0_offset, outlier_cap=cap)
    res.finalize()
    xo = s.decompress(res, flags=flags)
    torch.cuda.synchronize()
    n = res.n_outliers
    gpu = dict(codes=res.codes.cpu().numpy(), coef_codes=res.coef_codes.cpu().numpy(),
               coef_raw=res.coef_raw.cpu().numpy(),
               outlier_idx=res.outlier_idx[:n].cpu().numpy().view(np.uint64),
               outlier_val=res.outlier_val[:n].cpu().numpy(),
               hist=res.hist.cpu().numpy(), eb_abs=res.eb_abs)
    return gpu, xo.cpu().numpy(), res


def check(xh: np.ndarray, eb, mode, R, flags=0, rng_override=None, two_pass=False):
    x = torch.from_numpy(np.ascontiguousarray(xh)).cuda()
    gpu, xdec, res = run_gpu(x, eb, mode, R, flags, two_pass=two_pass)
    orc = oracle.compress(xh, eb, mode, radius=R, value_range_override=rng_override)
    dec_of_gpu = oracle.decompress(dims=orc.dims, dtype=xh.dtype, radius=R, eb_abs=orc.eb_abs, codes=gpu["codes"],
                                   coef_codes=gpu["coef_codes"], outlier_idx=gpu["outlier_idx"],
                                   outlier_val=gpu["outlier_val"])
    rep = compare(xh, gpu, orc, xdec_gpu=xdec, xdec_orc_of_gpu=dec_of_gpu)
    return rep


# ----------------------------------------------------------------------------- fuzz (both kernel paths)
def fuzz_case(t):
    rng = np.random.default_rng(1000 + t)
    shapes = [(13, 17, 96), (7, 11, 200), (20, 6, 64), (1, 1, 500), (3, 40, 8), (12, 12, 12), (40, 1, 36),
              (6, 6, 97), (9, 5, 104), (1, 37, 1)]
    dims = shapes[t % len(shapes)] if t < 20 else tuple(int(v) for v in rng.integers(1, 41, size=3))
    dtype = [np.float32, np.float64][t % 2]
    mode = ["abs", "rel"][(t // 2) % 2]
    R = [32768, 4, 64, 1, 32768][(t // 4) % 5]
    kind = t % 4
    if kind == 0:
        f = rng.normal(size=dims)
    elif kind == 1:
        f = np.cumsum(np.cumsum(rng.normal(size=dims), axis=-1), axis=0)
    elif kind == 2:
        f = np.exp(2 * rng.normal(size=dims))
    else:
        f = rng.uniform(-1e4, 1e4, size=dims)
    eb = float(rng.choice([1e-1, 1e-3, 1e-5]))
    if mode == "abs":
        eb *= float(np.ptp(f) + 1e-3)
    return f.astype(dtype), eb, mode, R


@pytest.mark.parametrize("flags", [0, GEN], ids=["tma", "plain"])
@pytest.mark.parametrize("t", list(range(40)))
def test_fuzz_parity(t, flags):
    f, eb, mode, R = fuzz_case(t)
    if mode == "rel" and np.ptp(f) == 0:
        pytest.skip("constant field")
    check(f, eb, mode, R, flags)


# rows of a multiple of 4 but not of 8 values (c2's 500): no TMA map for the codes, so the quantiser takes the
# 8-byte plain slab store and the f32 decompressor the shared-memory staged kernel (k_decompress_staged)
@pytest.mark.parametrize("two_pass", [False, True], ids=["fused", "two-pass"])
@pytest.mark.parametrize("dims", [(13, 17, 100), (7, 50, 292), (6, 6, 4), (1, 1, 500), (25, 8, 196), (12, 7, 12)])
@pytest.mark.parametrize("R", [32768, 8])
def test_rows_multiple_of_4_not_8(dims, R, two_pass):
    rng = np.random.default_rng(abs(hash((dims, R))) % (1 << 31))
    f = np.cumsum(rng.normal(size=dims), axis=-1).astype(np.float32)
    check(f, 1e-3, "rel", R, 0, two_pass=two_pass)


# ----------------------------------------------------------------------------- two-pass (analyze -> quantize)
def assert_same_outputs(a: dict, b: dict):
    """Bit-identical compression outputs (outliers compared as sets keyed by index)."""
    for k in ("codes", "coef_codes", "hist"):
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(a["coef_raw"].view(np.uint64), b["coef_raw"].view(np.uint64)), "beta"
    assert a["eb_abs"] == b["eb_abs"]
    oa, ob = np.argsort(a["outlier_idx"]), np.argsort(b["outlier_idx"])
    assert np.array_equal(a["outlier_idx"][oa], b["outlier_idx"][ob])
    assert np.array_equal(a["outlier_val"][oa].view(np.uint8), b["outlier_val"][ob].view(np.uint8))


@pytest.mark.parametrize("flags", [0, GEN], ids=["tma", "plain"])
@pytest.mark.parametrize("t", list(range(0, 40, 3)))
def test_two_pass_matches_fused(t, flags):
    """analyze + quantize reproduce the fused kernel bit for bit (beta, codes, histogram, outliers),
    and the analyze pass's range equals sz3g_value_range."""
    f, eb, mode, R = fuzz_case(t)
    if mode == "rel" and np.ptp(f) == 0:
        pytest.skip("constant field")
    x = torch.from_numpy(np.ascontiguousarray(f)).cuda()
    fused, xo_f, _ = run_gpu(x, eb, mode, R, flags)
    two, xo_t, _ = run_gpu(x, eb, mode, R, flags, two_pass=True)
    assert_same_outputs(fused, two)
    assert np.array_equal(xo_f.view(np.uint8), xo_t.view(np.uint8))
    mm, _ = sz().regression_analyze(x)
    assert torch.equal(mm, sz().value_range(x))


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_two_pass_config_parity(name):
    """The two-pass path against the oracle at full size (the bench's REL path)."""
    from synth import config_by_name, make_field
    cfg = config_by_name(name)
    x = make_field(cfg, device="cuda")
    rep = check(x.cpu().numpy(), cfg.eb, cfg.eb_mode, cfg.radius, two_pass=True)
    assert rep["exempt_blocks"] <= max(4, oracle.num_blocks(tuple(x.shape)) // 10000)


def test_two_pass_nonfinite_range():
    s = sz()
    f = np.linspace(-3, 3, 13 * 14 * 96, dtype=np.float32).reshape(13, 14, 96)
    f[1, 2, 3] = np.nan
    x = torch.from_numpy(f).cuda()
    mm, _ = s.regression_analyze(x)
    assert math.isnan(float(mm[1]))
    with pytest.raises(Exception):
        s.compress(x, 1e-3, "rel", two_pass=True)


# ----------------------------------------------------------------------------- configs at full size
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_config_full_size(name):
    from synth import config_by_name, make_field
    cfg = config_by_name(name)
    x = make_field(cfg, device="cuda")
    xh = x.cpu().numpy()
    rep = check(xh, cfg.eb, cfg.eb_mode, cfg.radius)
    print(name, rep)
    # blocks exempt as coefficient near-ties: the window width is set by the 1e-12 beta tolerance, so
    # expect ~ 8 * window * NB of them (a few per 10^5 blocks on c4); none may be a real mismatch beyond
    nb = oracle.num_blocks(xh.shape)
    assert rep["exempt_blocks"] <= max(4, nb // 10000)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_config_plain_path(name):
    from synth import config_by_name, make_field
    cfg = config_by_name(name)
    xh = make_field(cfg, device="cuda").cpu().numpy()
    check(xh, cfg.eb, cfg.eb_mode, cfg.radius, GEN)


# ----------------------------------------------------------------------------- edge cases
@pytest.mark.parametrize("flags", [0, GEN], ids=["tma", "plain"])
def test_degenerate_extents(flags):
    rng = np.random.default_rng(5)
    for dims in [(1, 1, 1), (1, 1, 7), (1, 7, 1), (7, 1, 1), (1, 6, 96), (6, 1, 100), (2, 2, 2)]:
        f = rng.normal(size=dims).astype(np.float32)
        check(f, 0.01, "abs", 32768, flags)


@pytest.mark.parametrize("flags", [0, GEN], ids=["tma", "plain"])
def test_nonfinite_inputs(flags):
    f = np.linspace(-3, 3, 13 * 14 * 96, dtype=np.float32).reshape(13, 14, 96)
    f[1, 2, 3] = np.nan
    f[12, 13, 95] = np.inf
    f[6, 6, 50] = -np.inf
    rep = check(f, 1e-3, "abs", 32768, flags)
    assert rep["counters"]["nonfinite_outliers"] == 3
    x = torch.from_numpy(f).cuda()
    with pytest.raises(Exception):
        sz().compress(x, 1e-3, "rel")   # bad range (status bit 1)


@pytest.mark.parametrize("flags", [0, GEN], ids=["tma", "plain"])
def test_checkerboard_ties_and_linear_field(flags):
    dims = (12, 18, 96)
    i, j, k = np.meshgrid(*[np.arange(n) for n in dims], indexing="ij")
    f = ((-1.0) ** (i + j + k)).astype(np.float32)
    rep = check(f, 1.0, "abs", 32768, flags)
    assert rep["counters"]["elem_near_ties"] == f.size
    g = (0.5 + 0.25 * i - 0.125 * j + 0.0625 * k).astype(np.float32)
    x = torch.from_numpy(g).cuda()
    res = sz().compress(x, 1e-2, "rel")
    assert bool((res.codes.long() == 32768).all())


def test_outlier_overflow_and_small_radius():
    rng = np.random.default_rng(3)
    f = rng.normal(size=(24, 24, 96)).astype(np.float32)
    x = torch.from_numpy(f).cuda()
    with pytest.raises(Exception, match="capacity"):
        sz().compress(x, 1e-4, "rel", radius=4, outlier_cap=10)
    rep = check(f, 1e-3, "rel", 4)
    assert rep["outliers"] > 1000


def test_invalid_arguments():
    s = sz()
    x = torch.zeros((0, 4, 4), device="cuda")
    with pytest.raises(Exception):
        s.compress(x, 1e-3, "abs")
    y = torch.ones((6, 6, 6), device="cuda")
    with pytest.raises(Exception):
        s.compress(y, -1.0, "abs")
    with pytest.raises(Exception):
        s.compress(y, 1e-3, "abs", radius=40000)


def test_value_range_and_histogram_standalone():
    s = sz()
    rng = np.random.default_rng(0)
    for dt in (np.float32, np.float64):
        f = rng.normal(size=(37, 11, 7)).astype(dt)
        mm = s.value_range(torch.from_numpy(f).cuda()).cpu().numpy()
        assert mm[0] == f.min() and mm[1] == f.max()
    for R in (1, 4, 100, 32768):
        codes = rng.integers(0, 2 * R, size=1_000_003).astype(np.uint16)
        h = s.histogram(torch.from_numpy(codes).cuda(), R).cpu().numpy()
        assert np.array_equal(h, np.bincount(codes, minlength=2 * R))


def test_gpu_slab_invariance():
    """Block-aligned slabs with dim0_offset and the global range reproduce the whole-field output."""
    s = sz()
    from synth import make_field
    x = make_field("c2", device="cuda", shape=(48, 64, 96))
    whole = s.compress(x, 1e-4, "rel", coef_raw=False)
    mm = s.value_range(x)
    codes, hist = [], torch.zeros_like(whole.hist)
    for a, b in [(0, 12), (12, 30), (30, 48)]:
        part = s.regression_compress(x[a:b].contiguous(), 1e-4, "rel", d_minmax=mm, dim0_offset=a)
        part.finalize()
        codes.append(part.codes.clone())
        hist += part.hist
    assert torch.equal(torch.cat(codes), whole.codes)
    assert torch.equal(hist, whole.hist)


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_repeat_determinism_full_size(name):
    """Back-to-back launches (the bench's pattern) must give bit-identical outputs every time.
    Catches pipeline races that a single parity run can miss."""
    from synth import config_by_name, make_field
    s = sz()
    cfg = config_by_name(name)
    x = make_field(cfg, device="cuda")
    bufs = s.CompressBuffers(x.shape, x.dtype, cfg.radius, device=x.device, coef_raw=True)
    ref = s.regression_compress(x, cfg.eb, cfg.eb_mode, cfg.radius, bufs=bufs, coef_raw=True).finalize()
    codes0, coef0, hist0, raw0 = ref.codes.clone(), ref.coef_codes.clone(), ref.hist.clone(), ref.coef_raw.clone()
    xo0 = s.decompress(ref).clone()
    out = torch.empty_like(x)
    for _ in range(20):
        r = s.regression_compress(x, cfg.eb, cfg.eb_mode, cfg.radius, bufs=bufs, coef_raw=True)
        s.regression_decompress(r.codes, r.coef_codes, r.outlier_idx, r.outlier_val, ref.n_outliers, ref.eb_abs,
                                cfg.radius, x.dtype, out=out)
    torch.cuda.synchronize()
    r.finalize()
    assert torch.equal(r.codes, codes0) and torch.equal(r.coef_codes, coef0) and torch.equal(r.hist, hist0)
    assert torch.equal(r.coef_raw, raw0)
    assert torch.equal(out.view(torch.int32 if x.dtype == torch.float32 else torch.int64),
                       xo0.view(torch.int32 if x.dtype == torch.float32 else torch.int64))


# ----------------------------------------------------------------------------- fast-path boundaries
def adversarial_case(kind):
    rng = np.random.default_rng(77)
    dims = (12, 18, 96)
    i, j, k = np.meshgrid(*[np.arange(n) for n in dims], indexing="ij")
    if kind == "half_bins":        # linear field + checkerboard of +-3.5 bins: moments unchanged, t = +-3.5 exactly
        eb = 2.0 ** -6
        f = 0.25 * i - 0.125 * j + 0.0625 * k + ((-1.0) ** (i + j + k)) * 3.5 * 2 * eb
        return f.astype(np.float32), eb, "abs", 32768
    if kind == "near_half":        # half-bins +- a few ulps
        eb = 2.0 ** -6
        f = (0.25 * i + (rng.integers(-40, 40, size=dims) + 0.5) * 2 * eb).astype(np.float32)
        f = np.nextafter(f, np.where(rng.random(dims) < 0.5, np.inf, -np.inf).astype(np.float32))
        return f.astype(np.float32), eb, "abs", 32768
    if kind == "offset":           # large offset: the fp32 bound rejects most elements
        return (1e6 + rng.normal(size=dims) * 0.5).astype(np.float32), 1e-3, "abs", 32768
    if kind == "float_resolution": # eb below half an f32 ulp of the data: x' rounding fails the verify
        return (100 + 0.01 * np.sin(0.3 * i + 0.2 * j + 0.1 * k) + 1e-4 * rng.normal(size=dims)).astype(np.float32), \
            5e-6, "abs", 32768   # ulp(100)/2 < eb < ulp(100)
    if kind == "denormal":
        return (rng.normal(size=dims) * 1e-39).astype(np.float32), 1e-41, "abs", 32768
    if kind == "huge_eb":
        return (rng.normal(size=dims) * 1e30).astype(np.float32), 1e31, "abs", 16
    if kind == "wide_range":       # heavy tails, REL eb, small radius
        return np.exp(4 * rng.normal(size=dims)).astype(np.float32), 1e-4, "rel", 256
    raise ValueError(kind)


@pytest.mark.parametrize("flags", [0, GEN], ids=["tma", "plain"])
@pytest.mark.parametrize("kind", ["half_bins", "near_half", "offset", "float_resolution", "denormal", "huge_eb",
                                  "wide_range"])
def test_fast_path_boundaries(kind, flags):
    f, eb, mode, R = adversarial_case(kind)
    rep = check(f, eb, mode, R, flags)
    if kind == "half_bins":
        assert rep["counters"]["elem_near_ties"] == f.size
    if kind == "float_resolution":
        assert rep["counters"]["verify_outliers"] > 0
