"""SZ3-Interp on the GPU (csrc/interp.cu through the C ABI) against the oracle (DEFINITION.md I1-I6),
element by element: codes, outlier sets (global indices), histogram and the compress-time reconstruction
bit-exact; decompression bit-exact against both the compress-time x' and the oracle's decompression; the
bound everywhere.  Fuzzed shapes (degenerate, ragged, 1-wide axes), both dtypes, ABS / REL, radii down to
1, and the configs at full size."""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402

pytestmark = pytest.mark.gpu


def sz():
    from paper_2111_02925_b200 import sz3g
    sz3g.load()
    return sz3g


def check(f: np.ndarray, eb: float, mode: str, R: int):
    s = sz()
    x = torch.from_numpy(np.ascontiguousarray(f)).cuda()
    res = s.interp_compress(x, eb, mode, R, outlier_cap=x.numel()).finalize()
    xo = s.interp_decompress(res.codes, res.outlier_idx, res.outlier_val, res.outlier_idx.numel(), res.eb_abs, R,
                             x.dtype, d_outlier_count=res.outlier_count)
    torch.cuda.synchronize()
    orc = oracle.interp_compress(f, eb, mode, radius=R)
    assert res.eb_abs == orc.eb_abs
    n = res.n_outliers
    assert np.array_equal(res.codes.cpu().numpy(), orc.codes)
    gi = res.outlier_idx[:n].cpu().numpy().view(np.uint64)
    gv = res.outlier_val[:n].cpu().numpy()
    o = np.argsort(gi)
    oo = np.argsort(orc.outlier_idx)
    assert np.array_equal(gi[o], orc.outlier_idx[oo])
    assert np.array_equal(gv[o].view(np.uint8), orc.outlier_val[oo].view(np.uint8))
    assert np.array_equal(res.hist.cpu().numpy(), orc.hist)
    xp = res.xprime.cpu().numpy()
    assert np.array_equal(xp.view(np.uint8), orc.xprime.view(np.uint8))
    xd = xo.cpu().numpy()
    assert np.array_equal(xd.view(np.uint8), xp.view(np.uint8))
    od = oracle.interp_decompress(dims=orc.dims, dtype=f.dtype, radius=R, eb_abs=orc.eb_abs, codes=orc.codes,
                                  outlier_idx=orc.outlier_idx, outlier_val=orc.outlier_val)
    assert np.array_equal(od.view(np.uint8), xd.reshape(od.shape).view(np.uint8))
    fin = np.isfinite(f)
    assert (np.abs(xd.reshape(f.shape).astype(np.float64)[fin] - f.astype(np.float64)[fin]) <= orc.eb_abs).all()
    return orc


def case(t):
    rng = np.random.default_rng(7000 + t)
    shapes = [(13, 17, 96), (1, 1, 500), (3, 40, 8), (12, 12, 12), (40, 1, 36), (1, 37, 1), (33, 9, 65), (1, 1, 1),
              (2, 3, 2), (64, 64, 64)]
    dims = shapes[t % len(shapes)] if t < 20 else tuple(int(v) for v in rng.integers(1, 41, size=3))
    dtype = [np.float32, np.float64][t % 2]
    mode = ["abs", "rel"][(t // 2) % 2]
    R = [32768, 4, 64, 1][(t // 3) % 4]
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


@pytest.mark.parametrize("t", list(range(32)))
def test_interp_fuzz_parity(t):
    f, eb, mode, R = case(t)
    if mode == "rel" and np.ptp(f) == 0:
        pytest.skip("constant field")
    check(f, eb, mode, R)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_interp_config_parity(name):
    from synth import config_by_name, make_field
    cfg = config_by_name(name)
    f = make_field(cfg, device="cuda").cpu().numpy()
    orc = check(f, cfg.eb, cfg.eb_mode, cfg.radius)
    print(name, "outliers", orc.outlier_idx.size, orc.counters)


def test_interp_nonfinite_and_multilinear():
    f = np.linspace(-3, 3, 13 * 14 * 96, dtype=np.float32).reshape(13, 14, 96)
    f[1, 2, 3] = np.nan
    f[12, 13, 95] = np.inf
    check(f, 1e-3, "abs", 32768)
    dims = (9, 17, 33)
    i, j, k = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in dims], indexing="ij")
    g = (0.5 + 0.25 * i - 0.125 * j + 0.0625 * k + 0.03125 * i * j).astype(np.float32)
    orc = check(g, 1e-3, "abs", 32768)
    assert int((orc.codes == 32768).sum()) == g.size - 10   # anchor + the 9 copy targets
