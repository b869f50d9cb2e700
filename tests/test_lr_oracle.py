"""Pins of the SZ3-LR oracle (NEXT-4; oracle/DEFINITION.md L1-L7, DESIGN G26-G29) against what the
definition and the mathematics fix, not against itself:

* L2 against numpy's own finite differences (np.diff of the zero-padded block along each axis);
* closed-form Lorenzo residuals of f = i + 2j + 3k + 5ijk tiled per block (eb = 0.5, so q = x exactly):
  delta = 0 at the origin, 1 / 2 / 3 on the three axes, 0 on the faces, 5 inside -- on full and
  ragged blocks, f32 and f64;
* the block choice against the closed-form Lorenzo cost and the independent regression oracle's codes;
* a linear field (regression exact): every block regression, and the output equal to the regression
  oracle's (codes, coefficient codes, outliers, histogram);
* a step inside the block: Lorenzo chosen, a single residual of 1000 (a radius outlier when R <= 1000);
* integer fields through Lorenzo blocks reconstruct exactly; random fields with NaN / Inf / huge values
  round-trip within eb (outliers exact) and decompression reproduces the compress-time x'."""
from __future__ import annotations

import numpy as np
import pytest

import oracle

R_BIG = 32768


def tiled(shape, f, dtype=np.float64):
    i, j, k = np.meshgrid(*(np.arange(n) % 6 for n in shape), indexing="ij")
    return f(i, j, k).astype(dtype)


def poly(i, j, k):
    return i + 2 * j + 3 * k + 5 * i * j * k


def closed_delta(i, j, k):
    nz = (i > 0).astype(int) + (j > 0) + (k > 0)
    d = np.zeros(np.broadcast(i, j, k).shape, np.int64)
    d = np.where((nz == 1) & (i > 0), 1, d)
    d = np.where((nz == 1) & (j > 0), 2, d)
    d = np.where((nz == 1) & (k > 0), 3, d)
    d = np.where(nz == 3, 5, d)
    return d


def blocks_of(shape):
    nb = [-(-n // 6) for n in shape]
    for a in range(nb[0]):
        for b in range(nb[1]):
            for c in range(nb[2]):
                yield (a * nb[1] + b) * nb[2] + c, (slice(6 * a, 6 * a + 6), slice(6 * b, 6 * b + 6),
                                                    slice(6 * c, 6 * c + 6))


def cost(codes, R):
    c = codes.astype(np.int64)
    return int(np.where(c == 0, R, np.abs(c - R)).sum())


def test_delta_matches_numpy_differences():
    rng = np.random.default_rng(0)
    for shape in [(6, 6, 6), (3, 5, 4), (1, 6, 2), (6, 1, 1)]:
        q = rng.integers(-10 ** 9, 10 ** 9, size=shape)
        d = np.pad(q, ((1, 0), (1, 0), (1, 0)))
        for ax in range(3):
            d = np.diff(d, axis=ax)
        for i, j, k in np.ndindex(*shape):
            assert oracle.lr_delta(q, i, j, k) == d[i, j, k]


@pytest.mark.parametrize("shape,dtype", [((12, 12, 18), np.float64), ((14, 13, 17), np.float32),
                                         ((6, 6, 6), np.float32)])
def test_closed_form_residuals_and_choice(shape, dtype):
    x = tiled(shape, poly, dtype)
    c = oracle.lr_compress(x, 0.5, "abs", R_BIG)
    reg = oracle.compress(x, 0.5, "abs", R_BIG)
    i, j, k = np.meshgrid(*(np.arange(n) % 6 for n in shape), indexing="ij")
    delta = closed_delta(i, j, k)
    for bid, sl in blocks_of(shape):
        cl = cost((delta[sl] + R_BIG), R_BIG)
        cr = cost(reg.codes[sl], R_BIG)
        assert c.flags[bid] == (1 if cl < cr else 0), (bid, cl, cr)
        if c.flags[bid]:
            assert np.array_equal(c.codes[sl].astype(np.int64), delta[sl] + R_BIG)
            assert not c.coef_codes[bid].any()
        else:
            assert np.array_equal(c.codes[sl], reg.codes[sl])
            assert np.array_equal(c.coef_codes[bid], reg.coef_codes[bid])
    assert c.n_lorenzo == int(c.flags.sum()) > 0
    y = oracle.lr_decompress(c)
    lor = np.zeros(shape, bool)
    for bid, sl in blocks_of(shape):
        lor[sl] = c.flags[bid] == 1
    assert np.array_equal(y[lor], x[lor])          # q = x exactly (2eb = 1): exact reconstruction
    assert np.abs(y.astype(np.float64) - x).max() <= 0.5


def test_linear_field_is_all_regression_and_equals_regression_oracle():
    shape = (13, 20, 31)
    i, j, k = np.meshgrid(*(np.arange(n) for n in shape), indexing="ij")
    x = (3.0 + 0.25 * i - 0.5 * j + 0.125 * k).astype(np.float64)
    c = oracle.lr_compress(x, 1e-3, "abs", 1024)
    reg = oracle.compress(x, 1e-3, "abs", 1024)
    assert c.n_lorenzo == 0 and not c.flags.any()
    assert np.array_equal(c.codes, reg.codes)
    assert np.array_equal(c.coef_codes, reg.coef_codes)
    assert np.array_equal(c.hist, reg.hist)
    assert np.array_equal(c.outlier_idx, reg.outlier_idx)
    assert np.array_equal(oracle.lr_decompress(c), oracle.decompress(reg))


@pytest.mark.parametrize("R", [R_BIG, 1000, 64])
def test_step_inside_block(R):
    shape = (6, 12, 12)
    x = tiled(shape, lambda i, j, k: 1000.0 * (k >= 3), np.float32)
    c = oracle.lr_compress(x, 0.5, "abs", R)
    assert c.flags.all()
    i, j, k = np.meshgrid(*(np.arange(n) % 6 for n in shape), indexing="ij")
    jump = (i == 0) & (j == 0) & (k == 3)
    if R > 1000:
        assert np.array_equal(c.codes.astype(np.int64), np.where(jump, R + 1000, R))
        assert len(c.outlier_idx) == 0
    else:   # the jump is a radius outlier: stored, and its q still feeds its neighbours
        assert np.array_equal(c.codes == 0, jump)
        assert np.array_equal(np.sort(c.outlier_idx), np.flatnonzero(jump.ravel()).astype(np.uint64))
        assert np.all(c.codes[~jump] == R)
    assert np.array_equal(oracle.lr_decompress(c), x)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_round_trip_with_specials(dtype):
    rng = np.random.default_rng(5)
    shape = (17, 23, 29)
    i, j, k = np.meshgrid(*(np.arange(n, dtype=np.float64) for n in shape), indexing="ij")
    curved = np.sin(i / 3.0) * np.cos(j / 5.0) + 0.01 * (k - 14) ** 2     # Lorenzo's blocks
    noisy = 0.1 * i - 0.05 * j + 0.02 * k + 1e-3 * rng.standard_normal(shape)  # regression's blocks
    x = np.where(i < 12, curved, noisy).astype(dtype)
    flat = x.reshape(-1)
    pos = rng.choice(flat.size, 40, replace=False)
    flat[pos[:10]] = np.nan
    flat[pos[10:20]] = np.inf
    flat[pos[20:30]] = -np.inf
    flat[pos[30:]] = 1e30 if dtype == np.float32 else 1e300
    c = oracle.lr_compress(x, 1e-4, "abs", 4096)
    assert 0 < c.n_lorenzo < c.flags.size
    y = oracle.lr_decompress(c)
    assert np.array_equal(y.view(np.uint8), c.xprime.view(np.uint8))
    out = np.zeros(flat.size, bool)
    out[c.outlier_idx.astype(np.int64)] = True
    assert out[pos].all()
    yo, xo = y.reshape(-1), flat
    assert np.array_equal(yo[out].view(np.uint8), xo[out].view(np.uint8))
    assert np.abs(yo[~out].astype(np.float64) - xo[~out].astype(np.float64)).max() <= 1e-4
    h = np.bincount(c.codes.reshape(-1), minlength=2 * 4096)
    assert np.array_equal(h, c.hist)
    assert h[0] == len(c.outlier_idx)
