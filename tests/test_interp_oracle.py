"""Pins of the SZ3-Interp oracle (oracle/DEFINITION.md I1-I6; "Both linear
interpolation and cubic spline interpolation are included"; the plan / boundary readings G30-G33 follow
SPEC S:161-165).  Each pin checks the oracle against something it does not compute
itself: SPEC's worked examples, exactness of the interpolation weights on polynomials, the coverage and
causality of the level plan by brute force over every index, exact multilinear fields (every code in the
zero bin), and the contract invariants (bound, round trip, histogram)."""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle


# ----------------------------------------------------------------------------- I3
def test_i3_spec_examples():
    assert oracle.interp_predict(0, 2.0, 4.0, 0, 1) == 3.0                    # linear midpoint
    assert oracle.interp_predict(-27.0, -1.0, 1.0, 27.0, 2) == 0.0            # t^3 at -3,-1,1,3 -> g(0) = 0
    assert oracle.interp_predict(7.25, 7.25, 7.25, 7.25, 2) == 7.25           # weights sum to 1
    assert oracle.interp_predict(1.0, 5.5, 9.0, 2.0, 0) == 5.5                # copy of the -s donor


@pytest.mark.parametrize("seed", range(20))
def test_i3_cubic_weights_exact_on_cubics(seed):
    """The cubic spline weights (-1, 9, 9, -1)/16 reproduce g(0) for every cubic g sampled at
    -3, -1, 1, 3 (dyadic coefficients: every intermediate is exact, so equality is exact)."""
    rng = np.random.default_rng(seed)
    a, b, c, d = (float(v) for v in rng.integers(-64, 64, size=4) / 8.0)
    g = lambda t: a + b * t + c * t * t + d * t * t * t   # noqa: E731
    assert oracle.interp_predict(g(-3), g(-1), g(1), g(3), 2) == g(0)
    # and the linear weights on lines
    assert oracle.interp_predict(0, a + b * -1, a + b * 1, 0, 1) == a


# ----------------------------------------------------------------------------- I2: plan coverage
@pytest.mark.parametrize("dims", [(1, 1, 1), (1, 1, 9), (3, 5, 7), (8, 8, 8), (9, 1, 17), (6, 13, 2), (16, 3, 33)])
def test_i2_every_index_once_and_donors_earlier(dims):
    n0, n1, n2 = dims
    S = 0
    m = max(dims)
    if m > 1:
        S = 1 << (math.ceil(math.log2(m)) - 1)
    passes = np.empty(dims, np.int64)
    for i in range(n0):
        for j in range(n1):
            for k in range(n2):
                passes[i, j, k] = oracle.interp_pass_of(dims, i, j, k)
    assert passes[0, 0, 0] == -1 and (passes.reshape(-1)[1:] >= 0).all()
    # causality: the +-s donors along the pass axis (and +-3s when they exist) come from earlier passes
    for i in range(n0):
        for j in range(n1):
            for k in range(n2):
                p = passes[i, j, k]
                if p < 0:
                    continue
                level, axis = divmod(int(p), 3)
                s = S >> level
                idx = [i, j, k]
                assert idx[axis] % (2 * s) == s
                for off in (-3 * s, -s, s, 3 * s):
                    q = list(idx)
                    q[axis] += off
                    if 0 <= q[axis] < dims[axis]:
                        assert passes[tuple(q)] < p, (dims, idx, off)


# ----------------------------------------------------------------------------- exact fields
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_multilinear_field_zero_codes_except_copies(dtype):
    """A field that is linear along every axis line (trilinear, dyadic coefficients, exact in f32):
    every cubic and linear interpolation is exact, so the only nonzero residuals are at the anchor and at
    the copy targets (no +s donor, I3), which the plan puts at index + s >= extent.  A wrong weight, sign
    or donor offset anywhere in I3 would leave codes off the zero bin at the interpolated targets."""
    dims = (9, 17, 33)
    i, j, k = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in dims], indexing="ij")
    f = (0.5 + 0.25 * i - 0.125 * j + 0.0625 * k + 0.03125 * i * j - 0.015625 * j * k + 0.0078125 * i * j * k)
    f = f.astype(dtype)
    c = oracle.interp_compress(f, 1e-3, "abs", radius=32768)
    S = 32
    copies = 0
    for a in range(dims[0]):
        for b in range(dims[1]):
            for d in range(dims[2]):
                p = oracle.interp_pass_of(dims, a, b, d)
                if p < 0:
                    assert c.codes[a, b, d] == 0
                    continue
                level, axis = divmod(p, 3)
                s = S >> level
                if (a, b, d)[axis] + s >= dims[axis]:
                    copies += 1
                    continue
                assert c.codes[a, b, d] == 32768, (a, b, d)
    assert copies == 9                      # 6 at level 8 (axis 0), 2 at level 16 (axis 1), 1 at level 32
    assert c.outlier_idx.tolist() == [0]
    assert (np.abs(c.xprime.astype(np.float64) - f) <= c.eb_abs).all()


def test_constant_and_degenerate_fields():
    c = oracle.interp_compress(np.full((5, 7, 6), 3.25, np.float32), 1e-2, "abs")
    assert (c.codes.reshape(-1)[1:] == 32768).all() and c.outlier_idx.tolist() == [0]
    one = oracle.interp_compress(np.array([[[1.5]]], np.float64), 1e-3, "abs")
    assert one.codes.tolist() == [[[0]]] and one.outlier_val.tolist() == [1.5]


# ----------------------------------------------------------------------------- invariants (P3 analogue)
@pytest.mark.parametrize("case", range(24))
def test_bound_round_trip_histogram(case):
    rng = np.random.default_rng(500 + case)
    dims = tuple(int(v) for v in rng.integers(1, 30, size=3))
    dtype = [np.float32, np.float64][case % 2]
    kind = case % 3
    if kind == 0:
        f = rng.normal(size=dims)
    elif kind == 1:
        f = np.cumsum(np.cumsum(rng.normal(size=dims), axis=-1), axis=0)
    else:
        f = np.exp(2 * rng.normal(size=dims))
    f = f.astype(dtype)
    R = [32768, 8, 64][(case // 3) % 3]
    mode = ["abs", "rel"][(case // 2) % 2]
    eb = float(rng.choice([1e-1, 1e-3, 1e-5]))
    if mode == "abs":
        eb *= float(np.ptp(f) + 1e-3)
    if mode == "rel" and np.ptp(f) == 0:
        pytest.skip("constant")
    c = oracle.interp_compress(f, eb, mode, radius=R)
    err = np.abs(c.xprime.astype(np.float64) - f.astype(np.float64))
    assert (err <= c.eb_abs).all()
    back = oracle.interp_decompress(c)
    assert np.array_equal(back.view(np.uint8), c.xprime.view(np.uint8))
    assert int(c.hist.sum()) == f.size and int(c.hist[0]) == c.outlier_idx.size
    assert c.outlier_idx[0] == 0 and (c.codes < 2 * R).all()
    # an outlier's reconstruction is its value, every other element carries a nonzero code
    z = c.codes.reshape(-1) == 0
    assert np.array_equal(np.sort(c.outlier_idx), np.flatnonzero(z).astype(np.uint64))


def test_sign_symmetry():
    """Every step is odd under round-to-nearest-even: compress(-x) negates q (code c -> 2R - c) and
    the outlier values (P4 analogue)."""
    rng = np.random.default_rng(9)
    f = np.cumsum(rng.normal(size=(12, 10, 20)), axis=2).astype(np.float32)
    a = oracle.interp_compress(f, 1e-2, "abs", radius=64)
    b = oracle.interp_compress(-f, 1e-2, "abs", radius=64)
    ca, cb = a.codes.astype(np.int64), b.codes.astype(np.int64)
    nz = ca != 0
    assert np.array_equal(nz, cb != 0) and np.array_equal(cb[nz], 128 - ca[nz])
    assert np.array_equal(a.outlier_idx, b.outlier_idx) and np.array_equal(a.outlier_val, -b.outlier_val)
