"""Pins for the CPU oracle (oracle/) against what the paper and the mathematics fix -- never against
the oracle itself.  CPU only.

P1  Lemma 1 vs brute-force least squares: Gaussian elimination on the normal equations of
    Eq. (betasol) (system P:76-97), exact rationals for integer data, numpy lstsq, and the
    paper's own reduced system.
P2  exact linear fields: coefficients recovered, every quantisation code is the zero bin.
P3  contract invariants: |x - x'| <= eb, round trip, histogram sums.
P4  sign symmetry, P5 power-of-two scaling, P7 checkerboard ties, P8 slab invariance,
P9  radius outliers only where |x - p| >= (2R - 1) eb.
P6  worked examples printed in SPEC.md (tests/golden/spec_examples.json).
"""
from __future__ import annotations

import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")
R16 = 32768


# ----------------------------------------------------------------------------- helpers (independent)
def design_matrix(m0, m1, m2):
    """X of Eq. (betasol): rows x' = (1, i, j, k), y ordered f_000, f_001, ... (k fastest)."""
    rows = [(1, i, j, k) for i in range(m0) for j in range(m1) for k in range(m2)]
    return np.array(rows, dtype=np.float64)


def gauss_solve(A, b):
    """Plain Gaussian elimination with partial pivoting (works on floats or Fractions)."""
    n = len(b)
    M = [list(A[r]) + [b[r]] for r in range(n)]
    for col in range(n):
        piv = max(range(col, n), key=lambda r: abs(M[r][col]))
        M[col], M[piv] = M[piv], M[col]
        for r in range(col + 1, n):
            f = M[r][col] / M[col][col]
            for c in range(col, n + 1):
                M[r][c] = M[r][c] - f * M[col][c]
    x = [0] * n
    for r in range(n - 1, -1, -1):
        s = M[r][n]
        for c in range(r + 1, n):
            s = s - M[r][c] * x[c]
        x[r] = s / M[r][r]
    return x


def ls_normal_equations(f, exact=False):
    """beta' = (X^T X)^-1 X^T y by GE on the normal equations; extent-1 axes dropped (slope 0, G2)."""
    m = f.shape
    X = design_matrix(*m)
    keep = [0] + [d + 1 for d in range(3) if m[d] > 1]
    Xk = X[:, keep]
    y = f.reshape(-1)
    if exact:
        Xf = [[Fraction(int(v)) for v in row] for row in Xk]
        yf = [Fraction(int(v)) for v in y]
        A = [[sum(Xf[r][a] * Xf[r][b] for r in range(len(Xf))) for b in range(len(keep))] for a in range(len(keep))]
        rhs = [sum(Xf[r][a] * yf[r] for r in range(len(Xf))) for a in range(len(keep))]
    else:
        A = (Xk.T @ Xk).tolist()
        rhs = (Xk.T @ y).tolist()
    sol = gauss_solve(A, rhs)
    beta = [Fraction(0) if exact else 0.0] * 4
    for idx, col in enumerate(keep):
        beta[col] = sol[idx]
    return beta


def random_block(rng, exts, kind):
    if kind == "normal":
        return rng.normal(size=exts) * rng.uniform(0.1, 100)
    if kind == "offset":   # large intercept, small slopes: cancellation-prone
        return 1e6 + rng.normal(size=exts) * 1e-3
    if kind == "int":
        return rng.integers(-1000, 1000, size=exts).astype(np.float64)
    raise ValueError(kind)


def local_prediction(bhat, m):
    i = np.arange(m[0]).reshape(-1, 1, 1)
    j = np.arange(m[1]).reshape(1, -1, 1)
    k = np.arange(m[2]).reshape(1, 1, -1)
    return bhat[0] + i * bhat[1] + j * bhat[2] + k * bhat[3]


def blocks_of(dims, B=6):
    n0, n1, n2 = dims
    for a in range(math.ceil(n0 / B)):
        for b in range(math.ceil(n1 / B)):
            for c in range(math.ceil(n2 / B)):
                yield (a * B, min(a * B + B, n0)), (b * B, min(b * B + B, n1)), (c * B, min(c * B + B, n2))


# ----------------------------------------------------------------------------- P1
@pytest.mark.parametrize("kind", ["normal", "offset"])
def test_p1_lemma_matches_gaussian_elimination(kind):
    rng = np.random.default_rng(1234 if kind == "normal" else 99)
    worst = 0.0
    for _ in range(250):
        exts = tuple(int(e) for e in rng.integers(1, 7, size=3))
        f = random_block(rng, exts, kind)
        _, beta = oracle.block_beta(f)
        ref = ls_normal_equations(f)
        scale = max(np.mean(np.abs(f)), 1e-300)
        for d in range(4):
            err = abs(beta[d] - ref[d]) / max(abs(ref[d]), scale)
            worst = max(worst, err)
    # GE itself carries rounding error; the Lemma has to agree to ~1e-12 of the block scale (P1)
    assert worst < 1e-11, worst


def test_p1_lemma_matches_exact_rational_solution():
    rng = np.random.default_rng(7)
    worst = 0.0
    for _ in range(120):
        exts = tuple(int(e) for e in rng.integers(1, 7, size=3))
        f = random_block(rng, exts, "int")
        _, beta = oracle.block_beta(f)
        exact = ls_normal_equations(f, exact=True)
        scale = max(float(np.mean(np.abs(f))), 1.0)
        for d in range(4):
            err = abs(beta[d] - float(exact[d])) / max(abs(float(exact[d])), scale)
            worst = max(worst, err)
    assert worst < 1e-14, worst


def test_p1_lemma_matches_lstsq_and_reduced_system():
    """numpy lstsq (a library routine) and the paper's simplified 4x4 system."""
    rng = np.random.default_rng(11)
    for _ in range(100):
        exts = tuple(int(e) for e in rng.integers(2, 7, size=3))
        f = rng.normal(size=exts) * 3 + 1
        V, beta = oracle.block_beta(f)
        X = design_matrix(*exts)
        ref, *_ = np.linalg.lstsq(X, f.reshape(-1), rcond=None)
        np.testing.assert_allclose(beta, ref, rtol=0, atol=1e-12 * np.mean(np.abs(f)) * 10)
        n1, n2, n3 = exts
        N = n1 * n2 * n3
        A = np.array([
            [1, (n1 - 1) / 2, (n2 - 1) / 2, (n3 - 1) / 2],
            [1, (2 * n1 - 1) / 3, (n2 - 1) / 2, (n3 - 1) / 2],
            [1, (n1 - 1) / 2, (2 * n2 - 1) / 3, (n3 - 1) / 2],
            [1, (n1 - 1) / 2, (n2 - 1) / 2, (2 * n3 - 1) / 3]])
        rhs = np.array([V[0] / N, 2 * V[1] / (N * (n1 - 1)), 2 * V[2] / (N * (n2 - 1)), 2 * V[3] / (N * (n3 - 1))])
        np.testing.assert_allclose(A @ beta, rhs, rtol=0, atol=1e-12 * np.mean(np.abs(f)) * 10)
        # moments are the plain sums of P:62-64
        i, j, k = np.meshgrid(np.arange(n1), np.arange(n2), np.arange(n3), indexing="ij")
        np.testing.assert_allclose(V, [f.sum(), (i * f).sum(), (j * f).sum(), (k * f).sum()], rtol=1e-13, atol=1e-12)


def test_p99_sum_identities_and_normal_matrix():
    """P:99 identities, and X^T X of the design matrix equals the closed sums the proof uses."""
    g = json.load(open(GOLDEN))["identities"]
    for n in g["n"]:
        assert sum(range(n)) == n * (n - 1) // 2
        assert sum(i * i for i in range(n)) == (2 * n - 1) * n * (n - 1) // 6
    for exts in [(6, 6, 6), (4, 6, 2), (5, 3, 6)]:
        X = design_matrix(*exts)
        G = X.T @ X
        n1, n2, n3 = exts
        N = n1 * n2 * n3
        assert G[0, 0] == N
        assert G[0, 1] == N * (n1 - 1) / 2
        assert G[1, 1] == N * (2 * n1 - 1) * (n1 - 1) / 6
        assert G[1, 2] == N * (n1 - 1) * (n2 - 1) / 4


def test_p1_extent_one_axes_give_zero_slope():
    rng = np.random.default_rng(5)
    for exts in [(1, 6, 6), (6, 1, 6), (6, 6, 1), (1, 1, 6), (1, 1, 1)]:
        f = rng.normal(size=exts)
        _, beta = oracle.block_beta(f)
        for d in range(3):
            if exts[d] == 1:
                assert beta[d + 1] == 0.0
        ref = ls_normal_equations(f)
        np.testing.assert_allclose(beta, ref, rtol=0, atol=1e-12 * np.abs(f).mean() * 10)


# ----------------------------------------------------------------------------- P6 golden examples
def test_p6_spec_worked_examples():
    g = json.load(open(GOLDEN))
    for ex in g["coefficients"]:
        m = ex["extents"]
        i, j, k = np.meshgrid(*[np.arange(e) for e in m], indexing="ij")
        f = {"const": np.full(m, ex.get("value", 0.0)), "i": i * 1.0, "j": j * 1.0, "k": k * 1.0}[ex["field"]]
        _, beta = oracle.block_beta(f)
        np.testing.assert_allclose(beta, ex["beta"], rtol=0, atol=1e-13, err_msg=ex["cite"])
    for ex in g["predict"]:
        assert oracle.predict(ex["bhat"], *ex["ijk"]) == ex["p"], ex["cite"]
    for ex in g["quantize"]:
        dt = np.float32 if ex["dtype"] == "f32" else np.float64
        x = float(ex["x"])
        code, xp, kind = oracle.quantize_element(x, ex["p"], ex["eb"], ex["R"], dt)
        assert code == ex["code"], ex["cite"]
        assert kind == ex["kind"], ex["cite"]
        if ex["xprime"] == "nan":
            assert math.isnan(xp)
        else:
            assert abs(xp - float(ex["xprime"])) <= 2e-16 * max(1.0, abs(xp)), (ex["cite"], xp)
            if dt == np.float32:
                assert np.float32(xp) == np.float32(ex["xprime"])
        if kind == 0:
            assert abs(xp - x) <= ex["eb"], ex["cite"]
    for ex in g["tiling"]:
        assert oracle.num_blocks(ex["dims"], ex["B"]) == ex["nblocks"], ex["cite"]


# ----------------------------------------------------------------------------- P2 exact linear fields
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("dims", [(13, 17, 20), (6, 6, 6), (7, 12, 31)])
def test_p2_exact_linear_field(dtype, dims):
    rng = np.random.default_rng(sum(dims))
    a, b, c, d = (rng.integers(-512, 512, size=4) / 256.0)   # dyadic: exact in f32 and f64
    i, j, k = np.meshgrid(*[np.arange(n) for n in dims], indexing="ij")
    f = (a + b * i + c * j + d * k).astype(dtype)
    assert np.all(f.astype(np.float64) == a + b * i + c * j + d * k)
    res = oracle.compress(f, 1e-2, "rel")
    # coefficients recovered (north_star: 1e-12 relative), block-local intercept
    for bid, ((i0, i1), (j0, j1), (k0, k1)) in enumerate(blocks_of(dims)):
        want = np.array([a + b * i0 + c * j0 + d * k0, b, c, d])
        for ax, ext in enumerate((i1 - i0, j1 - j0, k1 - k0)):
            if ext == 1:
                want[ax + 1] = 0.0   # extent-1 axis: slope 0 (G2); the plane still fits exactly
        got = res.coef_raw[bid]
        assert np.all(np.abs(got - want) <= 1e-12 * np.maximum(np.abs(want), 1.0)), (bid, got, want)
    assert np.all(res.codes == res.radius), "all quantisation codes must be the zero bin (G1 bound)"
    assert res.outlier_idx.size == 0
    xr = oracle.decompress(res)
    assert np.all(np.abs(xr.astype(np.float64) - f.astype(np.float64)) <= res.eb_abs)


# ----------------------------------------------------------------------------- P3 invariants / fuzz
def fuzz_cases(n=40, seed=2024):
    rng = np.random.default_rng(seed)
    for t in range(n):
        dims = tuple(int(v) for v in rng.integers(1, 21, size=3))
        dtype = [np.float32, np.float64][t % 2]
        mode = ["abs", "rel"][(t // 2) % 2]
        R = [1, 4, 64, 32768][(t // 4) % 4]
        kind = t % 5
        if kind == 0:
            f = rng.normal(size=dims)
        elif kind == 1:
            f = np.cumsum(rng.normal(size=dims), axis=2)
        elif kind == 2:
            f = np.exp(2 * rng.normal(size=dims))
        elif kind == 3:
            f = rng.uniform(-1e4, 1e4, size=dims)
        else:
            f = np.sin(np.arange(np.prod(dims)).reshape(dims) * 0.1) + rng.normal(size=dims) * 1e-3
        eb = float(rng.choice([1e-1, 1e-2, 1e-3, 1e-5])) * (1.0 if mode == "rel" else float(np.ptp(f) + 1e-3))
        yield f.astype(dtype), eb, mode, R


@pytest.mark.parametrize("case", list(range(40)))
def test_p3_invariants_fuzz(case):
    f, eb, mode, R = list(fuzz_cases())[case]
    if mode == "rel" and np.ptp(f) == 0:
        pytest.skip("constant field in REL mode")
    res = oracle.compress(f, eb, mode, radius=R)
    N = f.size
    assert res.hist.sum() == N
    assert res.hist[0] == res.outlier_idx.size
    assert res.codes.max() < 2 * R
    assert np.array_equal(np.sort(res.outlier_idx), np.flatnonzero(res.codes.reshape(-1) == 0).astype(np.uint64))
    np.testing.assert_array_equal(np.bincount(res.codes.reshape(-1), minlength=2 * R), res.hist)
    xr = oracle.decompress(res)
    # strict bound everywhere (G8), checked in fp64
    assert np.all(np.abs(xr.astype(np.float64) - f.astype(np.float64)) <= res.eb_abs)
    # decompression reproduces the compress-time x' bit for bit
    assert np.array_equal(xr.view(np.uint8), res.xprime.view(np.uint8))
    # outliers are stored losslessly
    flat = f.reshape(-1)
    assert np.array_equal(res.outlier_val.view(np.uint8), flat[res.outlier_idx.astype(np.int64)].view(np.uint8))
    if mode == "rel":
        assert res.eb_abs == eb * (float(f.max()) - float(f.min()))


# ----------------------------------------------------------------------------- P4 sign symmetry
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_p4_sign_symmetry(dtype):
    rng = np.random.default_rng(3)
    f = (np.cumsum(rng.normal(size=(14, 19, 25)), axis=1) * 3).astype(dtype)
    for mode, eb, R in [("rel", 1e-3, 32768), ("abs", 0.05, 8)]:
        p = oracle.compress(f, eb, mode, radius=R)
        m = oracle.compress(-f, eb, mode, radius=R)
        assert np.array_equal(m.coef_codes, -p.coef_codes)
        nz = p.codes != 0
        assert np.array_equal(m.codes != 0, nz)
        assert np.array_equal(m.codes[nz].astype(np.int64), 2 * R - p.codes[nz].astype(np.int64))
        assert np.array_equal(m.outlier_idx, p.outlier_idx)
        assert np.array_equal(m.outlier_val, -p.outlier_val)
        assert m.counters == p.counters


# ----------------------------------------------------------------------------- P5 power-of-two scaling
@pytest.mark.parametrize("s", [-7, 3, 20])
def test_p5_power_of_two_scaling(s):
    rng = np.random.default_rng(4)
    f = (rng.normal(size=(12, 13, 30)) + 5).astype(np.float32)
    for mode, eb in [("rel", 1e-3), ("abs", 0.01)]:
        a = oracle.compress(f, eb, mode, radius=64)
        b = oracle.compress(f * np.float32(2.0 ** s), eb * (2.0 ** s if mode == "abs" else 1.0), mode, radius=64)
        assert np.array_equal(a.codes, b.codes)
        assert np.array_equal(a.coef_codes, b.coef_codes)
        assert b.eb_abs == a.eb_abs * 2.0 ** s


# ----------------------------------------------------------------------------- P7 checkerboard ties
def test_p7_checkerboard_ties():
    dims = (12, 12, 18)
    i, j, k = np.meshgrid(*[np.arange(n) for n in dims], indexing="ij")
    f = ((-1.0) ** (i + j + k)).astype(np.float32)
    res = oracle.compress(f, 1.0, "abs")
    assert np.all(res.coef_codes == 0)
    assert np.all(res.codes == res.radius)          # rint(+-1/2) = 0 under ties-to-even (G4)
    assert res.counters["elem_near_ties"] == f.size
    xr = oracle.decompress(res)
    assert np.all(xr == 0)
    assert np.all(np.abs(xr - f) <= 1.0)              # bound holds with equality


# ----------------------------------------------------------------------------- P8 slab invariance
@pytest.mark.parametrize("G", [2, 3])
def test_p8_slab_invariance(G):
    rng = np.random.default_rng(8)
    f = np.cumsum(rng.normal(size=(40, 11, 23)), axis=0).astype(np.float32)
    whole = oracle.compress(f, 1e-3, "rel", radius=16)
    lo, hi = oracle.value_range(f)
    NB0 = math.ceil(f.shape[0] / 6)
    rows = [NB0 // G + (1 if r < NB0 % G else 0) for r in range(G)]
    start = 0
    codes, coefs, oidx, oval = [], [], [], []
    hist = np.zeros_like(whole.hist)
    for r in range(G):
        a, b = start * 6, min((start + rows[r]) * 6, f.shape[0])
        part = oracle.compress(f[a:b], 1e-3, "rel", radius=16, dim0_offset=a, value_range_override=(lo, hi))
        codes.append(part.codes)
        coefs.append(part.coef_codes)
        oidx.append(part.outlier_idx)
        oval.append(part.outlier_val)
        hist += part.hist
        start += rows[r]
    assert np.array_equal(np.concatenate(codes), whole.codes)
    assert np.array_equal(np.concatenate(coefs), whole.coef_codes)
    assert np.array_equal(np.concatenate(oidx), whole.outlier_idx)
    assert np.array_equal(np.concatenate(oval), whole.outlier_val)
    assert np.array_equal(hist, whole.hist)


# ----------------------------------------------------------------------------- P9 radius outliers
def test_p9_radius_outliers_only_far_from_prediction():
    rng = np.random.default_rng(9)
    dims = (18, 18, 24)
    f = rng.normal(size=dims).astype(np.float64)
    R = 4
    res = oracle.compress(f, 0.02, "abs", radius=R)
    assert res.counters["radius_outliers"] > 0
    eb = res.eb_abs
    w0, ws = eb / 2, eb / 12
    for bid, ((i0, i1), (j0, j1), (k0, k1)) in enumerate(blocks_of(dims)):
        bh = res.coef_codes[bid] * np.array([w0, ws, ws, ws])
        p = local_prediction(bh, (i1 - i0, j1 - j0, k1 - k0))
        x = f[i0:i1, j0:j1, k0:k1]
        c = res.codes[i0:i1, j0:j1, k0:k1]
        resid = np.abs(x - p)
        # predictable: |q| <= R-1 so |x-p| < (2R-1) eb (+ rounding); outliers here are radius outliers
        assert np.all(resid[c != 0] <= (2 * R - 1) * eb * (1 + 1e-12))
        assert np.all(resid[c == 0] >= (2 * R - 1) * eb * (1 - 1e-12))


def test_p9_no_radius_outliers_at_config_bounds():
    """|x - p| <= (1 + 2.214) range/2 + 0.875 eb < (2R - 1) eb when eb_rel > 2.45e-5."""
    from synth import make_field
    for name, shape in [("c1", (64, 64, 64)), ("c3", (48, 48, 48)), ("c2", (24, 60, 60))]:
        f = make_field(name, shape=shape).numpy()
        res = oracle.compress(f, 1e-3 if name != "c2" else 1e-4, "rel")
        assert res.counters["radius_outliers"] == 0, name


# ----------------------------------------------------------------------------- brute force: coefficient codes
def test_brute_force_coefficient_codes_tiny_grids():
    """On tiny grids, coefficient codes equal rint(beta_ls / w) with beta_ls from numpy lstsq per block."""
    rng = np.random.default_rng(10)
    for t in range(12):
        dims = tuple(int(v) for v in rng.integers(1, 14, size=3))
        f = (rng.normal(size=dims) * 10).astype(np.float64)
        res = oracle.compress(f, 1e-3, "rel")
        w = np.array([res.eb_abs / 2, res.eb_abs / 12, res.eb_abs / 12, res.eb_abs / 12])
        for bid, ((i0, i1), (j0, j1), (k0, k1)) in enumerate(blocks_of(dims)):
            blk = f[i0:i1, j0:j1, k0:k1]
            m = blk.shape
            X = design_matrix(*m)
            keep = [0] + [d + 1 for d in range(3) if m[d] > 1]
            sol, *_ = np.linalg.lstsq(X[:, keep], blk.reshape(-1), rcond=None)
            beta = np.zeros(4)
            beta[keep] = sol
            u = beta / w
            near = np.abs(u - np.floor(u) - 0.5) < 1e-6
            want = np.rint(u).astype(np.int64)
            got = res.coef_codes[bid].astype(np.int64)
            assert np.all((want == got) | near), (dims, bid, want, got)


def test_nonfinite_inputs_zero_predictor_and_outliers():
    f = np.linspace(0, 1, 7 * 8 * 9, dtype=np.float32).reshape(7, 8, 9)
    f[1, 2, 3] = np.nan
    f[6, 7, 8] = np.inf
    res = oracle.compress(f, 1e-3, "abs")
    assert res.counters["zero_predictor_blocks"] == 2
    assert res.counters["nonfinite_outliers"] == 2
    assert np.array_equal(res.coef_codes[0], [0, 0, 0, 0])
    xr = oracle.decompress(res)
    assert np.isnan(xr[1, 2, 3]) and np.isinf(xr[6, 7, 8])
    ok = np.isfinite(f)
    assert np.all(np.abs(xr[ok].astype(np.float64) - f[ok]) <= res.eb_abs)
    with pytest.raises(ValueError):
        oracle.compress(f, 1e-3, "rel")   # REL with a non-finite range is a bad range (G14)


@pytest.mark.parametrize("delta,flagged", [(2.0 ** -43, True), (5e-7, False), (0.0, True), (-2.0 ** -43, True)])
def test_coefficient_tie_window_bounds(delta, flagged):
    """The parity tie window (SURVEY 8(c) clarification 1): a constant 6^3 block of value
    c has beta0 = c (P:57 with zero slopes) and, at ABS eb = 1, w0 = eb / 2 = 0.5, so beta0 / w0 =
    2c.  c = 1.25 + delta puts it 2 delta from the half-integer 2.5: 2^-42 (~2.3e-13) lies inside the
    1e-9 window and must exempt the block; 1e-6 lies outside and must not.  (c = 1.25 + 2^-43 and all
    partial sums of the moments are exact doubles.)"""
    f = np.full((6, 6, 6), 1.25 + delta, dtype=np.float64)
    c = oracle.compress(f, 1.0, "abs", radius=32768)
    assert abs(c.coef_raw.reshape(-1)[0] / 0.5 - 2.5) == pytest.approx(abs(2 * delta), rel=1e-6, abs=1e-15)
    assert bool(c.block_exempt[0]) is flagged
    assert c.counters["coef_tie_blocks"] == int(flagged)
    assert c.counters["coef_near_ties"] == int(flagged)
