"""Pins of the truncation oracle (oracle/truncation_oracle.cpp, DEFINITION.md T1-T2) against what the
SPEC worked examples and IEEE-754 arithmetic fix (none re-runs the oracle's byte loops):
* f32 1.0 (0x3F800000) with k = 2 -> 0x3F80 -> 1.0 exactly; pi (0x40490FDB), k = 2 ->
  0x40490000 = 3.140625, |error| ~ 9.67e-4;
* k = bytes-per-sample is bitwise lossless;
* closed-form bound for finite normal values: x' has the sign of x, |x'| <= |x| and
  (|x| - |x'|) < 2^-(8k - 1 - E) |x| with E = exponent bits (8 for f32, 11 for f64) -- the kept
  mantissa bits are 8k - 1 - E;
* the stream holds exactly k bytes per element and its first byte is the sign + exponent byte."""
from __future__ import annotations

import numpy as np
import pytest

import oracle


def test_spec_one_and_pi():
    x = np.array([1.0, np.float32(np.pi)], np.float32)
    b = oracle.trunc_compress(x, 2)
    assert b.tolist() == [0x3F, 0x80, 0x40, 0x49]
    y = oracle.trunc_decompress(b, 2, 2, np.float32)
    assert y[0] == 1.0 and y[1] == np.float32(3.140625)
    assert abs(float(y[1]) - float(x[1])) == pytest.approx(9.67e-4, abs=1e-6)


@pytest.mark.parametrize("dt,s", [(np.float32, 4), (np.float64, 8)])
def test_full_width_is_lossless(dt, s):
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(1001) * 10.0 ** rng.integers(-30, 30, 1001)).astype(dt)
    x[:4] = [np.nan, np.inf, -np.inf, -0.0]
    y = oracle.trunc_decompress(oracle.trunc_compress(x, s), x.size, s, dt)
    assert np.array_equal(y.view(np.uint8), x.view(np.uint8))


@pytest.mark.parametrize("dt,s,E", [(np.float32, 4, 8), (np.float64, 8, 11)])
def test_relative_error_bound(dt, s, E):
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(20000) * 10.0 ** rng.integers(-20, 20, 20000)).astype(dt)
    tiny = np.finfo(dt).tiny
    x = x[np.abs(x) >= tiny]
    for k in range(2, s + 1):
        b = oracle.trunc_compress(x, k)
        assert b.size == k * x.size
        y = oracle.trunc_decompress(b, x.size, k, dt)
        assert np.all(np.sign(y) == np.sign(x)) and np.all(np.abs(y) <= np.abs(x))
        kept = 8 * k - 1 - E
        rel = (np.abs(x).astype(np.float64) - np.abs(y).astype(np.float64)) / np.abs(x).astype(np.float64)
        assert rel.max() < 2.0 ** -kept
        # the first stored byte carries the sign and the top exponent bits
        first = b[::k]
        assert np.array_equal(first >> 7, (x < 0).astype(np.uint8))


def test_invalid_k():
    with pytest.raises(ValueError):
        oracle.trunc_compress(np.ones(3, np.float32), 5)
    with pytest.raises(ValueError):
        oracle.trunc_compress(np.ones(3, np.float32), 0)
