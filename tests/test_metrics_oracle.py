"""Pins of the metric definitions (DEFINITION.md M1-M3) against SPEC's worked examples and
hand-computed cases."""
from __future__ import annotations

import math

import numpy as np

import oracle


def test_psnr_spec_examples():
    assert oracle.psnr(1.0, 0.0) == math.inf                     # S:546 identical grids -> inf
    x = np.linspace(0, 1, 1001)
    mx, sq, cnt = oracle.error_stats(x, x + 0.01, eb=0.005)       # S:547 range 1, every element off by 0.01
    assert abs(mx - 0.01) < 1e-15 and abs(sq / x.size - 1e-4) < 1e-15 and cnt == x.size
    assert abs(oracle.psnr(1.0, sq / x.size) - 40.0) < 1e-9
    assert oracle.psnr(3.0, 9.0) == 0.0                           # S:548 MSE == range^2 -> 0 dB


def test_bit_rate_spec_examples():
    assert oracle.bit_rate(32, 32.0) == 1.0
    assert oracle.bit_rate(64, 8.0) == 8.0
    assert oracle.bit_rate(32, 1.0) == 32.0


def test_error_stats_special_values():
    x = np.array([1.0, np.nan, np.inf, 2.0, 5.0], np.float32)
    y = np.array([1.0, np.nan, np.inf, 2.5, 4.0], np.float32)     # NaN / Inf preserved bitwise -> 0
    mx, sq, cnt = oracle.error_stats(x, y, eb=0.6)
    assert mx == 1.0 and sq == 0.25 + 1.0 and cnt == 1
    y2 = y.copy()
    y2[3] = np.nan
    mx2, _, cnt2 = oracle.error_stats(x, y2, eb=10.0)
    assert math.isnan(mx2) and cnt2 == 1
