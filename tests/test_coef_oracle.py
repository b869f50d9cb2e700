"""Pins of the coefficient delta coding (DEFINITION.md C1-C2): hand-worked example, the SPEC's zero-
delta case ("identical coefficients in consecutive blocks -> all delta codes map to the zero
bin"), first block against 0, escapes for large jumps incl. int32 extremes, round trip."""
from __future__ import annotations

import numpy as np

import oracle


def test_hand_example():
    coef = np.array([[3, -1, 0, 2], [3, 0, 0, -2], [-4, 0, 70000, -2]], np.int32)
    sym, esc = oracle.coef_delta_encode(coef)
    # channel 0: deltas 3, 0, -7 -> zigzag 6, 0, 13; channel 1: -1, 1, 0 -> 1, 2, 0;
    # channel 2: 0, 0, 70000 -> 0, 0, 140000 (escape); channel 3: 2, -4, 0 -> 4, 7, 0
    assert sym.tolist() == [6, 0, 13, 1, 2, 0, 0, 0, 65535, 4, 7, 0]
    assert esc.tolist() == [140000]
    assert np.array_equal(oracle.coef_delta_decode(sym, 3, esc), coef)


def test_identical_blocks_zero_bin():
    coef = np.tile(np.array([[5, -3, 2, 9]], np.int32), (100, 1))
    sym, esc = oracle.coef_delta_encode(coef)
    assert esc.size == 0
    assert np.all(sym.reshape(4, 100)[:, 1:] == 0)                 # every delta after the first is 0
    assert sym.reshape(4, 100)[:, 0].tolist() == [10, 5, 4, 18]      # first block against (0,0,0,0)


def test_extremes_and_round_trip():
    rng = np.random.default_rng(0)
    coef = rng.integers(-50, 50, size=(10_000, 4)).cumsum(axis=0).astype(np.int32)
    coef[17] = [2**31 - 1, -2**31, 0, 1]
    coef[18] = [-2**31, 2**31 - 1, 0, 1]
    sym, esc = oracle.coef_delta_encode(coef)
    assert esc.size >= 4 and int(esc.max()) == 2 * (2**32 - 1)       # d = 2^32 - 1 -> zigzag 2d
    assert np.array_equal(oracle.coef_delta_decode(sym, coef.shape[0], esc), coef)
