"""Pins of the Huffman oracle (oracle/huffman_oracle.cpp, DEFINITION.md H1-H5) against what the paper,
SPEC and the mathematics fix -- none of these re-run the oracle's own algorithm:

* SPEC worked examples: {a:2, b:1, c:1} -> 6 bits and "aabc" round-trips in 6 bits; one
  symbol -> length 1; 2^k uniform symbols -> all lengths k;
* optimality: brute force over every length vector with Kraft sum <= 1 (a prefix code with those
  lengths exists iff Kraft <= 1) on tiny alphabets, with and without a binding length limit;
* unlimited length: the cost equals the classic greedy Huffman cost (heap merging: sum of the
  internal node weights), an independent algorithm;
* structure: complete code (Kraft = 1), lengths non-increasing in the count, canonical codewords
  prefix-free and consecutive per length (H3);
* the stream: bit length = sum of code lengths, chunks padded to whole words, round trip through a
  table-free bit-by-bit decoder, empty input, and a code absent from the table is refused.
"""
from __future__ import annotations

import heapq
import itertools

import numpy as np
import pytest

import oracle


def cost(hist, lens):
    return int(np.sum(hist.astype(np.int64) * lens.astype(np.int64)))


def kraft(lens):
    l = lens[lens > 0].astype(np.float64)
    return float(np.sum(2.0 ** -l))


def brute_min_cost(counts, max_len):
    """Minimum sum count*len over all length vectors in [1, max_len]^n with Kraft <= 1."""
    best = None
    for ls in itertools.product(range(1, max_len + 1), repeat=len(counts)):
        if sum(2.0 ** -l for l in ls) <= 1.0 + 1e-12:
            c = sum(a * b for a, b in zip(counts, ls))
            best = c if best is None else min(best, c)
    return best


def heap_huffman_cost(counts):
    """Classic greedy Huffman (two smallest merged first): total cost = sum of merged weights."""
    h = [int(c) for c in counts if c > 0]
    if len(h) == 1:
        return h[0]   # one symbol, length 1
    heapq.heapify(h)
    total = 0
    while len(h) > 1:
        a, b = heapq.heappop(h), heapq.heappop(h)
        total += a + b
        heapq.heappush(h, a + b)
    return total


# ----------------------------------------------------------------------------- SPEC worked examples
def test_spec_example_abc():
    # S:354 "frequencies {a:2, b:1, c:1} -> total encoded length 2*1+1*2+1*2 = 6 bits"
    hist = np.array([2, 1, 1], np.int64)
    lens = oracle.huffman_lengths(hist)
    assert cost(hist, lens) == 6
    codes = oracle.huffman_canonical(lens)
    # S:360 "the {a:2,b:1,c:1} stream 'aabc' -> 6-bit payload, round-trips"
    q = np.array([0, 0, 1, 2], np.uint16)
    offs, words = oracle.huffman_encode(q, lens, codes)
    assert int(offs[-1]) == 1 and sum(int(lens[v]) for v in q) == 6
    assert words[0] & ((1 << 26) - 1) == 0          # only the top 6 bits are used
    assert np.array_equal(oracle.huffman_decode(words, offs, q.size, lens, codes), q)


def test_single_symbol_length_one():
    # S:353 "single symbol -> assigned length 1"
    hist = np.zeros(64, np.int64)
    hist[17] = 1000
    lens = oracle.huffman_lengths(hist)
    assert lens[17] == 1 and lens.sum() == 1
    codes = oracle.huffman_canonical(lens)
    q = np.full(100, 17, np.uint16)
    offs, words = oracle.huffman_encode(q, lens, codes, chunk=64)
    assert list(offs) == [0, 2, 4]                   # 64 bits, then 36 bits -> 2 words
    assert np.array_equal(oracle.huffman_decode(words, offs, q.size, lens, codes, chunk=64), q)


@pytest.mark.parametrize("k", [1, 2, 5, 8])
def test_uniform_power_of_two(k):
    # S:355 "uniform frequencies over 2^k symbols -> all lengths k"
    hist = np.zeros(2 ** k + 3, np.int64)
    hist[3:] = 7
    lens = oracle.huffman_lengths(hist)
    assert np.all(lens[3:] == k) and np.all(lens[:3] == 0)


def test_no_symbol_is_an_error():
    with pytest.raises(ValueError):
        oracle.huffman_lengths(np.zeros(8, np.int64))


# ----------------------------------------------------------------------------- optimality
@pytest.mark.parametrize("seed", range(40))
def test_brute_force_optimal(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 7))
    counts = rng.integers(1, 50, size=n) if seed % 3 else (2 ** rng.integers(0, 12, size=n))
    max_len = int(rng.integers(int(np.ceil(np.log2(n))), n + 1)) if seed % 2 else 24
    max_len = max(max_len, int(np.ceil(np.log2(n))), 1)
    hist = np.zeros(n + 5, np.int64)
    pos = rng.permutation(n + 5)[:n]
    hist[pos] = counts
    lens = oracle.huffman_lengths(hist, max_len)
    assert np.all(lens[hist == 0] == 0) and np.all(lens[hist > 0] >= 1) and lens.max() <= max_len
    assert kraft(lens) <= 1.0 + 1e-12
    # lengths above n - 1 are never optimal, so the brute force may stop at min(max_len, n)
    assert cost(hist, lens) == brute_min_cost([int(hist[p]) for p in sorted(pos)], min(max_len, n))


def test_length_limit_binds_fibonacci():
    # Fibonacci counts give the deepest Huffman trees (depth n-1); a limit of 4 must bind
    fib = [1, 1, 2, 3, 5, 8, 13]
    hist = np.array(fib, np.int64)
    free = oracle.huffman_lengths(hist, 24)
    assert free.max() == 6 and cost(hist, free) == heap_huffman_cost(fib)
    for L in (3, 4, 5):
        lens = oracle.huffman_lengths(hist, L)
        assert lens.max() <= L and kraft(lens) <= 1.0 + 1e-12
        assert cost(hist, lens) == brute_min_cost(fib, L)


@pytest.mark.parametrize("seed", range(12))
def test_unlimited_equals_greedy_huffman(seed):
    rng = np.random.default_rng(100 + seed)
    nsym = int(rng.integers(2, 3000))
    a = 1.05 + rng.random() * 1.5
    hist = np.floor(1e6 / np.arange(1, nsym + 1) ** a).astype(np.int64)   # Zipf-like, many ties
    hist = rng.permutation(hist)
    hist[rng.random(nsym) < 0.2] = 0
    if (hist > 0).sum() < 2:
        hist[:2] = 1
    lens = oracle.huffman_lengths(hist, 40)
    assert cost(hist, lens) == heap_huffman_cost(hist)
    assert abs(kraft(lens) - 1.0) < 1e-12                 # complete code
    act = np.flatnonzero(hist)
    order = act[np.argsort(hist[act], kind="stable")]
    assert np.all(np.diff(lens[order].astype(int)) <= 0)   # higher count -> no longer code


# ----------------------------------------------------------------------------- canonical codes
@pytest.mark.parametrize("seed", range(6))
def test_canonical_prefix_free_and_consecutive(seed):
    rng = np.random.default_rng(200 + seed)
    hist = rng.integers(0, 1000, size=300) * (rng.random(300) < 0.5)
    hist[:2] += 1
    lens = oracle.huffman_lengths(hist.astype(np.int64), 12)
    codes = oracle.huffman_canonical(lens)
    act = [s for s in range(lens.size) if lens[s]]
    strings = {s: format(int(codes[s]), f"0{int(lens[s])}b") for s in act}
    assert all(len(strings[s]) == lens[s] for s in act)
    vals = sorted(strings.values())
    for x, y in zip(vals, vals[1:]):
        assert not y.startswith(x)                          # prefix-free
    by_key = sorted(act, key=lambda s: (lens[s], s))
    for s, t in zip(by_key, by_key[1:]):                     # consecutive per length, (len, symbol) order
        assert int(codes[t]) == (int(codes[s]) + 1) << (int(lens[t]) - int(lens[s]))
    assert int(codes[by_key[0]]) == 0


# ----------------------------------------------------------------------------- the stream
@pytest.mark.parametrize("chunk", [1, 7, 2048])
def test_stream_round_trip_and_sizes(chunk):
    rng = np.random.default_rng(chunk)
    R = 512
    q = np.clip(np.round(rng.standard_cauchy(100_003) * 3) + R, 1, 2 * R - 1).astype(np.uint16)
    q[rng.random(q.size) < 0.001] = 0                       # outliers (code 0)
    hist = np.bincount(q, minlength=2 * R).astype(np.int64)
    lens = oracle.huffman_lengths(hist, 24)
    codes = oracle.huffman_canonical(lens)
    offs, words = oracle.huffman_encode(q, lens, codes, chunk)
    nch = -(-q.size // chunk)
    assert offs.size == nch + 1
    for c in range(0, nch, max(1, nch // 50)):
        bits = int(lens[q[c * chunk:(c + 1) * chunk]].astype(np.int64).sum())
        assert int(offs[c + 1] - offs[c]) == -(-bits // 32)
    assert int(offs[-1]) <= -(-cost(hist, lens) // 32) + nch
    assert np.array_equal(oracle.huffman_decode(words, offs, q.size, lens, codes, chunk), q)


def test_empty_stream():
    lens = oracle.huffman_lengths(np.array([0, 3, 1], np.int64))
    codes = oracle.huffman_canonical(lens)
    offs, words = oracle.huffman_encode(np.zeros(0, np.uint16), lens, codes)
    assert offs.tolist() == [0] and words.size == 0
    assert oracle.huffman_decode(words, offs, 0, lens, codes).size == 0


def test_absent_symbol_refused():
    lens = oracle.huffman_lengths(np.array([0, 3, 1], np.int64))
    codes = oracle.huffman_canonical(lens)
    with pytest.raises(ValueError):
        oracle.huffman_encode(np.array([1, 0], np.uint16), lens, codes)
