"""GPU parity of the encoder stage (NEXT-1: sz3g_huffman_*) against the Huffman oracle
(oracle/huffman_oracle.cpp, DEFINITION.md H1-H5), on the same seeded inputs:

* code lengths and canonical codewords: bit-exact (same definition, same tie rule);
* chunk offsets and payload words: bit-exact given the same table;
* decode(encode(codes)) == codes (the payload being bit-exact, the GPU decoder reads the oracle's stream);
* edge cases: one active symbol, two symbols (R = 1), a binding length limit (Fibonacci counts),
  codes longer than the decoder's 12-bit table, empty input, a ragged last chunk, odd chunk sizes,
  a code without a codeword, payload overflow, a corrupt stream;
* the configs' real code streams (c1-c4 at full size through the compressor)."""
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


def gpu_table(hist_np, max_len=16):
    s = sz()
    t = s.huffman_codebook(torch.from_numpy(hist_np.astype(np.int64)).cuda(), max_len).check()
    packed = t.codewords.cpu().numpy().view(np.uint32)
    assert np.array_equal(packed >> 24, t.lengths.cpu().numpy())
    return t, t.lengths.cpu().numpy(), packed & 0xFFFFFF


def round_trip(q_np, hist_np=None, chunk=2048, max_len=16):
    """Full GPU path vs the oracle; returns the oracle's (lens, codes, offs, words)."""
    s = sz()
    if hist_np is None:
        hist_np = np.bincount(q_np, minlength=int(q_np.max()) + 1 if q_np.size else 1)
    t, lens, cws = gpu_table(hist_np, max_len)
    olens = oracle.huffman_lengths(hist_np.astype(np.int64), max_len)
    ocws = oracle.huffman_canonical(olens)
    assert np.array_equal(lens, olens), "code lengths"
    assert np.array_equal(cws, ocws), "canonical codewords"
    q = torch.from_numpy(q_np.astype(np.uint16)).cuda()
    hs = s.huffman_encode(q, t, chunk).check()
    offs_g = hs.offsets.cpu().numpy().view(np.uint64)
    offs_o, words_o = oracle.huffman_encode(q_np, olens, ocws, chunk)
    assert np.array_equal(offs_g, offs_o), "chunk offsets"
    words_g = hs.payload[:hs.words()].cpu().numpy().view(np.uint32)
    assert np.array_equal(words_g, words_o), "payload"
    dec = s.huffman_decode(hs, t)
    torch.cuda.synchronize()
    assert int(hs.status.item()) == 0
    assert np.array_equal(dec.cpu().numpy(), q_np.astype(np.uint16)), "decode(encode(q))"
    return olens, ocws, offs_o, words_o


@pytest.mark.parametrize("seed", range(8))
def test_random_streams(seed):
    rng = np.random.default_rng(seed)
    R = [4, 64, 512, 32768][seed % 4]
    n = int(rng.integers(1, 300_000))
    scale = [0.5, 3, 30, 300][seed % 4]
    q = np.clip(np.round(rng.standard_cauchy(n) * scale) + R, 1, 2 * R - 1).astype(np.uint16)
    q[rng.random(n) < 0.002] = 0
    hist = np.bincount(q, minlength=2 * R)
    chunk = [2048, 2048, 1000, 7, 2048, 1, 33, 2048][seed]
    round_trip(q, hist, chunk)


def test_single_symbol_and_two_symbols():
    q = np.full(10_001, 5, np.uint16)
    lens, *_ = round_trip(q, np.bincount(q, minlength=8))
    assert lens[5] == 1 and lens.sum() == 1
    q2 = np.array([1, 1, 0, 1, 0], np.uint16)               # R = 1: codes {0, 1}
    lens2, *_ = round_trip(q2, np.bincount(q2, minlength=2))
    assert list(lens2) == [1, 1]


def test_length_limit_binds_and_long_codes():
    # Fibonacci counts: the unlimited Huffman depth is n - 1 = 29 > 16, so the limit binds, and many
    # codes are longer than the decoder's 12-bit table (its slow path)
    fib = [1, 1]
    while len(fib) < 30:
        fib.append(fib[-1] + fib[-2])
    hist = np.array(fib, np.int64)
    q = np.repeat(np.arange(30, dtype=np.uint16), fib)
    np.random.default_rng(1).shuffle(q)
    assert oracle.huffman_lengths(hist, 40).max() == 29
    lens, *_ = round_trip(q, hist)
    assert lens.max() == 16 and (lens > 12).sum() > 3
    for L in (5, 8, 12, 13):
        round_trip(q, hist, max_len=L)


def test_uniform_65536_symbols():
    q = np.arange(65536, dtype=np.uint16).repeat(3)
    np.random.default_rng(2).shuffle(q)
    lens, *_ = round_trip(q, np.bincount(q, minlength=65536))
    assert np.all(lens == 16)


def test_empty_input_and_errors():
    s = sz()
    t, *_ = gpu_table(np.array([0, 5, 3], np.int64))
    hs = s.huffman_encode(torch.zeros(0, dtype=torch.uint16, device="cuda"), t).check()
    assert hs.words() == 0
    # a code without a codeword
    bad = s.huffman_encode(torch.tensor([1, 0, 2], dtype=torch.uint16, device="cuda"), t)
    with pytest.raises(Exception):
        bad.check()
    # payload capacity too small
    q = torch.full((10_000,), 1, dtype=torch.uint16, device="cuda")
    small = s.huffman_encode(q, t, payload=torch.empty(10, dtype=torch.int32, device="cuda"))
    with pytest.raises(Exception, match="capacity"):
        small.check()
    # empty histogram
    with pytest.raises(Exception):
        gpu_table(np.zeros(16, np.int64))


def test_corrupt_stream_flagged():
    s = sz()
    rng = np.random.default_rng(3)
    q_np = rng.integers(0, 20, size=50_000).astype(np.uint16)
    hist = np.bincount(q_np, minlength=32)
    t, *_ = gpu_table(hist)
    hs = s.huffman_encode(torch.from_numpy(q_np).cuda(), t).check()
    hs.offsets[1:] -= 1                               # every chunk loses its last word
    hs.offsets[0] = 0
    hs.status.zero_()
    s.huffman_decode(hs, t)
    torch.cuda.synchronize()
    assert int(hs.status.item()) & s.STATUS_BAD_HUFFMAN


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_config_code_streams(name):
    """The compressor's own codes at full size: histogram -> codebook -> encode -> decode."""
    s = sz()
    from synth import config_by_name, make_field
    cfg = config_by_name(name)
    x = make_field(cfg, device="cuda")
    res = s.compress(x, cfg.eb, cfg.eb_mode, cfg.radius)
    hist = res.hist.cpu().numpy()
    q = res.codes.cpu().numpy().reshape(-1)
    olens, ocws, offs, words = round_trip(q, hist)
    bits = int((hist * olens.astype(np.int64)).sum())
    print(name, "bits/code", bits / q.size, "words", int(offs[-1]))


def test_full_chunk_path_alignments_and_window():
    """The full-chunk fast path (2048-code chunks, 16-byte aligned codes) against the oracle's stream,
    written into a 16-byte aligned payload and into one offset by a word (scalar copy-out), from
    aligned codes and from codes offset by one element (generic kernels); codes spread over 65536
    symbols so that warps leave the shared table window."""
    s = sz()
    rng = np.random.default_rng(11)
    R = 32768
    n = 2048 * 37 + 5
    q = np.clip(np.round(rng.standard_cauchy(n + 1) * 40) + R, 0, 2 * R - 1).astype(np.uint16)
    q[rng.random(n + 1) < 0.01] = rng.integers(0, 2 * R, size=int((rng.random(n + 1) < 0.01).sum()) or 1)[0]
    hist = np.bincount(q, minlength=2 * R)
    t, lens, cws = gpu_table(hist)
    qd = torch.from_numpy(q).cuda()
    for view in (qd[:n], qd[1:]):
        q_np = view.cpu().numpy()
        offs_o, words_o = oracle.huffman_encode(q_np, lens, cws, 2048)
        for shift in (0, 1, 2, 3):
            cap = int(offs_o[-1]) + 8
            buf = torch.zeros(cap + shift, dtype=torch.int32, device="cuda")
            hs = s.huffman_encode(view, t, payload=buf[shift:]).check()
            assert np.array_equal(hs.offsets.cpu().numpy().view(np.uint64), offs_o)
            got = buf[shift:shift + int(offs_o[-1])].cpu().numpy().view(np.uint32)
            assert np.array_equal(got, words_o), f"payload (shift {shift})"
            dec = s.huffman_decode(hs, t)
            torch.cuda.synchronize()
            assert np.array_equal(dec.cpu().numpy(), q_np)


def test_full_chunk_path_flags_missing_codeword():
    """A code without a codeword inside full chunks (in the table window, and >= nsym) is flagged."""
    s = sz()
    R = 512
    q = np.full(2048 * 4, R, np.uint16)
    q[::7] = R + 1
    hist = np.bincount(q, minlength=2 * R)
    t, *_ = gpu_table(hist)
    for bad_code in (R + 5, 2 * R + 3):
        qb = q.copy()
        qb[3000] = bad_code
        hs = s.huffman_encode(torch.from_numpy(qb).cuda(), t)
        torch.cuda.synchronize()
        assert int(hs.status.item()) & s.STATUS_BAD_HUFFMAN


@pytest.mark.parametrize("n", [2047, 2048, 2049, 4096, 2048 * 33, 2048 * 33 + 1])
def test_full_chunk_boundaries(n):
    """Sizes at and around multiples of the 2048-code chunk: only full chunks (fast kernels alone), one
    ragged tail (fast + generic), no full chunk (generic alone) -- against the oracle's stream."""
    rng = np.random.default_rng(n)
    R = 512
    q = np.clip(np.round(rng.standard_normal(n) * 20) + R, 1, 2 * R - 1).astype(np.uint16)
    round_trip(q, np.bincount(q, minlength=2 * R))


def test_persistent_decoder_shape_large_stream():
    """Past 32 groups of 32 full chunks per SM the decoder runs as one persistent 32-warp CTA per SM
    (csrc/huffman.cu, k_huff_decode_full<32>); smaller streams take the 8-warp CTAs the other tests
    cover.  A 312 M-code stream with a heavy tail (codes longer than the 12-bit LUT, slow path taken by
    many warps), a partial last group and a ragged last chunk: codebook vs the oracle, decode(encode(q))
    == q on the GPU, and the payload of sampled chunks (every chunk starts on a word boundary, DEFINITION
    H4) bit-exact vs the oracle's encoding of the same chunk."""
    s = sz()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = 2048 * (sms * 32 * 32 + 1000 + 17) + 123
    g = torch.Generator(device="cuda")
    g.manual_seed(2111)
    R = 32768
    z = torch.randn(n, generator=g, device="cuda") * 6.0
    tail = torch.rand(n, generator=g, device="cuda") < 0.01
    z = torch.where(tail, z * 300.0, z)
    q = (torch.round(z) + R).clamp_(1, 2 * R - 1).to(torch.int32)
    hist = torch.bincount(q, minlength=2 * R)
    q = q.to(torch.uint16)
    del z, tail
    hist_np = hist.cpu().numpy()
    t, lens, cws = gpu_table(hist_np)
    olens = oracle.huffman_lengths(hist_np.astype(np.int64), 16)
    ocws = oracle.huffman_canonical(olens)
    assert np.array_equal(lens, olens) and np.array_equal(cws, ocws)
    assert (hist_np[olens > 12].sum() / n) > 1e-3, "the stream must exercise the long-code slow path"
    hs = s.huffman_encode(q, t, 2048).check()
    dec = s.huffman_decode(hs, t)
    torch.cuda.synchronize()
    assert int(hs.status.item()) == 0
    assert torch.equal(dec.view(torch.int16), q.view(torch.int16)), "decode(encode(q))"
    offs = hs.offsets.cpu().numpy().view(np.uint64)
    nch = (n + 2047) // 2048
    rng = np.random.default_rng(7)
    sample = sorted(set(rng.integers(0, nch, 48).tolist()) | {0, nch - 2, nch - 1})
    for c in sample:
        lo, hi = c * 2048, min(n, (c + 1) * 2048)
        qc = q[lo:hi].view(torch.int16).cpu().numpy().view(np.uint16)
        o_offs, o_words = oracle.huffman_encode(qc, olens, ocws, 2048)
        w = hs.payload[int(offs[c]):int(offs[c + 1])].cpu().numpy().view(np.uint32)
        assert int(offs[c + 1] - offs[c]) == int(o_offs[-1]) and np.array_equal(w, o_words), f"chunk {c}"
