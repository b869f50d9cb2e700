"""Memory safety without compute-sanitizer (closed on this pool): red zones and poison.

* Red zones (memcheck analogue): every input and output buffer of a call sits inside a larger
  allocation whose guard bands are filled with a byte pattern (0xFF: NaN for floats).  After the call
  the output guards must be intact (no out-of-bounds write) and the results must equal those from
  plain buffers (an out-of-bounds READ of the NaN guard around the input would change them).
* Poison (initcheck analogue): output and scratch buffers pre-filled with 0x00 and with 0xFF give
  bit-identical results, so no kernel reads an output before writing it (beyond the documented
  accumulators: histogram, outlier counter, status, which the API zeroes or accumulates into).

Covers the regression path (analyze, quantise, fused compress, decompress + outlier scatter; TMA and
plain variants; full tiles, ragged edges, a shape without a 16-byte row pitch), SZ3-LR, Huffman encode /
decode, truncation and the tie counters.
"""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

G = 4096   # guard elements on each side (keeps 16-byte alignment for every dtype used)
GEN = 0x1


def sz():
    from paper_2111_02925_b200 import sz3g
    sz3g.load()
    return sz3g


class Guarded:
    """A view of n elements in the middle of a buffer with guard bands filled with `fill`."""

    def __init__(self, shape, dtype, fill: int):
        n = int(np.prod(shape)) if len(shape) else 1
        self.n, self.fill = n, fill
        self.base = torch.empty(n + 2 * G, dtype=dtype, device="cuda")
        self.base.view(torch.uint8).fill_(fill)
        self.t = self.base[G:G + n].view(shape)

    def intact(self) -> bool:
        b, es = self.base.view(torch.uint8), self.base.element_size()
        return bool((b[:G * es] == self.fill).all()) and bool((b[(G + self.n) * es:] == self.fill).all())


def shapes():
    from synth import make_field
    rng = np.random.default_rng(11)
    return {"c1": make_field("c1", device="cuda"),
            "c2crop": make_field("c2", device="cuda", shape=(30, 100, 200)),
            "c4crop": make_field("c4", device="cuda", shape=(20, 50, 96)),
            "odd": torch.from_numpy(rng.normal(size=(7, 13, 97)).astype(np.float32)).cuda(),
            # rows of a multiple of 4 but not of 8 values: no TMA map for the codes -> the 8-byte plain slab
            # store and k_decompress_staged
            "rows4": torch.from_numpy(np.cumsum(rng.normal(size=(14, 20, 100)), axis=-1).astype(np.float32)).cuda()}


def run_regression(x, R, flags, fill, guard_input):
    """analyze -> quantise -> decompress and the fused kernel, every buffer guarded; returns host
    outputs and the guard objects."""
    s = sz()
    gs = []

    def g(shape, dtype):
        o = Guarded(shape, dtype, fill)
        gs.append(o)
        return o.t

    if guard_input:
        xg = Guarded(tuple(x.shape), x.dtype, 0xFF)
        xg.t.copy_(x)
        gs.append(xg)
        x = xg.t
    N, nb = x.numel(), s.num_blocks(x.shape)
    bufs = s.CompressBuffers(x.shape, x.dtype, R, outlier_cap=N, device=x.device)
    bufs.codes, bufs.coef_codes = g(tuple(x.shape), torch.uint16), g((nb, 4), torch.int32)
    bufs.outlier_idx, bufs.outlier_val = g((N,), torch.int64), g((N,), x.dtype)
    bufs.outlier_count, bufs.hist = g((1,), torch.int64), g((2 * R,), torch.int64)
    bufs.eb_abs, bufs.status, bufs.minmax = g((1,), torch.float64), g((1,), torch.int32), g((2,), torch.float64)
    bufs.beta = g((nb, 4), torch.float64)
    mm, beta = s.regression_analyze(x, bufs.minmax, bufs.beta)
    res = s.regression_quantize(x, 1e-3, "rel", R, mm, beta, bufs=bufs, flags=flags).finalize()
    out = g(tuple(x.shape), x.dtype)
    s.regression_decompress(res.codes, res.coef_codes, res.outlier_idx, res.outlier_val, N, 1e-3, R, x.dtype,
                            out=out, flags=flags, d_outlier_count=res.outlier_count, eb_mode="rel", d_minmax=mm)
    n = res.n_outliers
    oi = res.outlier_idx[:n].cpu().numpy()
    o = np.argsort(oi)
    host = dict(mm=mm.cpu().numpy(), beta=beta.cpu().numpy(), codes=res.codes.cpu().numpy(),
                coef=res.coef_codes.cpu().numpy(), hist=res.hist.cpu().numpy(), oi=oi[o],
                ov=res.outlier_val[:n].cpu().numpy()[o], out=out.cpu().numpy())
    # fused kernel into guarded buffers (coef_raw too)
    b2 = s.CompressBuffers(x.shape, x.dtype, R, outlier_cap=N, device=x.device, coef_raw=True)
    b2.codes, b2.coef_codes, b2.coef_raw = g(tuple(x.shape), torch.uint16), g((nb, 4), torch.int32), g((nb, 4), torch.float64)
    b2.outlier_idx, b2.outlier_val = g((N,), torch.int64), g((N,), x.dtype)
    b2.outlier_count, b2.hist, b2.eb_abs, b2.status = (g((1,), torch.int64), g((2 * R,), torch.int64),
                                                      g((1,), torch.float64), g((1,), torch.int32))
    r2 = s.regression_compress(x, 1e-3, "rel", R, d_minmax=mm, bufs=b2, coef_raw=True, flags=flags).finalize()
    host["fused_codes"], host["fused_raw"] = r2.codes.cpu().numpy(), r2.coef_raw.cpu().numpy()
    # SZ3-LR into guarded buffers
    b3 = s.CompressBuffers(x.shape, x.dtype, R, outlier_cap=N, device=x.device)
    b3.codes, b3.coef_codes = g(tuple(x.shape), torch.uint16), g((nb, 4), torch.int32)
    b3.outlier_idx, b3.outlier_val = g((N,), torch.int64), g((N,), x.dtype)
    b3.outlier_count, b3.hist, b3.eb_abs, b3.status = (g((1,), torch.int64), g((2 * R,), torch.int64),
                                                      g((1,), torch.float64), g((1,), torch.int32))
    b3.lr_flags = g((nb,), torch.uint8)
    lr = s.lr_quantize(x, 1e-3, "rel", R, mm, beta, bufs=b3, flags=flags).finalize()
    lout = g(tuple(x.shape), x.dtype)
    s.lr_decompress(lr.codes, lr.coef_codes, lr.lr_flags, lr.outlier_idx, lr.outlier_val, N, 1e-3, R, x.dtype,
                    out=lout, flags=flags, d_outlier_count=lr.outlier_count, eb_mode="rel", d_minmax=mm)
    host["lr_codes"], host["lr_flags"], host["lr_out"] = lr.codes.cpu().numpy(), lr.lr_flags.cpu().numpy(), lout.cpu().numpy()
    # tie counters (read-only on x and the codes)
    cnt = g((4,), torch.int64)
    cnt.zero_()
    host["ties"] = s.tie_counts(x, 1e-3, "rel", R, mm, res.coef_codes, beta, counts=cnt).cpu().numpy()
    torch.cuda.synchronize()
    return host, gs


def same(a: dict, b: dict) -> list:
    return [k for k in a if not np.array_equal(np.ascontiguousarray(a[k]).view(np.uint8),
                                               np.ascontiguousarray(b[k]).view(np.uint8))]


@pytest.mark.parametrize("flags", [0, GEN], ids=["tma", "plain"])
@pytest.mark.parametrize("R", [32768, 8])
def test_redzones_and_poison_regression_lr(flags, R):
    for name, x in shapes().items():
        a, ga = run_regression(x, R, flags, 0x00, guard_input=False)
        b, gb = run_regression(x, R, flags, 0xFF, guard_input=True)
        assert all(o.intact() for o in ga + gb), f"{name}: a guard band was overwritten"
        diff = same(a, b)
        assert not diff, f"{name}: outputs depend on prior buffer contents / input guard: {diff}"


def test_redzones_and_poison_huffman_truncation():
    s = sz()
    for name, x in shapes().items():
        res = s.compress(x, 1e-3, "rel", 32768)
        table = s.huffman_codebook(res.hist).check()
        codes = res.codes.view(-1)
        lib = s.load()
        for n in (codes.numel(), codes.numel() - 1, 2048 * 3 + 5):
            got = []
            for fill in (0x00, 0xFF):
                c = Guarded((n,), torch.uint16, 0xFF)
                c.t.copy_(codes[:n])
                nch = -(-n // s.HUFF_CHUNK)
                pay = Guarded((-(-n * 16 // 32) + nch,), torch.int32, fill)
                offs = Guarded((nch + 1,), torch.int64, fill)
                scr = Guarded((int(lib.sz3g_huffman_encode_scratch_bytes(n, s.HUFF_CHUNK)),), torch.uint8, fill)
                hs = s.huffman_encode(c.t, table, payload=pay.t, offsets=offs.t, scratch=scr.t).check()
                dec = Guarded((n,), torch.uint16, fill)
                s.huffman_decode(hs, table, out=dec.t)
                torch.cuda.synchronize()
                assert all(o.intact() for o in (c, pay, offs, scr, dec)), (name, n, fill)
                assert torch.equal(dec.t, codes[:n])
                got.append((hs.offsets.cpu(), hs.payload[:hs.words()].cpu()))
            assert torch.equal(got[0][0], got[1][0]) and torch.equal(got[0][1], got[1][1])
        for k in range(1, x.element_size() + 1):
            outs = []
            for fill in (0x00, 0xFF):
                b = Guarded((x.numel() * k,), torch.uint8, fill)
                s.truncation_compress(x.view(-1), k, out=b.t)
                y = Guarded((x.numel(),), x.dtype, fill)
                s.truncation_decompress(b.t, x.numel(), k, x.dtype, out=y.t)
                torch.cuda.synchronize()
                assert b.intact() and y.intact()
                outs.append((b.t.cpu(), y.t.view(torch.uint8).cpu()))
            assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
