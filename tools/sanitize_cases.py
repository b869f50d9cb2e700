"""Small invocations of every libsz3g kernel family, for compute-sanitizer (SURVEY §4 T5 / §5 race
detection).  Run as

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} --error-exitcode 9 \\
        python tools/sanitize_cases.py [--only FAMILY ...]

Cases: analyze + quantise (two-pass, BETA), fused compress, decompress, value range, standalone
histogram (TMA and plain variants; full tiles and ragged tails), SZ3-LR compress / decompress,
Huffman codebook / encode / decode (full-chunk fast paths and the generic tail), truncation, coefficient
delta coding, error statistics.  Each case also checks its result against a second path (so a hazard
that changes data is visible), but the point of this script is the sanitizer's report.
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_02925_b200 import sz3g  # noqa: E402

GEN = sz3g.FLAG_FORCE_GENERIC


def fields():
    from synth import make_field
    rng = np.random.default_rng(7)
    c1 = make_field("c1", device="cuda")                                     # 64^3 f32, ragged edge blocks
    c2 = make_field("c2", device="cuda", shape=(30, 100, 200))               # c2 recipe, cropped
    c4 = make_field("c4", device="cuda", shape=(20, 50, 96))                 # f64
    odd = torch.from_numpy(rng.normal(size=(7, 13, 97)).astype(np.float32)).cuda()   # no 16-B row pitch
    return {"c1": c1, "c2": c2, "c4": c4, "odd": odd}


def regression(F):
    for name, x in F.items():
        for flags in (0, GEN):
            for R in (32768, 8):
                bufs = sz3g.CompressBuffers(x.shape, x.dtype, R, outlier_cap=x.numel(), device=x.device)
                mm, beta = sz3g.regression_analyze(x, bufs.minmax, bufs.beta_buffer())
                r2 = sz3g.regression_quantize(x, 1e-3, "rel", R, mm, beta, bufs=bufs, flags=flags).finalize()
                c2 = r2.codes.clone()
                r1 = sz3g.regression_compress(x, 1e-3, "rel", R, coef_raw=True, flags=flags,
                                              outlier_cap=x.numel()).finalize()
                assert torch.equal(c2, r1.codes), (name, flags, R)
                xo = sz3g.decompress(r1, flags=flags)
                xo2 = sz3g.regression_decompress(r2.codes, r2.coef_codes, r2.outlier_idx, r2.outlier_val, r2.n_outliers,
                                                 1e-3, R, x.dtype, flags=flags, d_outlier_count=r2.outlier_count,
                                                 eb_mode="rel", d_minmax=mm)
                torch.cuda.synchronize()
                assert torch.equal(xo, xo2)
                st = sz3g.error_stats(x, xo, r1.eb_abs).cpu().tolist()
                assert st[2] == 0
        v = sz3g.value_range(x)
        h = sz3g.histogram(r1.codes.view(-1), 8)
        torch.cuda.synchronize()
        assert int(h.sum()) == x.numel() and float(v[0]) == float(x.min())


def lr(F):
    for name, x in F.items():
        for flags in (0, GEN):
            res = sz3g.lr_compress(x, 1e-3, "rel", 32768, outlier_cap=x.numel(), flags=flags)
            xo = sz3g.decompress(res, flags=flags)
            torch.cuda.synchronize()
            st = sz3g.error_stats(x, xo, res.eb_abs).cpu().tolist()
            assert st[2] == 0, (name, flags)


def huffman(F):
    for name, x in F.items():
        res = sz3g.compress(x, 1e-3, "rel", 32768)
        table = sz3g.huffman_codebook(res.hist).check()
        codes = res.codes.view(-1)
        for n in (codes.numel(), codes.numel() - 1, 2048 * 3, 1000):    # full chunks + generic tails
            c = codes[:n].contiguous()
            hs = sz3g.huffman_encode(c, table).check()
            back = sz3g.huffman_decode(hs, table)
            torch.cuda.synchronize()
            assert torch.equal(back, c), (name, n)
        cs = sz3g.encode_coefficients(res.coef_codes)
        assert torch.equal(sz3g.decode_coefficients(cs), res.coef_codes)


def truncation(F):
    for name, x in F.items():
        for k in range(1, x.element_size() + 1):
            b = sz3g.truncation_compress(x.view(-1), k)
            y = sz3g.truncation_decompress(b, x.numel(), k, x.dtype)
            torch.cuda.synchronize()
            if k == x.element_size():
                assert torch.equal(y, x.view(-1))


def stream(F):
    for name, x in F.items():
        res = sz3g.compress(x, 1e-3, "rel", 32768)
        xo = sz3g.decompress(res)
        assert torch.equal(sz3g.from_bytes(sz3g.to_bytes(res)), xo)


FAMILIES = {"regression": regression, "lr": lr, "huffman": huffman, "truncation": truncation, "stream": stream}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*", default=list(FAMILIES))
    a = ap.parse_args()
    sz3g.load()
    F = fields()
    for fam in a.only:
        FAMILIES[fam](F)
        print("ok", fam, flush=True)
    print("launches", sz3g.launch_count())


if __name__ == "__main__":
    main()
