"""SHA-256 digests of every output of a fixed set of small libsz3g invocations (all kernel families, TMA
and plain variants, full tiles and ragged tails).  Run under different library builds (SZ3G_LIB) and
compare the JSON: tests/test_gpu_chaos.py runs it against the chaos build (-DSZ3G_CHAOS, random
delays at every pipeline hand-off) and requires digests identical to the normal build's.

    SZ3G_LIB=paper_2111_02925_b200/lib/chaos/libsz3g.so python tools/digest_cases.py > chaos.json

Outlier lists are appended through a device counter in a nondeterministic order: they are hashed
sorted by index.  Everything else is hashed as produced.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_02925_b200 import sz3g  # noqa: E402

GEN = sz3g.FLAG_FORCE_GENERIC


def h(*ts) -> str:
    m = hashlib.sha256()
    for t in ts:
        if isinstance(t, torch.Tensor):
            t = t.detach().contiguous().cpu().numpy()
        m.update(np.ascontiguousarray(t).view(np.uint8).tobytes())
    return m.hexdigest()[:24]


def outliers(res):
    n = res.n_outliers
    idx = res.outlier_idx[:n].cpu().numpy()
    o = np.argsort(idx, kind="stable")
    return idx[o], res.outlier_val[:n].cpu().numpy()[o]


def fields():
    from synth import make_field
    rng = np.random.default_rng(7)
    return {
        "c1": make_field("c1", device="cuda"),                                  # 64^3 f32, ragged edge blocks
        "c2": make_field("c2", device="cuda", shape=(30, 100, 200)),            # c2 recipe, cropped
        "c3": make_field("c3", device="cuda", shape=(36, 96, 192)),             # lognormal, hot bin
        "c4": make_field("c4", device="cuda", shape=(20, 50, 96)),              # f64
        "odd": torch.from_numpy(rng.normal(size=(7, 13, 97)).astype(np.float32)).cuda(),   # no 16-B pitch
        "big": make_field("c5", device="cuda", shape=(96, 512, 1024)),          # many tiles per CTA
        # rows of a multiple of 4 but not of 8 values: plain 8-byte slab store + k_decompress_staged
        "rows4": torch.from_numpy(np.cumsum(rng.normal(size=(14, 20, 100)), axis=-1).astype(np.float32)).cuda(),
    }


def cases():
    out = {}
    F = fields()
    for name, x in F.items():
        for flags in (0, GEN):
            for R in (32768, 8):
                tag = f"{name}/{'plain' if flags else 'tma'}/R{R}"
                bufs = sz3g.CompressBuffers(x.shape, x.dtype, R, outlier_cap=x.numel(), device=x.device)
                mm, beta = sz3g.regression_analyze(x, bufs.minmax, bufs.beta_buffer())
                r2 = sz3g.regression_quantize(x, 1e-3, "rel", R, mm, beta, bufs=bufs, flags=flags).finalize()
                out[f"{tag}/analyze"] = h(mm, beta)
                out[f"{tag}/quantize"] = h(r2.codes, r2.coef_codes, r2.hist, *outliers(r2))
                xo2 = sz3g.regression_decompress(r2.codes, r2.coef_codes, r2.outlier_idx, r2.outlier_val,
                                                 r2.outlier_idx.numel(), 1e-3, R, x.dtype, flags=flags,
                                                 d_outlier_count=r2.outlier_count, eb_mode="rel", d_minmax=mm)
                out[f"{tag}/decompress"] = h(xo2)
                r1 = sz3g.regression_compress(x, 1e-3, "rel", R, coef_raw=True, flags=flags,
                                              outlier_cap=x.numel()).finalize()
                out[f"{tag}/fused"] = h(r1.codes, r1.coef_codes, r1.coef_raw, r1.hist, *outliers(r1))
                lr = sz3g.lr_compress(x, 1e-3, "rel", R, outlier_cap=x.numel(), flags=flags)
                out[f"{tag}/lr"] = h(lr.codes, lr.coef_codes, lr.lr_flags, lr.hist, *outliers(lr))
                out[f"{tag}/lr_dec"] = h(sz3g.decompress(lr, flags=flags))
        ir = sz3g.interp_compress(x, 1e-3, "rel", 64, outlier_cap=x.numel()).finalize()
        out[f"{name}/interp"] = h(ir.codes, ir.xprime, ir.hist, *outliers(ir))
        out[f"{name}/interp_dec"] = h(sz3g.interp_decompress(ir.codes, ir.outlier_idx, ir.outlier_val, ir.n_outliers,
                                                             ir.eb_abs, 64, x.dtype))
        out[f"{name}/value_range"] = h(sz3g.value_range(x))
        res = sz3g.compress(x, 1e-3, "rel", 32768)
        out[f"{name}/histogram"] = h(sz3g.histogram(res.codes.view(-1), 32768))
        table = sz3g.huffman_codebook(res.hist).check()
        out[f"{name}/codebook"] = h(table.lengths, table.codewords, table.dtable)
        codes = res.codes.view(-1)
        for n in (codes.numel(), codes.numel() - 1, 2048 * 3, 1000):
            c = codes[:n].contiguous()
            hs = sz3g.huffman_encode(c, table).check()
            out[f"{name}/huff_enc/{n}"] = h(hs.offsets, hs.payload[:hs.words()])
            out[f"{name}/huff_dec/{n}"] = h(sz3g.huffman_decode(hs, table))
        cs = sz3g.encode_coefficients(res.coef_codes)
        out[f"{name}/coef_enc"] = h(cs.stream.payload[:cs.stream.words()], cs.escapes)
        out[f"{name}/coef_dec"] = h(sz3g.decode_coefficients(cs))
        for k in range(1, x.element_size() + 1):
            b = sz3g.truncation_compress(x.view(-1), k)
            out[f"{name}/trunc{k}"] = h(b, sz3g.truncation_decompress(b, x.numel(), k, x.dtype))
        xo = sz3g.decompress(res)
        out[f"{name}/error_stats"] = h(sz3g.error_stats(x, xo, res.eb_abs))
        out[f"{name}/ties"] = h(sz3g.tie_counts(x, 1e-3, "rel", 32768, sz3g.value_range(x), res.coef_codes))
        out[f"{name}/stream"] = h(sz3g.from_bytes(sz3g.to_bytes(res)))
    torch.cuda.synchronize()
    return out


if __name__ == "__main__":
    sz3g.load()
    d = cases()
    d["_lib"] = os.environ.get("SZ3G_LIB", "default")
    d["_launches"] = sz3g.launch_count()
    print(json.dumps(d))
