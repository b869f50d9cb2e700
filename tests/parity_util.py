"""GPU-vs-oracle comparison rules (SURVEY 8(c) "Parity rules").

* coefficient codes, element codes, outlier sets and histograms: bit-exact, except blocks the oracle
  flags as coefficient near-ties (their beta/w sits within the tolerance window of a half-integer,
  so a beta that differs by the allowed 1e-12 block-scale may round to the neighbouring code);
  those blocks are counted and removed from both sides;
* unquantised beta: |b_gpu - b_orc| <= 1e-12 * max(|b_orc|, mean|f| over the block);
* decompressed values: bit-exact given identical codes (GPU decompress vs oracle decompress of the
  GPU's own codes, everywhere, and vs the oracle's compress-time x' outside exempt blocks);
* the error bound |x - x'| <= eb_abs holds for every element.
"""
from __future__ import annotations

import math

import numpy as np

BETA_TOL = 1e-12


def block_ids(shape, B=6):
    """Block id of every element (row-major block order), shape = field shape."""
    n0, n1, n2 = shape
    NB1, NB2 = math.ceil(n1 / B), math.ceil(n2 / B)
    a = (np.arange(n0) // B).reshape(-1, 1, 1)
    b = (np.arange(n1) // B).reshape(1, -1, 1)
    c = (np.arange(n2) // B).reshape(1, 1, -1)
    return (a * NB1 + b) * NB2 + c


def block_mean_abs(f, B=6):
    n0, n1, n2 = f.shape
    P = [math.ceil(n / B) * B for n in f.shape]
    pad = np.zeros(P, np.float64)
    pad[:n0, :n1, :n2] = np.abs(f.astype(np.float64))
    cnt = np.zeros(P, np.float64)
    cnt[:n0, :n1, :n2] = 1
    s = pad.reshape(P[0] // B, B, P[1] // B, B, P[2] // B, B).sum(axis=(1, 3, 5))
    c = cnt.reshape(P[0] // B, B, P[1] // B, B, P[2] // B, B).sum(axis=(1, 3, 5))
    return (s / c).reshape(-1)


def compare(x: np.ndarray, gpu: dict, orc, *, check_beta: bool = True, xdec_gpu: np.ndarray | None = None,
            xdec_orc_of_gpu: np.ndarray | None = None) -> dict:
    """Compare GPU outputs (numpy dict) with an oracle.Compressed on the same input bytes.

    gpu keys: codes, coef_codes, coef_raw (optional), outlier_idx, outlier_val, hist (optional), eb_abs.
    Returns a report dict; raises AssertionError on any violation.
    """
    shape = orc.dims
    x3 = x.reshape(shape)
    rep = {"N": int(x3.size), "eb_abs": orc.eb_abs, "counters": dict(orc.counters)}
    assert gpu["eb_abs"] == orc.eb_abs, (gpu["eb_abs"], orc.eb_abs)
    exempt = orc.block_exempt.astype(bool)
    rep["exempt_blocks"] = int(exempt.sum())
    ok_blocks = ~exempt
    # coefficient codes
    cc_g, cc_o = gpu["coef_codes"].reshape(-1, 4), orc.coef_codes.reshape(-1, 4)
    bad = np.flatnonzero(ok_blocks & np.any(cc_g != cc_o, axis=1))
    assert bad.size == 0, f"coef codes differ in {bad.size} non-exempt blocks, e.g. {bad[:5]}: {cc_g[bad[:3]]} vs {cc_o[bad[:3]]}"
    rep["coef_code_mismatch_exempt"] = int(np.sum(exempt & np.any(cc_g != cc_o, axis=1)))
    # raw beta
    if check_beta and gpu.get("coef_raw") is not None:
        scale = block_mean_abs(x3)
        bg, bo = gpu["coef_raw"].reshape(-1, 4), orc.coef_raw.reshape(-1, 4)
        fin = np.isfinite(bo).all(axis=1)
        tol = BETA_TOL * np.maximum(np.abs(bo), scale[:, None])
        err = np.abs(bg - bo)
        viol = fin[:, None] & ~(err <= tol)
        assert not viol.any(), f"beta outside 1e-12 block-scale tolerance in {int(viol.any(axis=1).sum())} blocks; worst rel {np.max(err[fin] / np.maximum(tol[fin], 1e-300)) * BETA_TOL}"
        rel = err[fin] / np.maximum(np.maximum(np.abs(bo[fin]), scale[fin][:, None]), 1e-300)
        rep["beta_max_rel_err"] = float(rel.max()) if rel.size else 0.0
    # element codes
    if exempt.any():
        emask = ~exempt[block_ids(shape)]
    else:
        emask = None
    cg, co = gpu["codes"].reshape(shape), orc.codes
    if emask is None:
        neq = np.flatnonzero((cg != co).reshape(-1))
    else:
        neq = np.flatnonzero(((cg != co) & emask).reshape(-1))
    assert neq.size == 0, f"{neq.size} element codes differ, first at {neq[:5]}: gpu {cg.reshape(-1)[neq[:5]]} orc {co.reshape(-1)[neq[:5]]}"
    # outliers as sets keyed by global index
    gi = gpu["outlier_idx"].astype(np.uint64)
    order = np.argsort(gi, kind="stable")
    gi, gv = gi[order], gpu["outlier_val"][order]
    oi_, ov = orc.outlier_idx, orc.outlier_val
    o2 = np.argsort(oi_, kind="stable")
    oi_, ov = oi_[o2], ov[o2]
    if emask is not None:
        base = orc.dim0_offset * shape[1] * shape[2]
        keep_g = emask.reshape(-1)[(gi - base).astype(np.int64)]
        keep_o = emask.reshape(-1)[(oi_ - base).astype(np.int64)]
        gi, gv, oi_, ov = gi[keep_g], gv[keep_g], oi_[keep_o], ov[keep_o]
    assert np.array_equal(gi, oi_), f"outlier index sets differ ({gi.size} vs {oi_.size})"
    assert np.array_equal(gv.view(np.uint8), ov.view(np.uint8)), "outlier values differ"
    rep["outliers"] = int(orc.outlier_idx.size)
    # histogram
    if gpu.get("hist") is not None:
        if emask is None:
            assert np.array_equal(gpu["hist"], orc.hist), "histograms differ"
        else:
            assert np.array_equal(gpu["hist"], np.bincount(cg.reshape(-1), minlength=gpu["hist"].size)), \
                "GPU histogram inconsistent with GPU codes"
        rep["hist_zero_bin"] = int(gpu["hist"][0])
    # decompression
    if xdec_gpu is not None:
        xd = xdec_gpu.reshape(shape)
        if xdec_orc_of_gpu is not None:
            assert np.array_equal(xd.view(np.uint8), xdec_orc_of_gpu.reshape(shape).view(np.uint8)), \
                "GPU decompression differs from the oracle's decompression of the same codes"
        xp = orc.xprime
        if emask is None:
            assert np.array_equal(xd.view(np.uint8), xp.view(np.uint8)), "decompressed values differ from oracle x'"
        else:
            assert np.array_equal(xd[emask].view(np.uint8), xp[emask].view(np.uint8))
        fin = np.isfinite(x3)
        err = np.abs(xd.astype(np.float64)[fin] - x3.astype(np.float64)[fin])
        assert np.all(err <= orc.eb_abs), f"error bound violated: max {err.max()} > {orc.eb_abs}"
        rep["max_abs_err"] = float(err.max()) if err.size else 0.0
        nonfin = ~fin
        if nonfin.any():
            assert np.array_equal(xd[nonfin].view(np.uint8), x3[nonfin].view(np.uint8))
    return rep
