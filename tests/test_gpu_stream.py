"""End to end through the container: compress on the GPU -> to_bytes (Huffman codes, delta+Huffman
coefficients, outliers) -> from_bytes (parse, validate, GPU decode) gives bit-identical output to the
direct decompression, on configs and on an outlier-heavy case; a corrupted byte is rejected."""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def sz():
    from paper_2111_02925_b200 import sz3g
    sz3g.load()
    return sz3g


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_bytes_round_trip(name):
    s = sz()
    from synth import config_by_name, make_field
    cfg = config_by_name(name)
    x = make_field(cfg, device="cuda")
    res = s.compress(x, cfg.eb, cfg.eb_mode, cfg.radius)
    direct = s.decompress(res)
    b = s.to_bytes(res, eb=cfg.eb, eb_mode=cfg.eb_mode)
    back = s.from_bytes(b)
    assert back.shape == x.shape and back.dtype == x.dtype
    assert torch.equal(back.view(torch.uint8), direct.view(torch.uint8))
    ratio = x.numel() * x.element_size() / len(b)
    print(name, "stream bytes", len(b), "ratio", round(ratio, 3))
    assert ratio > 1.5


def test_outliers_and_corruption():
    s = sz()
    rng = np.random.default_rng(4)
    f = rng.standard_normal((24, 30, 100)).astype(np.float32)
    x = torch.from_numpy(f).cuda()
    res = s.compress(x, 1e-3, "rel", radius=64, outlier_cap=x.numel())
    assert res.n_outliers > 100
    direct = s.decompress(res)
    b = bytearray(s.to_bytes(res, eb=1e-3, eb_mode="rel"))
    assert torch.equal(s.from_bytes(bytes(b)), direct)
    b[len(b) // 2] ^= 1
    with pytest.raises(Exception, match="corrupt"):
        s.from_bytes(bytes(b))


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_lr_bytes_round_trip(name):
    """SZ3-LR results through the container: the flags travel as a bitmap section, from_bytes takes the
    LR decompressor, the output equals the direct LR decompression bit for bit."""
    s = sz()
    from synth import config_by_name, make_field
    cfg = config_by_name(name)
    x = make_field(cfg, device="cuda")
    res = s.lr_compress(x, cfg.eb, cfg.eb_mode, cfg.radius)
    assert int(res.lr_flags.sum()) > 0
    direct = s.decompress(res)
    b = s.to_bytes(res, eb=cfg.eb, eb_mode=cfg.eb_mode)
    back = s.from_bytes(b)
    assert torch.equal(back.view(torch.uint8), direct.view(torch.uint8))
    err = (back.double() - x.double()).abs().max().item()
    assert err <= res.eb_abs


def test_bytes_round_trip_slab_with_dim0_offset():
    """A sharded slab (dim0_offset != 0, so its outlier indices are global) through the container: the
    offset travels in the header and from_bytes scatters every outlier to its place."""
    s = sz()
    rng = np.random.default_rng(5)
    f = rng.standard_normal((24, 30, 100)).astype(np.float32)
    x = torch.from_numpy(f).cuda()
    mm = torch.tensor([-8.0, 8.0], dtype=torch.float64, device="cuda")   # a "global" range
    res = s.regression_compress(x, 1e-3, "rel", radius=64, d_minmax=mm, dim0_offset=600,
                                outlier_cap=x.numel()).finalize()
    assert res.n_outliers > 100
    direct = s.decompress(res)
    assert ((direct.double() - x.double()).abs().max().item()) <= res.eb_abs
    back = s.from_bytes(s.to_bytes(res, eb=1e-3, eb_mode="rel"))
    assert torch.equal(back.view(torch.int32), direct.view(torch.int32))


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_interp_bytes_round_trip(name):
    """SZ3-Interp results through the container (no coefficient sections): from_bytes takes the Interp
    decompressor and returns the direct decompression bit for bit."""
    s = sz()
    from synth import config_by_name, make_field
    cfg = config_by_name(name)
    x = make_field(cfg, device="cuda")
    res = s.interp_compress(x, cfg.eb, cfg.eb_mode, cfg.radius, outlier_cap=x.numel()).finalize()
    direct = s.interp_decompress(res.codes, res.outlier_idx, res.outlier_val, res.n_outliers, res.eb_abs, cfg.radius,
                                 x.dtype)
    b = s.to_bytes(res, eb=cfg.eb, eb_mode=cfg.eb_mode)
    back = s.from_bytes(b)
    assert back.shape == x.shape and torch.equal(back.view(torch.uint8), direct.view(torch.uint8))
    assert (back.double() - x.double()).abs().max().item() <= res.eb_abs
    print(name, "interp stream ratio", round(x.numel() * x.element_size() / len(b), 3))
