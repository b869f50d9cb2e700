"""GPU parity of the coefficient-code delta coding (NEXT-3: sz3g_coef_delta_*) with the oracle
(DEFINITION.md C1-C2): symbols and escapes bit-exact, decode exact, the full chain through the Huffman
stage on the configs' real coefficient codes, escapes at int32 extremes, nb not a multiple of the
tile, nb = 0 / 1."""
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


@pytest.mark.parametrize("nb", [1, 7, 2048, 2049, 100_003])
def test_delta_parity(nb):
    rng = np.random.default_rng(nb)
    coef = rng.integers(-40, 40, size=(nb, 4)).cumsum(axis=0).astype(np.int32)
    if nb > 10:
        coef[5] = [2**31 - 1, -2**31, 0, 1]
        coef[6] = [-2**31, 2**31 - 1, 123456, 1]
    c = torch.from_numpy(coef).cuda()
    sym, esc = sz().coef_delta_encode(c)
    osym, oesc = oracle.coef_delta_encode(coef)
    assert np.array_equal(sym.cpu().numpy(), osym)
    assert np.array_equal(esc.cpu().numpy().view(np.uint64), oesc)
    back = sz().coef_delta_decode(sym, nb, esc)
    torch.cuda.synchronize()
    assert np.array_equal(back.cpu().numpy(), coef)


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_config_coefficients_through_huffman(name):
    s = sz()
    from synth import config_by_name, make_field
    cfg = config_by_name(name)
    x = make_field(cfg, device="cuda")
    res = s.compress(x, cfg.eb, cfg.eb_mode, cfg.radius)
    cs = s.encode_coefficients(res.coef_codes)
    back = s.decode_coefficients(cs)
    torch.cuda.synchronize()
    assert torch.equal(back, res.coef_codes)
    raw = res.coef_codes.numel() * 4
    print(name, "coefficient bytes", raw, "->", cs.nbytes(), f"({raw / cs.nbytes():.1f}x)")
    assert cs.nbytes() < raw


@pytest.mark.parametrize("lo", [0, 100, 60000])
def test_histogram_bins_window(lo):
    rng = np.random.default_rng(lo)
    sym = np.minimum(rng.geometric(0.05, size=1_000_003) - 1 + (lo // 2), 65535).astype(np.uint16)
    h = sz().histogram_bins(torch.from_numpy(sym).cuda(), 65536, lo).cpu().numpy()
    assert np.array_equal(h, np.bincount(sym, minlength=65536))
    h2 = sz().histogram_bins(torch.from_numpy(sym).cuda(), 300, lo).cpu().numpy()   # symbols >= nbins ignored
    assert np.array_equal(h2, np.bincount(sym[sym < 300], minlength=300))
