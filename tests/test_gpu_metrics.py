"""GPU parity of sz3g_error_stats (DEFINITION.md M1) with the oracle, and the metric chain on a real
round trip (bound holds: no element above eb, max error <= eb)."""
from __future__ import annotations

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402

pytestmark = pytest.mark.gpu


def sz():
    from paper_2111_02925_b200 import sz3g
    sz3g.load()
    return sz3g


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("n", [0, 1, 7, 4096, 1_000_003])
def test_error_stats_parity(dt, n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n).astype(dt)
    y = (x + rng.standard_normal(n) * 1e-3).astype(dt)
    if n > 10:
        y[:5] = x[:5]
        x[5] = y[5] = np.nan
        x[6] = y[6] = -np.inf
    got = sz().error_stats(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), 2e-3).cpu().numpy()
    mx, sq, cnt = oracle.error_stats(x, y, 2e-3)
    assert got[0] == mx                                   # max: exact
    assert abs(got[1] - sq) <= 1e-12 * max(sq, 1e-300)    # fp64 sum, another order
    assert got[2] == cnt


def test_round_trip_metrics_c2():
    s = sz()
    from synth import config_by_name, make_field
    cfg = config_by_name("c2")
    x = make_field(cfg, device="cuda")
    res = s.compress(x, cfg.eb, cfg.eb_mode, cfg.radius)
    xo = s.decompress(res)
    st = s.error_stats(x, xo, res.eb_abs).cpu().numpy()
    assert st[0] <= res.eb_abs and st[2] == 0
    lo, hi = (float(v) for v in s.value_range(x).cpu())
    p = s.psnr(hi - lo, st[1] / x.numel())
    # uniform error within +-eb: MSE ~ eb^2 / 3 -> PSNR ~ 20 log10(range / eb) + 4.77 dB
    assert abs(p - (20 * math.log10((hi - lo) / res.eb_abs) + 10 * math.log10(3))) < 1.0
