"""The reported counters (north_star: near-ties "are counted, and the count is reported"; SURVEY 8(c)
"Reported counters" (i)-(iii)) computed on the GPU by sz3g_tie_counts equal the oracle's counters
exactly when both use the same coefficient codes and beta (the oracle's)."""
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


def gpu_counts(xh, eb, mode, R, orc):
    s = sz()
    x = torch.from_numpy(np.ascontiguousarray(xh)).cuda()
    mm = s.value_range(x) if mode == "rel" else None
    cc = torch.from_numpy(orc.coef_codes.reshape(-1, 4).copy()).cuda()
    beta = torch.from_numpy(orc.coef_raw.reshape(-1, 4).copy()).cuda()
    return s.tie_counts(x, eb, mode, R, mm, cc, beta).cpu().tolist()


def expected(orc):
    from paper_2111_02925_b200.sz3g import TIE_COUNTER_NAMES
    return [int(orc.counters[k]) for k in TIE_COUNTER_NAMES]


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_tie_counts_match_oracle_configs(name):
    from synth import config_by_name, make_field
    cfg = config_by_name(name)
    xh = make_field(cfg, device="cuda").cpu().numpy()
    orc = oracle.compress(xh, cfg.eb, cfg.eb_mode, radius=cfg.radius)
    assert gpu_counts(xh, cfg.eb, cfg.eb_mode, cfg.radius, orc) == expected(orc)


def test_tie_counts_adversarial():
    from tests.test_gpu_parity import adversarial_case
    for kind in ("half_bins", "near_half", "offset", "wide_range"):
        f, eb, mode, R = adversarial_case(kind)
        orc = oracle.compress(f, eb, mode, radius=R)
        got = gpu_counts(f, eb, mode, R, orc)
        assert got == expected(orc), kind
        if kind == "half_bins":
            assert got[0] == f.size
    # checkerboard (P7): every element a tie
    dims = (12, 18, 96)
    i, j, k = np.meshgrid(*[np.arange(n) for n in dims], indexing="ij")
    f = ((-1.0) ** (i + j + k)).astype(np.float32)
    orc = oracle.compress(f, 1.0, "abs", radius=32768)
    assert gpu_counts(f, 1.0, "abs", 32768, orc) == expected(orc) and expected(orc)[0] == f.size


@pytest.mark.parametrize("delta,flagged", [(2.0 ** -43, 1), (5e-7, 0)])
def test_tie_counts_coefficient_window(delta, flagged):
    f = np.full((12, 6, 18), 1.25 + delta, dtype=np.float64)    # 6 constant blocks, beta0 / w0 = 2.5 + 2 delta
    orc = oracle.compress(f, 1.0, "abs", radius=32768)
    got = gpu_counts(f, 1.0, "abs", 32768, orc)
    assert got == expected(orc) and got[3] == 6 * flagged
