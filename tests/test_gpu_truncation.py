"""GPU parity of SZ3-Truncation (NEXT-2: sz3g_truncation_*) with the oracle (DEFINITION.md T1-T2):
byte-exact streams and reconstructions for every k and both dtypes, ragged lengths (n mod 16 != 0),
n = 0 / 1, special values (NaN, +-Inf, -0, subnormals), the bench's c5 slab layout, bad k."""
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


def field(n, dt, seed):
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal(n) * 10.0 ** rng.integers(-30, 30, n)).astype(dt)
    if n >= 6:
        x[:6] = [np.nan, np.inf, -np.inf, -0.0, np.finfo(dt).tiny / 4, -np.finfo(dt).max]
    return x


@pytest.mark.parametrize("dt,s", [(np.float32, 4), (np.float64, 8)])
@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 1000, 123_457])
def test_parity_all_k(dt, s, n):
    x = field(n, dt, n)
    xt = torch.from_numpy(x).cuda()
    for k in range(1, s + 1):
        b = sz().truncation_compress(xt, k)
        y = sz().truncation_decompress(b, n, k, xt.dtype)
        torch.cuda.synchronize()
        ob = oracle.trunc_compress(x, k)
        assert np.array_equal(b.cpu().numpy(), ob), (k, "stream")
        oy = oracle.trunc_decompress(ob, n, k, dt)
        assert np.array_equal(y.cpu().numpy().view(np.uint8), oy.view(np.uint8)), (k, "reconstruction")


def test_config_field_k2():
    from synth import config_by_name, make_field
    cfg = config_by_name("c2")
    x = make_field(cfg, device="cuda").reshape(-1)
    b = sz().truncation_compress(x, 2)
    y = sz().truncation_decompress(b, x.numel(), 2)
    xh = x.cpu().numpy()
    assert np.array_equal(b.cpu().numpy(), oracle.trunc_compress(xh, 2))
    assert np.array_equal(y.cpu().numpy(), oracle.trunc_decompress(oracle.trunc_compress(xh, 2), xh.size, 2, np.float32))


def test_bad_k():
    x = torch.ones(32, device="cuda")
    with pytest.raises(Exception):
        sz().truncation_compress(x, 5)
    with pytest.raises(Exception):
        sz().truncation_compress(x, 0)
