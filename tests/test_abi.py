"""The C-ABI library loads and exports every symbol include/sz3g.h declares; host-side argument
validation works without a GPU (no compute calls here).  CPU only."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sz3g.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sz3g_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2111_02925_b200 import build, sz3g
    build.build()
    return sz3g.load()


def test_header_declares_the_north_star_calls():
    syms = header_symbols()
    for s in ("sz3g_regression_compress", "sz3g_regression_decompress", "sz3g_histogram", "sz3g_value_range"):
        assert s in syms


def test_library_exports_every_header_symbol(lib):
    from paper_2111_02925_b200 import sz3g
    for s in header_symbols():
        assert hasattr(lib, s), s
    assert set(header_symbols()) == set(sz3g.EXPORTED_SYMBOLS)
    nm = os.popen(f"nm -D --defined-only {sz3g.lib_path()}").read()
    for s in header_symbols():
        assert re.search(rf"\bT {s}\b", nm), s


def test_host_validation_without_gpu(lib):
    from paper_2111_02925_b200 import sz3g
    g = sz3g.make_grid((10, 10, 10), __import__("torch").float32)
    p = sz3g.make_params(1e-3, "abs", 32768)
    # null pointers -> EINVAL, before any CUDA call
    assert lib.sz3g_regression_compress(None, None, None, None, None, None, None, None, None, 0, None, None,
                                        None, None, None) == -1
    assert lib.sz3g_regression_compress(ctypes.byref(g), ctypes.byref(p), None, None, None, None, None, None,
                                        None, 0, None, None, None, None, None) == -1
    bad = sz3g.make_params(1e-3, "abs", 40000)
    x = ctypes.c_void_p(16)
    assert lib.sz3g_regression_compress(ctypes.byref(g), ctypes.byref(bad), x, None, x, x, None, None, None, 0,
                                        x, None, None, x, None) == -3
    b5 = sz3g.Params(5, 32768, 0, 1e-3, 0)
    assert lib.sz3g_regression_compress(ctypes.byref(g), ctypes.byref(b5), x, None, x, x, None, None, None, 0,
                                        x, None, None, x, None) == -2
    neg = sz3g.make_params(-1.0, "abs", 16)
    assert lib.sz3g_regression_compress(ctypes.byref(g), ctypes.byref(neg), x, None, x, x, None, None, None, 0,
                                        x, None, None, x, None) == -1
    z = sz3g.make_grid((0, 10, 10), __import__("torch").float32)
    assert lib.sz3g_value_range(ctypes.byref(z), x, x, None) == -1
    assert lib.sz3g_histogram(None, 10, 16, x, None) == -1
    assert lib.sz3g_histogram(x, 10, 0, x, None) == -3
    assert lib.sz3g_num_blocks(ctypes.byref(g), 6) == 8
    assert lib.sz3g_strerror(-3) == b"radius out of range [1, 32768]"


def test_num_blocks_matches_oracle(lib):
    import oracle
    from paper_2111_02925_b200 import sz3g
    for shape in [(64, 64, 64), (100, 500, 500), (1024, 2048, 2048), (1, 1, 5), (7, 7, 7)]:
        assert sz3g.num_blocks(shape) == oracle.num_blocks(shape)


def test_product_path_has_no_oracle_or_cpu_fallback():
    """The product package never imports oracle/ and has no CPU compute path."""
    pkg = os.path.join(ROOT, "paper_2111_02925_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "sz3_oracle" not in src, f
