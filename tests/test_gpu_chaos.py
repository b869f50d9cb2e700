"""Race detection without compute-sanitizer (closed on this pool): the chaos build of
the library (-DSZ3G_CHAOS=2000: a pseudo-random 0..2 us sleep at every mbarrier arrive / completed
wait, TMA issue, bulk-group wait, cp.async wait, __syncwarp and __syncthreads) must produce outputs
bit-identical to the normal build on every kernel family (tools/digest_cases.py: regression analyze /
quantise / fused / decompress in TMA and plain variants at R = 32768 and 8, SZ3-LR, value range,
histogram, Huffman codebook / encode / decode incl. ragged tails, coefficient coding, truncation, error
statistics, tie counters, the stream container), in repeated runs (different interleavings)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def digest(lib: str) -> dict:
    env = dict(os.environ, SZ3G_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "digest_cases.py")], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_chaos_build_is_bit_identical():
    from paper_2111_02925_b200 import build
    normal = digest(build.LIB)
    chaos_lib = build.chaos_lib()
    for rep in range(2):
        chaos = digest(chaos_lib)
        assert chaos["_lib"] == chaos_lib
        bad = [k for k in normal if not k.startswith("_") and chaos.get(k) != normal[k]]
        assert not bad, f"run {rep}: {len(bad)} outputs differ under injected delays, e.g. {bad[:8]}"
    print(f"{len(normal) - 2} digests identical; launches per run {normal['_launches']}")
