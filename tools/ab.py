#!/usr/bin/env python
"""A/B timing of library variants on the GPU: alternate processes of tools/tune.py, one per variant
(SZ3G_LIB=<path>), so that power-cap / clock drift hits every variant alike.

  python tools/ab.py --config c5 --rounds 4 A=lib/ab/A.so B=paper_2111_02925_b200/lib/libsz3g.so
  python tools/ab.py --build A=<git-rev>      (here: builds <git-rev>'s sz3g.cu into lib/ab/A.so)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_rev(name: str, rev: str):
    """rev = a git revision, or "@" (the working tree) followed by space-separated -D defines"""
    import tempfile
    sys.path.insert(0, ROOT)
    from paper_2111_02925_b200 import build as B
    out = os.path.join(ROOT, "paper_2111_02925_b200", "lib", "ab", f"{name}.so")
    if rev.startswith("@"):
        B.build(force=True, out=out, defines=rev[1:].split())
        print("built", name, rev, "->", out)
        return
    d = tempfile.mkdtemp()
    files = subprocess.run(["git", "ls-tree", "-r", "--name-only", rev, "paper_2111_02925_b200/csrc", "include"],
                           cwd=ROOT, capture_output=True, text=True, check=True).stdout.split()
    for f in files:
        os.makedirs(os.path.join(d, os.path.dirname(f)), exist_ok=True)
        src = subprocess.run(["git", "show", f"{rev}:{f}"], cwd=ROOT, capture_output=True, text=True, check=True).stdout
        open(os.path.join(d, f), "w").write(src)
    B.build(force=True, src=[os.path.join(d, f) for f in files if f.endswith(".cu")], out=out)
    print("built", name, rev, "->", out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--setting", default="")
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--path", default="fused", choices=["fused", "two-pass"])
    ap.add_argument("--tool", default="tune.py", help="tools/<tool> printing tune.py's JSON (e.g. huff_time.py)")
    ap.add_argument("--flush", action="store_true")
    ap.add_argument("--graphs", action="store_true")
    ap.add_argument("variants", nargs="+")
    a = ap.parse_args()
    vs = [v.split("=", 1) for v in a.variants]
    if a.build:
        for n, rev in vs:
            build_rev(n, rev)
        return
    res = {n: ([], [], []) for n, _ in vs}
    for r in range(a.rounds):
        for n, path in vs:
            env = dict(os.environ, SZ3G_LIB=os.path.join(ROOT, path) if not os.path.isabs(path) else path)
            out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", a.tool), "--config", a.config,
                                  "--reps", str(a.reps), "--rounds", "1", "--path", a.path,
                                  *(["--flush"] if a.flush else []), *(["--graphs"] if a.graphs else []),
                                  a.setting or "CHUNK_C=2"],
                                 env=env, capture_output=True, text=True)
            line = [l for l in out.stdout.splitlines() if l.startswith("{")]
            if not line:
                print(n, "FAILED", out.stderr[-2000:], flush=True)
                continue
            d = json.loads(line[-1])
            res[n][0].append(d["compress_ms"][0])
            res[n][1].append(d["decompress_ms"][0])
            res[n][2].append(d.get("analyze_ms", [0.0])[0])
            print(json.dumps({"round": r, "variant": n, "compress_ms": d["compress_ms"][0],
                              "decompress_ms": d["decompress_ms"][0], "analyze_ms": res[n][2][-1]}), flush=True)
    for n, (c, dd, aa) in res.items():
        if c:
            print(json.dumps({"variant": n, "compress_median_ms": statistics.median(c), "compress_min_ms": min(c),
                              "decompress_median_ms": statistics.median(dd),
                              "analyze_median_ms": statistics.median(aa)}))


if __name__ == "__main__":
    main()
