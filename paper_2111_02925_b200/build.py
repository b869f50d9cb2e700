"""Build libsz3g.so in-tree with nvcc for sm_100a (the .so travels to the GPU box with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "sz3g.cu")
SRCS = [SRC, os.path.join(HERE, "csrc", "huffman.cu"), os.path.join(HERE, "csrc", "truncation.cu"),
        os.path.join(HERE, "csrc", "metrics.cu"), os.path.join(HERE, "csrc", "coefcode.cu"),
        os.path.join(HERE, "csrc", "container.cu"), os.path.join(HERE, "csrc", "interp.cu")]
DEPS = [*SRCS, os.path.join(HERE, "csrc", "tile.cuh"), os.path.join(HERE, "csrc", "ptx.cuh"),
        os.path.join(HERE, "csrc", "lr.cuh"),
        os.path.join(ROOT, "include", "sz3g.h")]
LIB = os.path.join(HERE, "lib", "libsz3g.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CFLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]
LFLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static"]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def _obj_dir(out: str, defines) -> str:
    tag = "default" if not defines else "d" + format(abs(hash(tuple(defines))) % (1 << 32), "08x")
    return os.path.join(os.path.dirname(out), "obj", tag)


def build(force: bool = False, verbose: bool = False, src=None, out: str = LIB, defines=()) -> str:
    """nvcc `src` -> `out` (defaults: the in-tree library; another src/out builds an A/B variant).
    Each translation unit is compiled to its own object in parallel (a unit is recompiled only when it
    or a shared header changed, unless `force`), then linked with the static CUDA runtime."""
    if not force and out == LIB and not needs_build():
        return LIB
    os.makedirs(os.path.dirname(out), exist_ok=True)
    srcs = SRCS if src is None else ([src] if isinstance(src, str) else list(src))
    inc = ["-I", os.path.join(ROOT, "include")]
    cflags = [NVCC, *CFLAGS, *defines, *(["-Xptxas", "-v"] if verbose else []), *inc]
    odir = _obj_dir(out, defines) if src is None else os.path.join(os.path.dirname(out), "obj", "ab")
    os.makedirs(odir, exist_ok=True)
    hdr_t = max(os.path.getmtime(d) for d in DEPS if not d.endswith(".cu"))
    procs, objs = [], []
    for s in srcs:
        o = os.path.join(odir, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if not force and src is None and os.path.exists(o) and os.path.getmtime(o) > max(hdr_t, os.path.getmtime(s)):
            continue
        procs.append((s, subprocess.Popen([*cflags, "-c", "-o", o + ".tmp", s])))
    for s, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, f"nvcc {s}")
        os.replace(os.path.join(odir, os.path.basename(s)[:-3] + ".o.tmp"),
                   os.path.join(odir, os.path.basename(s)[:-3] + ".o"))
    tmp = out + f".tmp{os.getpid()}"
    subprocess.run([NVCC, *LFLAGS, "-o", tmp, *objs], check=True)
    os.replace(tmp, out)
    return out


CHAOS_LIB = os.path.join(HERE, "lib", "chaos", "libsz3g.so")


def chaos_lib(force: bool = False) -> str:
    """The race-detection build: -DSZ3G_CHAOS=2000 (random 0..2 us delays at every pipeline hand-off,
    csrc/ptx.cuh).  Test infrastructure only; the product loads LIB."""
    if force or not os.path.exists(CHAOS_LIB) or any(os.path.getmtime(d) > os.path.getmtime(CHAOS_LIB) for d in DEPS):
        build(force=True, out=CHAOS_LIB, defines=["-DSZ3G_CHAOS=2000"])
    return CHAOS_LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
