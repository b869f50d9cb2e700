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
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-cudart", "static"]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, src=None, out: str = LIB, defines=()) -> str:
    """nvcc `src` -> `out` (defaults: the in-tree library; another src/out builds an A/B variant)."""
    if not force and out == LIB and not needs_build():
        return LIB
    os.makedirs(os.path.dirname(out), exist_ok=True)
    tmp = out + f".tmp{os.getpid()}"
    srcs = SRCS if src is None else ([src] if isinstance(src, str) else list(src))
    cmd = [NVCC, *FLAGS, *defines, *(["-Xptxas", "-v"] if verbose else []), "-I", os.path.join(ROOT, "include"),
           "-o", tmp, *srcs]
    subprocess.run(cmd, check=True)
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
