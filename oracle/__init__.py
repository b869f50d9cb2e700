"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper around the plain C++ oracle (oracle/*.cpp).

The oracle is the single-threaded CPU definition of SZ3's block-regression predictor with
linear-scaling quantisation (sz3_oracle.cpp: PAPER.md Lemma 1, prediction P:156, quantiser
P:406-409, App. A loop P:980-992, value-range eb P:833), of the Huffman encoder stage
(huffman_oracle.cpp: P:156), of SZ3-Truncation and the coefficient delta coding
(truncation_oracle.cpp: P:848-850) and of the distortion metrics (below: P:525); the exact
definitions are oracle/DEFINITION.md (O1-O11, D, H1-H5, T1-T2, C1-C2, M1-M3, L1-L7: SZ3-LR, P:845,
I1-I6: SZ3-Interp).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this package.  It shares
no code with ``paper_2111_02925_b200`` and never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sz3_oracle.cpp")
_SRCS = [_SRC, os.path.join(_HERE, "huffman_oracle.cpp"), os.path.join(_HERE, "truncation_oracle.cpp")]
_LIB_PATH = os.path.join(_HERE, "liboracle_sz3.so")
_lock = threading.Lock()
_lib = None

OK, EINVAL, EUNSUPPORTED, ERANGE, EBADRANGE, EOVERFLOW = 0, -1, -2, -3, -5, -6
BLOCK = 6


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (-O2, no FP contraction)."""
    if force or not os.path.exists(_LIB_PATH) or any(os.path.getmtime(_LIB_PATH) < os.path.getmtime(f) for f in _SRCS):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-o", tmp, *_SRCS]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class Counters(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "elem_near_ties", "elem_div_mismatch", "coef_near_ties", "coef_tie_blocks",
        "radius_outliers", "verify_outliers", "nonfinite_outliers", "zero_predictor_blocks")]

    def as_dict(self) -> dict:
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P, U64, U32, I32, D = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_double
            lib.orc_value_range.argtypes = [I32, U64, P, P]
            lib.orc_compress.argtypes = [I32, P, U64, U32, U32, I32, D, P, P, P, P, P, P, P, P, U64, P, P, P, P, P]
            lib.orc_decompress.argtypes = [I32, P, U64, U32, U32, D, P, P, P, P, U64, P]
            lib.orc_block_beta.argtypes = [P, I32, I32, I32, P, P]
            lib.orc_block_beta.restype = None
            lib.orc_coef_codes.argtypes = [P, D, U32, P, P]
            lib.orc_predict.argtypes = [P, I32, I32, I32]
            lib.orc_predict.restype = D
            lib.orc_quantize_element.argtypes = [I32, D, D, D, U32, P, P]
            lib.orc_num_blocks.argtypes = [P, U32]
            lib.orc_num_blocks.restype = U64
            lib.orc_huffman_lengths.argtypes = [P, U32, U32, P]
            lib.orc_huffman_canonical.argtypes = [P, U32, P]
            lib.orc_huffman_canonical.restype = None
            lib.orc_huffman_chunk_offsets.argtypes = [P, U64, U32, P, P]
            lib.orc_huffman_chunk_offsets.restype = None
            lib.orc_huffman_encode.argtypes = [P, U64, U32, P, P, P, P]
            lib.orc_huffman_decode.argtypes = [P, P, U64, U32, P, P, U32, P]
            lib.orc_trunc_compress.argtypes = [I32, U64, P, U32, P]
            lib.orc_trunc_decompress.argtypes = [I32, U64, P, U32, P]
            lib.orc_coef_delta_encode.argtypes = [P, U64, P, P, U64]
            lib.orc_coef_delta_encode.restype = U64
            lib.orc_coef_delta_decode.argtypes = [P, U64, P, U64, P]
            lib.orc_lr_compress.argtypes = [I32, P, U64, U32, U32, I32, D, P, P, P, P, P, P, P, P, P, U64, P, P, P,
                                            P, P]
            lib.orc_lr_decompress.argtypes = [I32, P, U64, U32, U32, D, P, P, P, P, P, U64, P]
            lib.orc_interp_compress.argtypes = [I32, P, U64, U32, I32, D, P, P, P, P, P, U64, P, P, P, P, P]
            lib.orc_interp_decompress.argtypes = [I32, P, U64, U32, D, P, P, P, U64, P]
            lib.orc_interp_predict.argtypes = [D, D, D, D, I32]
            lib.orc_interp_predict.restype = D
            lib.orc_interp_pass_of.argtypes = [P, U64, U64, U64]
            lib.orc_interp_pass_of.restype = ctypes.c_int64
            lib.orc_lr_delta.argtypes = [P, I32, I32, I32, I32, I32, I32]
            lib.orc_lr_delta.restype = ctypes.c_int64
            _lib = lib
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _dtype_id(dt) -> int:
    dt = np.dtype(dt)
    if dt == np.float32:
        return 0
    if dt == np.float64:
        return 1
    raise ValueError(f"unsupported dtype {dt}")


def num_blocks(dims, B: int = BLOCK) -> int:
    d = np.ascontiguousarray(dims, dtype=np.uint64)
    return int(_load().orc_num_blocks(_ptr(d), B))


def value_range(x: np.ndarray) -> tuple[float, float]:
    x = np.ascontiguousarray(x)
    out = np.zeros(2, np.float64)
    rc = _load().orc_value_range(_dtype_id(x.dtype), x.size, _ptr(x), _ptr(out))
    if rc != OK:
        raise ValueError(f"orc_value_range rc={rc}")
    return float(out[0]), float(out[1])


@dataclass
class Compressed:
    dims: tuple
    dtype: np.dtype
    radius: int
    eb_abs: float
    codes: np.ndarray          # uint16, same shape as the field
    coef_codes: np.ndarray     # int32 [NB, 4]
    coef_raw: np.ndarray       # float64 [NB, 4]  unquantised beta
    block_exempt: np.ndarray   # uint8 [NB] coefficient near-tie blocks
    outlier_idx: np.ndarray    # uint64 global linear index, emission order (block-major)
    outlier_val: np.ndarray    # T
    hist: np.ndarray           # int64 [2R]
    counters: dict = field(default_factory=dict)
    dim0_offset: int = 0
    xprime: np.ndarray | None = None   # compress-time reconstruction (T), same shape as the field


def compress(x: np.ndarray, eb: float, eb_mode: str = "rel", radius: int = 32768,
             dim0_offset: int = 0, value_range_override: tuple | None = None,
             B: int = BLOCK) -> Compressed:
    """Oracle O1-O11 over a 3D field (1D/2D are embedded with leading extents 1, DESIGN G18)."""
    x = np.ascontiguousarray(x)
    shape = (1,) * (3 - x.ndim) + tuple(x.shape)
    dims = np.array(shape, np.uint64)
    N = int(np.prod(shape))
    nb = num_blocks(dims, B)
    codes = np.empty(shape, np.uint16)
    coef = np.empty((nb, 4), np.int32)
    coef_raw = np.empty((nb, 4), np.float64)
    exempt = np.empty(nb, np.uint8)
    cap = N
    oidx = np.empty(cap, np.uint64)
    oval = np.empty(cap, x.dtype)
    nout = np.zeros(1, np.uint64)
    hist = np.empty(2 * radius, np.int64)
    eb_abs = np.zeros(1, np.float64)
    xprime = np.empty(shape, x.dtype)
    cnt = Counters()
    rng = None if value_range_override is None else np.array(value_range_override, np.float64)
    mode = {"abs": 0, "rel": 1}[eb_mode]
    rc = _load().orc_compress(_dtype_id(x.dtype), _ptr(dims), dim0_offset, B, radius, mode, float(eb),
                              _ptr(rng), _ptr(x), _ptr(codes), _ptr(coef), _ptr(coef_raw), _ptr(exempt),
                              _ptr(oidx), _ptr(oval), cap, _ptr(nout), _ptr(hist), _ptr(eb_abs),
                              ctypes.byref(cnt), _ptr(xprime))
    if rc != OK:
        raise ValueError(f"orc_compress rc={rc}")
    n = int(nout[0])
    return Compressed(tuple(int(s) for s in shape), x.dtype, radius, float(eb_abs[0]), codes, coef, coef_raw,
                      exempt, oidx[:n].copy(), oval[:n].copy(), hist, cnt.as_dict(), dim0_offset, xprime)


def decompress(c: Compressed | None = None, *, dims=None, dtype=None, radius=None, eb_abs=None, codes=None,
               coef_codes=None, outlier_idx=None, outlier_val=None, dim0_offset=0, B: int = BLOCK) -> np.ndarray:
    if c is not None:
        dims, dtype, radius, eb_abs = c.dims, c.dtype, c.radius, c.eb_abs
        codes, coef_codes, outlier_idx, outlier_val, dim0_offset = (
            c.codes, c.coef_codes, c.outlier_idx, c.outlier_val, c.dim0_offset)
    d = np.array(dims, np.uint64)
    out = np.empty(tuple(int(s) for s in dims), dtype)
    codes = np.ascontiguousarray(codes, np.uint16)
    coef_codes = np.ascontiguousarray(coef_codes, np.int32)
    oidx = np.ascontiguousarray(outlier_idx, np.uint64)
    oval = np.ascontiguousarray(outlier_val, dtype)
    rc = _load().orc_decompress(_dtype_id(dtype), _ptr(d), dim0_offset, B, radius, float(eb_abs), _ptr(codes),
                                _ptr(coef_codes), _ptr(oidx), _ptr(oval), oidx.size, _ptr(out))
    if rc != OK:
        raise ValueError(f"orc_decompress rc={rc}")
    return out


def block_beta(f: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """O4 + O5 on one dense block; returns (V0,Vx,Vy,Vz), (b0,b1,b2,b3)."""
    f = np.ascontiguousarray(f, np.float64)
    assert f.ndim == 3
    V = np.zeros(4)
    beta = np.zeros(4)
    _load().orc_block_beta(_ptr(f), f.shape[0], f.shape[1], f.shape[2], _ptr(V), _ptr(beta))
    return V, beta


def coef_codes(beta, eb_abs: float, B: int = BLOCK):
    b = np.ascontiguousarray(beta, np.float64)
    c = np.zeros(4, np.int32)
    bh = np.zeros(4)
    zero = _load().orc_coef_codes(_ptr(b), float(eb_abs), B, _ptr(c), _ptr(bh))
    return c, bh, bool(zero)


def predict(bhat, i: int, j: int, k: int) -> float:
    b = np.ascontiguousarray(bhat, np.float64)
    return float(_load().orc_predict(_ptr(b), i, j, k))


def quantize_element(x: float, p: float, eb_abs: float, radius: int = 32768, dtype=np.float64):
    """O8-O10 for one element; returns (code, x', kind) with kind 0 ok / 1 radius / 2 verify / 3 non-finite."""
    code = ctypes.c_uint16(0)
    xp = ctypes.c_double(0)
    kind = _load().orc_quantize_element(_dtype_id(dtype), float(x), float(p), float(eb_abs), radius,
                                        ctypes.byref(code), ctypes.byref(xp))
    return int(code.value), float(xp.value), int(kind)


# ------------------------------------------------------------------------------------------- Huffman
# The encoder stage after the quantiser (DEFINITION.md H1-H5; huffman_oracle.cpp).
HUFF_MAX_LEN = 16    # G20: length limit of the codebook
HUFF_CHUNK = 2048    # G21: codes per independently decodable chunk


def huffman_lengths(hist: np.ndarray, max_len: int = HUFF_MAX_LEN) -> np.ndarray:
    """H2: optimal code lengths under max_len by package-merge (uint8 per symbol, 0 = absent)."""
    h = np.ascontiguousarray(hist, dtype=np.int64)
    lens = np.zeros(h.size, np.uint8)
    rc = _load().orc_huffman_lengths(_ptr(h), h.size, max_len, _ptr(lens))
    if rc != 0:
        raise ValueError(f"orc_huffman_lengths failed ({rc})")
    return lens


def huffman_canonical(lens: np.ndarray) -> np.ndarray:
    """H3: canonical codewords (uint32, right-aligned) for the given lengths."""
    L = np.ascontiguousarray(lens, dtype=np.uint8)
    codes = np.zeros(L.size, np.uint32)
    _load().orc_huffman_canonical(_ptr(L), L.size, _ptr(codes))
    return codes


def huffman_encode(q: np.ndarray, lens: np.ndarray, codes: np.ndarray, chunk: int = HUFF_CHUNK):
    """H4: (chunk word offsets uint64[nchunks + 1], payload uint32[offs[-1]])."""
    q = np.ascontiguousarray(q, dtype=np.uint16).reshape(-1)
    lens = np.ascontiguousarray(lens, dtype=np.uint8)
    codes = np.ascontiguousarray(codes, dtype=np.uint32)
    nch = -(-q.size // chunk)
    offs = np.zeros(nch + 1, np.uint64)
    _load().orc_huffman_chunk_offsets(_ptr(q), q.size, chunk, _ptr(lens), _ptr(offs))
    words = np.zeros(int(offs[-1]), np.uint32)
    rc = _load().orc_huffman_encode(_ptr(q), q.size, chunk, _ptr(lens), _ptr(codes), _ptr(offs), _ptr(words))
    if rc != 0:
        raise ValueError("a code has no codeword")
    return offs, words


def huffman_decode(words: np.ndarray, offs: np.ndarray, n: int, lens: np.ndarray, codes: np.ndarray,
                   chunk: int = HUFF_CHUNK) -> np.ndarray:
    """H5: decode n codes."""
    words = np.ascontiguousarray(words, dtype=np.uint32)
    offs = np.ascontiguousarray(offs, dtype=np.uint64)
    lens = np.ascontiguousarray(lens, dtype=np.uint8)
    codes = np.ascontiguousarray(codes, dtype=np.uint32)
    q = np.zeros(n, np.uint16)
    rc = _load().orc_huffman_decode(_ptr(words), _ptr(offs), n, chunk, _ptr(lens), _ptr(codes), lens.size, _ptr(q))
    if rc != 0:
        raise ValueError(f"corrupt stream ({rc})")
    return q


# ------------------------------------------------------------------------------------------- Truncation
# SZ3-Truncation (DEFINITION.md T1-T2; truncation_oracle.cpp).
def trunc_compress(x: np.ndarray, k: int) -> np.ndarray:
    """T1: the k most-significant bytes of every element, most significant first (uint8[n*k])."""
    x = np.ascontiguousarray(x).reshape(-1)
    out = np.zeros(x.size * k, np.uint8)
    rc = _load().orc_trunc_compress(_dtype_id(x.dtype), x.size, _ptr(x), k, _ptr(out))
    if rc != 0:
        raise ValueError(f"orc_trunc_compress failed ({rc})")
    return out


def trunc_decompress(b: np.ndarray, n: int, k: int, dtype) -> np.ndarray:
    """T2: zero-fill the discarded bytes."""
    b = np.ascontiguousarray(b, dtype=np.uint8)
    x = np.zeros(n, dtype)
    rc = _load().orc_trunc_decompress(_dtype_id(dtype), n, _ptr(b), k, _ptr(x))
    if rc != 0:
        raise ValueError(f"orc_trunc_decompress failed ({rc})")
    return x


# ------------------------------------------------------------------------------------------- metrics
# Distortion metrics (DEFINITION.md M1-M3).
def error_stats(x: np.ndarray, y: np.ndarray, eb: float = float("inf")) -> tuple[float, float, int]:
    """M1: (max |x - y|, sum (x - y)^2, #(|x - y| > eb)) in fp64; bitwise-identical pairs contribute 0."""
    x = np.ascontiguousarray(x).reshape(-1)
    y = np.ascontiguousarray(y).reshape(-1)
    if x.size == 0:
        return 0.0, 0.0, 0
    same = x.view(np.uint8).reshape(x.size, -1) == y.view(np.uint8).reshape(y.size, -1)
    diff = np.where(same.all(axis=1), 0.0, x.astype(np.float64) - y.astype(np.float64))
    ad = np.abs(diff)
    mx = float(np.nan) if np.isnan(ad).any() else float(ad.max(initial=0.0))
    return mx, float(np.sum(diff * diff)), int(np.sum((ad > eb) | np.isnan(ad)))


def psnr(value_range: float, mse: float) -> float:
    """M2: 20 log10(range) - 10 log10(MSE); +inf for MSE = 0."""
    import math
    if mse == 0:
        return math.inf
    return 20.0 * math.log10(value_range) - 10.0 * math.log10(mse)


def bit_rate(bits_per_sample: int, ratio: float) -> float:
    """M3: bits / cr."""
    return bits_per_sample / ratio


# ------------------------------------------------------------------------------------------- coefficient deltas
# NEXT-3 coefficient-code delta coding (DEFINITION.md C1-C2, truncation_oracle.cpp).
COEF_ESC = 65535


def coef_delta_encode(coef: np.ndarray):
    """C1: (sym uint16 [4 * nb] channel-major, escapes uint64 in position order)."""
    c = np.ascontiguousarray(coef, dtype=np.int32).reshape(-1, 4)
    nb = c.shape[0]
    sym = np.zeros(4 * nb, np.uint16)
    esc = np.zeros(4 * nb, np.uint64)
    ne = _load().orc_coef_delta_encode(_ptr(c), nb, _ptr(sym), _ptr(esc), esc.size)
    return sym, esc[:ne].copy()


def coef_delta_decode(sym: np.ndarray, nb: int, esc: np.ndarray) -> np.ndarray:
    """C2: back to int32 [nb, 4]."""
    sym = np.ascontiguousarray(sym, dtype=np.uint16)
    esc = np.ascontiguousarray(esc, dtype=np.uint64)
    c = np.zeros((nb, 4), np.int32)
    if _load().orc_coef_delta_decode(_ptr(sym), nb, _ptr(esc), esc.size, _ptr(c)) != 0:
        raise ValueError("escapes exhausted")
    return c


# ------------------------------------------------------------------------------------------- SZ3-LR
# The composite Lorenzo / regression predictor (DEFINITION.md L1-L7; sz3_oracle.cpp lr_*).
@dataclass
class LRCompressed(Compressed):
    flags: np.ndarray | None = None    # uint8 [NB]: 1 = Lorenzo block, 0 = regression block
    n_lorenzo: int = 0


def lr_compress(x: np.ndarray, eb: float, eb_mode: str = "rel", radius: int = 32768, dim0_offset: int = 0,
                value_range_override: tuple | None = None, B: int = BLOCK) -> LRCompressed:
    """L1-L6 over a 3D field (1D/2D embedded with leading extents 1)."""
    x = np.ascontiguousarray(x)
    shape = (1,) * (3 - x.ndim) + tuple(x.shape)
    dims = np.array(shape, np.uint64)
    N = int(np.prod(shape))
    nb = num_blocks(dims, B)
    codes = np.empty(shape, np.uint16)
    coef = np.empty((nb, 4), np.int32)
    coef_raw = np.empty((nb, 4), np.float64)
    exempt = np.empty(nb, np.uint8)
    flags = np.empty(nb, np.uint8)
    oidx = np.empty(N, np.uint64)
    oval = np.empty(N, x.dtype)
    nout = np.zeros(1, np.uint64)
    nlor = np.zeros(1, np.uint64)
    hist = np.empty(2 * radius, np.int64)
    eb_abs = np.zeros(1, np.float64)
    xprime = np.empty(shape, x.dtype)
    rng = None if value_range_override is None else np.array(value_range_override, np.float64)
    rc = _load().orc_lr_compress(_dtype_id(x.dtype), _ptr(dims), dim0_offset, B, radius, {"abs": 0, "rel": 1}[eb_mode],
                                 float(eb), _ptr(rng), _ptr(x), _ptr(codes), _ptr(coef), _ptr(coef_raw), _ptr(exempt),
                                 _ptr(flags), _ptr(oidx), _ptr(oval), N, _ptr(nout), _ptr(hist), _ptr(eb_abs),
                                 _ptr(xprime), _ptr(nlor))
    if rc != OK:
        raise ValueError(f"orc_lr_compress rc={rc}")
    n = int(nout[0])
    return LRCompressed(tuple(int(s) for s in shape), x.dtype, radius, float(eb_abs[0]), codes, coef, coef_raw,
                        exempt, oidx[:n].copy(), oval[:n].copy(), hist, {}, dim0_offset, xprime, flags,
                        int(nlor[0]))


def lr_decompress(c: LRCompressed | None = None, *, dims=None, dtype=None, radius=None, eb_abs=None, codes=None,
                  coef_codes=None, flags=None, outlier_idx=None, outlier_val=None, dim0_offset=0,
                  B: int = BLOCK) -> np.ndarray:
    """L7."""
    if c is not None:
        dims, dtype, radius, eb_abs = c.dims, c.dtype, c.radius, c.eb_abs
        codes, coef_codes, flags, outlier_idx, outlier_val, dim0_offset = (
            c.codes, c.coef_codes, c.flags, c.outlier_idx, c.outlier_val, c.dim0_offset)
    d = np.array(dims, np.uint64)
    out = np.zeros(tuple(int(s) for s in dims), dtype)
    codes = np.ascontiguousarray(codes, np.uint16)
    coef_codes = np.ascontiguousarray(coef_codes, np.int32)
    flags = np.ascontiguousarray(flags, np.uint8)
    oidx = np.ascontiguousarray(outlier_idx, np.uint64)
    oval = np.ascontiguousarray(outlier_val, dtype)
    rc = _load().orc_lr_decompress(_dtype_id(dtype), _ptr(d), dim0_offset, B, radius, float(eb_abs), _ptr(codes),
                                   _ptr(coef_codes), _ptr(flags), _ptr(oidx), _ptr(oval), oidx.size, _ptr(out))
    if rc != OK:
        raise ValueError(f"orc_lr_decompress rc={rc}")
    return out


def lr_delta(q: np.ndarray, i: int, j: int, k: int) -> int:
    """L2 on one dense block of int64 values."""
    q = np.ascontiguousarray(q, np.int64)
    return int(_load().orc_lr_delta(_ptr(q), q.shape[0], q.shape[1], q.shape[2], i, j, k))


# SZ3-Interp (DEFINITION.md I1-I6; sz3_oracle.cpp interp_*)
@dataclass
class InterpCompressed:
    dims: tuple
    dtype: np.dtype
    radius: int
    eb_abs: float
    codes: np.ndarray          # uint16, field shape (the anchor's code is 0)
    outlier_idx: np.ndarray    # uint64 global indices (the anchor first)
    outlier_val: np.ndarray
    hist: np.ndarray
    counters: dict
    dim0_offset: int
    xprime: np.ndarray         # compress-time reconstruction


def interp_compress(x: np.ndarray, eb: float, eb_mode: str = "rel", radius: int = 32768, dim0_offset: int = 0,
                    value_range_override: tuple | None = None) -> InterpCompressed:
    """I1-I5 over a 3D field (1D/2D embedded with leading extents 1)."""
    x = np.ascontiguousarray(x)
    shape = (1,) * (3 - x.ndim) + tuple(x.shape)
    dims = np.array(shape, np.uint64)
    N = int(np.prod(shape))
    codes = np.empty(shape, np.uint16)
    oidx = np.empty(N, np.uint64)
    oval = np.empty(N, x.dtype)
    nout = np.zeros(1, np.uint64)
    hist = np.empty(2 * radius, np.int64)
    eb_abs = np.zeros(1, np.float64)
    xprime = np.empty(shape, x.dtype)
    cnt = Counters()
    rng = None if value_range_override is None else np.array(value_range_override, np.float64)
    rc = _load().orc_interp_compress(_dtype_id(x.dtype), _ptr(dims), dim0_offset, radius, {"abs": 0, "rel": 1}[eb_mode],
                                     float(eb), _ptr(rng), _ptr(x), _ptr(codes), _ptr(oidx), _ptr(oval), N, _ptr(nout),
                                     _ptr(hist), _ptr(eb_abs), _ptr(xprime), ctypes.byref(cnt))
    if rc != OK:
        raise ValueError(f"orc_interp_compress rc={rc}")
    n = int(nout[0])
    return InterpCompressed(tuple(int(s) for s in shape), x.dtype, radius, float(eb_abs[0]), codes, oidx[:n].copy(),
                            oval[:n].copy(), hist, cnt.as_dict(), dim0_offset, xprime)


def interp_decompress(c: InterpCompressed | None = None, *, dims=None, dtype=None, radius=None, eb_abs=None,
                      codes=None, outlier_idx=None, outlier_val=None, dim0_offset=0) -> np.ndarray:
    """I6."""
    if c is not None:
        dims, dtype, radius, eb_abs = c.dims, c.dtype, c.radius, c.eb_abs
        codes, outlier_idx, outlier_val, dim0_offset = c.codes, c.outlier_idx, c.outlier_val, c.dim0_offset
    d = np.array(dims, np.uint64)
    out = np.zeros(tuple(int(s) for s in dims), dtype)
    codes = np.ascontiguousarray(codes, np.uint16)
    oidx = np.ascontiguousarray(outlier_idx, np.uint64)
    oval = np.ascontiguousarray(outlier_val, dtype)
    rc = _load().orc_interp_decompress(_dtype_id(dtype), _ptr(d), dim0_offset, radius, float(eb_abs), _ptr(codes),
                                       _ptr(oidx), _ptr(oval), oidx.size, _ptr(out))
    if rc != OK:
        raise ValueError(f"orc_interp_decompress rc={rc}")
    return out


def interp_predict(a: float, b: float, c: float, e: float, method: int) -> float:
    """I3: method 2 cubic (donors -3s, -s, +s, +3s), 1 linear (-s, +s), 0 copy of -s."""
    return float(_load().orc_interp_predict(a, b, c, e, method))


def interp_pass_of(dims, i0: int, i1: int, i2: int) -> int:
    """I2: the pass (3 level + axis, level 0 = the largest stride) that predicts index (i0, i1, i2); -1 = anchor."""
    d = np.array(dims, np.uint64)
    return int(_load().orc_interp_pass_of(_ptr(d), i0, i1, i2))
