"""Python binding of libsz3g (include/sz3g.h): argument marshalling only.

Every step of the path runs in the library's sm_100a kernels; PyTorch only provides device memory,
streams and (in ``dist.py``) process groups.  There is no CPU fallback: if the library is missing or
no CUDA device is present, the calls raise.

Names follow the C ABI: ``value_range``, ``regression_compress``, ``regression_decompress``,
``histogram``, ``num_blocks``.  ``compress`` / ``decompress`` are the one-call conveniences on top.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

from . import build as _build

SZ3G_F32, SZ3G_F64 = 0, 1
SZ3G_EB_ABS, SZ3G_EB_REL_RANGE = 0, 1
FLAG_FORCE_GENERIC = 0x1
STATUS_OUTLIER_OVERFLOW, STATUS_BAD_RANGE = 0x1, 0x2
STATUS_BAD_HUFFMAN = 0x4
STATUS_PAYLOAD_OVERFLOW = 0x8
BLOCK = 6
_ERR = {0: "ok", -1: "EINVAL", -2: "EUNSUPPORTED", -3: "ERANGE", -4: "ECUDA", -5: "ECORRUPT"}


class SZ3GError(RuntimeError):
    pass


class Grid(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int), ("ndim", ctypes.c_int), ("dims", ctypes.c_uint64 * 3),
                ("dim0_offset", ctypes.c_uint64)]


class Params(ctypes.Structure):
    _fields_ = [("block_size", ctypes.c_uint32), ("radius", ctypes.c_uint32), ("eb_mode", ctypes.c_int),
                ("eb", ctypes.c_double), ("flags", ctypes.c_uint32)]


class StreamHeader(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int), ("ndim", ctypes.c_uint32), ("dims", ctypes.c_uint64 * 3),
                ("eb_mode", ctypes.c_int), ("eb", ctypes.c_double), ("eb_abs", ctypes.c_double),
                ("radius", ctypes.c_uint32), ("block_size", ctypes.c_uint32), ("chunk", ctypes.c_uint32),
                ("max_len", ctypes.c_uint32), ("flags", ctypes.c_uint32), ("n_outliers", ctypes.c_uint64),
                ("nblocks", ctypes.c_uint64), ("dim0_offset", ctypes.c_uint64)]


class Section(ctypes.Structure):
    _fields_ = [("tag", ctypes.c_uint32), ("data", ctypes.c_void_p), ("bytes", ctypes.c_uint64)]


SEC_CODE_BOOK, SEC_CODE_OFFS, SEC_CODE_DATA, SEC_COEF_BOOK, SEC_COEF_OFFS, SEC_COEF_DATA, SEC_COEF_ESC, \
    SEC_OUT_IDX, SEC_OUT_VAL, SEC_LR_FLAGS = range(1, 11)
STREAM_LR = 0x1   # sz3g_stream_header.flags: SZ3-LR stream
STREAM_INTERP = 0x2   # SZ3-Interp stream (no coefficient sections)


_lib = None


def lib_path() -> str:
    return _build.LIB


def load(allow_build: bool = False):
    """Load libsz3g.so (built in-tree by ``__graft_entry__.build()``); raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SZ3G_LIB", _build.LIB)   # SZ3G_LIB: an alternative build (A/B timing only)
    if not os.path.exists(path):
        if allow_build and path == _build.LIB:
            _build.build()
        else:
            raise SZ3GError(f"libsz3g.so not built ({path}); run `python -m paper_2111_02925_b200.build`")
    lib = ctypes.CDLL(path)
    P, U64, U32, I32, D = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_double
    GP, PP = ctypes.POINTER(Grid), ctypes.POINTER(Params)
    lib.sz3g_value_range.argtypes = [GP, P, P, P]
    lib.sz3g_regression_compress.argtypes = [GP, PP, P, P, P, P, P, P, P, U64, P, P, P, P, P]
    lib.sz3g_regression_decompress.argtypes = [GP, PP, P, P, P, P, P, U64, P, P, P]
    lib.sz3g_regression_analyze.argtypes = [GP, P, P, P, P]
    lib.sz3g_regression_quantize.argtypes = [GP, PP, P, P, P, P, P, P, P, U64, P, P, P, P, P]
    lib.sz3g_histogram.argtypes = [P, U64, U32, P, P]
    lib.sz3g_histogram_bins.argtypes = [P, U64, U32, U32, P, P]
    lib.sz3g_num_blocks.argtypes = [GP, U32]
    lib.sz3g_num_blocks.restype = U64
    lib.sz3g_uses_tma.argtypes = [GP, I32]
    lib.sz3g_launch_count.restype = U64
    if hasattr(lib, "sz3g_huffman_codebook"):   # absent only in older A/B builds
        lib.sz3g_huffman_scratch_bytes.argtypes = [U32, U32]
        lib.sz3g_huffman_scratch_bytes.restype = U64
        lib.sz3g_huffman_dtable_bytes.argtypes = [U32]
        lib.sz3g_huffman_dtable_bytes.restype = U64
        lib.sz3g_huffman_encode_scratch_bytes.argtypes = [U64, U32]
        lib.sz3g_huffman_encode_scratch_bytes.restype = U64
        lib.sz3g_huffman_codebook.argtypes = [P, U32, U32, P, P, P, P, P, P]
        lib.sz3g_huffman_encode.argtypes = [P, U64, U32, P, U32, P, P, U64, P, P, P]
        lib.sz3g_huffman_decode.argtypes = [P, P, U64, U32, P, U32, P, P, P]
    if hasattr(lib, "sz3g_truncation_compress"):   # absent only in older A/B builds
        lib.sz3g_truncation_compress.argtypes = [GP, P, U32, P, P]
        lib.sz3g_truncation_decompress.argtypes = [GP, P, U32, P, P]
    if hasattr(lib, "sz3g_error_stats"):   # absent only in older A/B builds
        lib.sz3g_error_stats_scratch_bytes.argtypes = [U64]
        lib.sz3g_error_stats_scratch_bytes.restype = U64
        lib.sz3g_error_stats.argtypes = [GP, P, P, D, P, P, P]
    if hasattr(lib, "sz3g_coef_delta_encode"):   # absent only in older A/B builds
        lib.sz3g_coef_delta_scratch_bytes.argtypes = [U64]
        lib.sz3g_coef_delta_scratch_bytes.restype = U64
        lib.sz3g_coef_delta_encode.argtypes = [P, U64, P, P, U64, P, P, P]
        lib.sz3g_coef_delta_decode.argtypes = [P, U64, P, U64, P, P, P, P]
    if hasattr(lib, "sz3g_stream_write"):   # absent only in older A/B builds
        lib.sz3g_huffman_codebook_from_lengths.argtypes = [P, U32, U32, P, P, P, P]
        lib.sz3g_stream_size.argtypes = [ctypes.POINTER(Section), U32]
        lib.sz3g_stream_size.restype = U64
        lib.sz3g_stream_write.argtypes = [ctypes.POINTER(StreamHeader), ctypes.POINTER(Section), U32, P, U64,
                                          ctypes.POINTER(U64)]
        lib.sz3g_stream_read.argtypes = [P, U64, ctypes.POINTER(StreamHeader), ctypes.POINTER(Section), U32,
                                         ctypes.POINTER(U32), ctypes.POINTER(U32)]
    if hasattr(lib, "sz3g_lr_quantize"):   # absent only in older A/B builds
        lib.sz3g_lr_quantize.argtypes = [GP, PP, P, P, P, P, P, P, P, P, U64, P, P, P, P, P]
        lib.sz3g_lr_decompress.argtypes = [GP, PP, P, P, P, P, P, P, U64, P, P, P]
    if hasattr(lib, "sz3g_interp_compress"):   # absent only in older A/B builds
        lib.sz3g_interp_compress.argtypes = [GP, PP, P, P, P, P, P, P, U64, P, P, P, P, P]
        lib.sz3g_interp_decompress.argtypes = [GP, PP, P, P, P, P, U64, P, P, P]
    if hasattr(lib, "sz3g_tie_counts"):   # absent only in older A/B builds
        lib.sz3g_tie_counts.argtypes = [GP, PP, P, P, P, P, P, P]
    if hasattr(lib, "sz3g_stream_validate"):
        lib.sz3g_stream_validate.argtypes = [ctypes.POINTER(StreamHeader), ctypes.POINTER(Section), U32,
                                             ctypes.POINTER(U32)]
    if hasattr(lib, "sz3g_set_tuning"):   # absent only in older A/B builds
        lib.sz3g_set_tuning.argtypes = [ctypes.c_char_p, ctypes.c_int64]
    for f in ("sz3g_strerror",):
        getattr(lib, f).argtypes = [I32]
        getattr(lib, f).restype = ctypes.c_char_p
    lib.sz3g_last_cuda_error.restype = ctypes.c_char_p
    lib.sz3g_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


EXPORTED_SYMBOLS = ("sz3g_value_range", "sz3g_regression_compress", "sz3g_regression_decompress", "sz3g_histogram",
                    "sz3g_histogram_bins",
                    "sz3g_regression_analyze", "sz3g_regression_quantize", "sz3g_huffman_scratch_bytes",
                    "sz3g_huffman_dtable_bytes", "sz3g_huffman_encode_scratch_bytes", "sz3g_huffman_codebook",
                    "sz3g_huffman_encode", "sz3g_huffman_decode", "sz3g_truncation_compress",
                    "sz3g_truncation_decompress", "sz3g_error_stats_scratch_bytes", "sz3g_error_stats",
                    "sz3g_coef_delta_scratch_bytes", "sz3g_coef_delta_encode", "sz3g_coef_delta_decode",
                    "sz3g_huffman_codebook_from_lengths", "sz3g_stream_size", "sz3g_stream_write",
                    "sz3g_stream_read", "sz3g_stream_validate", "sz3g_tie_counts", "sz3g_interp_compress",
                    "sz3g_interp_decompress", "sz3g_lr_quantize", "sz3g_lr_decompress",
                    "sz3g_num_blocks", "sz3g_uses_tma", "sz3g_launch_count", "sz3g_set_tuning", "sz3g_strerror",
                    "sz3g_last_cuda_error", "sz3g_version")


def _check(rc: int, what: str):
    if rc != 0:
        extra = ""
        if rc == -4:
            extra = ": " + load().sz3g_last_cuda_error().decode()
        raise SZ3GError(f"{what} failed: {_ERR.get(rc, rc)}{extra}")


def _dtype_id(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return SZ3G_F32
    if dt == torch.float64:
        return SZ3G_F64
    raise SZ3GError(f"unsupported dtype {dt}")


def _shape3(shape) -> tuple:
    shape = tuple(int(s) for s in shape)
    if not 1 <= len(shape) <= 3:
        raise SZ3GError("fields are 1D, 2D or 3D")
    return (1,) * (3 - len(shape)) + shape


def make_grid(shape, dtype: torch.dtype, dim0_offset: int = 0) -> Grid:
    s3 = _shape3(shape)
    return Grid(_dtype_id(dtype), len(tuple(shape)), (ctypes.c_uint64 * 3)(*s3), dim0_offset)


def make_params(eb: float, eb_mode: str = "rel", radius: int = 32768, flags: int = 0) -> Params:
    mode = {"abs": SZ3G_EB_ABS, "rel": SZ3G_EB_REL_RANGE}[eb_mode]
    return Params(BLOCK, radius, mode, float(eb), flags)


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _require_cuda(*ts):
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise SZ3GError("tensors passed to libsz3g must be contiguous CUDA tensors")


def num_blocks(shape) -> int:
    g = make_grid(shape, torch.float32)
    return int(load().sz3g_num_blocks(ctypes.byref(g), BLOCK))


def uses_tma(shape, dtype: torch.dtype, decompress: bool = False) -> bool:
    g = make_grid(shape, dtype)
    return bool(load().sz3g_uses_tma(ctypes.byref(g), int(decompress)))


def launch_count() -> int:
    return int(load().sz3g_launch_count())


def set_tuning(key: str, value: int) -> None:
    """Performance knob for later launches (sz3g_set_tuning); never changes a result."""
    _check(load().sz3g_set_tuning(key.encode(), int(value)), f"set_tuning({key})")


# ------------------------------------------------------------------------------------------- a0
def value_range(x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Device double[2] {min, max} of x (sz3g_value_range)."""
    _require_cuda(x)
    if out is None:
        out = torch.empty(2, dtype=torch.float64, device=x.device)
    g = make_grid(x.shape, x.dtype)
    _check(load().sz3g_value_range(ctypes.byref(g), _ptr(x), _ptr(out), _stream(stream)), "sz3g_value_range")
    return out


# ------------------------------------------------------------------------------------------- a1-a7
@dataclass
class Compressed:
    shape: tuple
    dtype: torch.dtype
    radius: int
    dim0_offset: int
    codes: torch.Tensor           # uint16, field shape
    coef_codes: torch.Tensor      # int32 [NB, 4]
    coef_raw: torch.Tensor | None  # float64 [NB, 4]
    outlier_idx: torch.Tensor     # int64 (uint64 bits) [cap]
    outlier_val: torch.Tensor     # T [cap]
    outlier_count: torch.Tensor   # int64 [1] (device)
    hist: torch.Tensor | None     # int64 [2R]
    eb_abs_dev: torch.Tensor      # float64 [1] (device)
    status: torch.Tensor          # int32 [1] (device)
    n_outliers: int | None = None
    eb_abs: float | None = None
    lr_flags: torch.Tensor | None = None   # SZ3-LR only: uint8 [NB], 1 = Lorenzo block

    def finalize(self) -> "Compressed":
        """Synchronise on the results, raise on device status bits, fill n_outliers / eb_abs."""
        st = int(self.status.item())
        cnt = int(self.outlier_count.item())
        if st & STATUS_BAD_RANGE:
            raise SZ3GError("bad value range: eb_abs is not finite or <= 0")
        if st & STATUS_OUTLIER_OVERFLOW:
            raise SZ3GError(f"outlier capacity {self.outlier_idx.numel()} exceeded ({cnt} outliers)")
        self.n_outliers = cnt
        self.eb_abs = float(self.eb_abs_dev.item())
        return self


class CompressBuffers:
    """Preallocated device outputs for repeated compression of one shape (no allocation per call)."""

    def __init__(self, shape, dtype: torch.dtype, radius: int = 32768, outlier_cap: int | None = None,
                 device=None, coef_raw: bool = False, hist: bool = True):
        device = device or torch.device("cuda", torch.cuda.current_device())
        N = 1
        for s in shape:
            N *= int(s)
        nb = num_blocks(shape)
        cap = outlier_cap if outlier_cap is not None else max(4096, N // 64)
        self.shape, self.dtype, self.radius = tuple(shape), dtype, radius
        self.codes = torch.empty(tuple(shape), dtype=torch.uint16, device=device)
        self.coef_codes = torch.empty((nb, 4), dtype=torch.int32, device=device)
        self.coef_raw = torch.empty((nb, 4), dtype=torch.float64, device=device) if coef_raw else None
        self.outlier_idx = torch.empty(cap, dtype=torch.int64, device=device)
        self.outlier_val = torch.empty(cap, dtype=dtype, device=device)
        self.outlier_count = torch.zeros(1, dtype=torch.int64, device=device)
        self.hist = torch.zeros(2 * radius, dtype=torch.int64, device=device) if hist else None
        self.eb_abs = torch.zeros(1, dtype=torch.float64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.minmax = torch.zeros(2, dtype=torch.float64, device=device)
        self.beta = None   # [NB, 4] float64, allocated by the two-pass path (regression_analyze)
        self.lr_flags = None   # [NB] uint8, allocated by the SZ3-LR path

    def beta_buffer(self) -> torch.Tensor:
        if self.beta is None:
            self.beta = torch.empty_like(self.coef_codes, dtype=torch.float64)
        return self.beta

    def flags_buffer(self) -> torch.Tensor:
        if self.lr_flags is None:
            self.lr_flags = torch.empty(self.coef_codes.shape[0], dtype=torch.uint8, device=self.coef_codes.device)
        return self.lr_flags

    def reset(self):
        """Zero the accumulating outputs (outlier counter, histogram, status)."""
        self.outlier_count.zero_()
        self.status.zero_()
        if self.hist is not None:
            self.hist.zero_()


def regression_compress(x: torch.Tensor, eb: float, eb_mode: str = "rel", radius: int = 32768,
                        d_minmax: torch.Tensor | None = None, bufs: CompressBuffers | None = None,
                        outlier_cap: int | None = None, coef_raw: bool = False, hist: bool = True,
                        dim0_offset: int = 0, flags: int = 0, stream=None, reset: bool = True) -> Compressed:
    """sz3g_regression_compress.  Asynchronous: call ``.finalize()`` on the result to sync and check.

    In REL mode ``d_minmax`` (device double[2]) is the global value range; when omitted it is computed
    here with ``value_range`` (unsharded use).  ``bufs`` reuses preallocated outputs; with
    ``reset=False`` the histogram / outlier counter / status are NOT zeroed first (caller did it).
    """
    _require_cuda(x)
    if bufs is None:
        bufs = CompressBuffers(x.shape, x.dtype, radius, outlier_cap, x.device, coef_raw, hist)
    elif reset:
        bufs.reset()
    if bufs is not None and bufs.radius != radius:
        raise SZ3GError("buffer radius mismatch")
    if bufs is not None and reset is True and bufs.hist is not None and hist is False:
        pass
    if eb_mode == "rel" and d_minmax is None:
        d_minmax = value_range(x, bufs.minmax, stream)
    g = make_grid(x.shape, x.dtype, dim0_offset)
    p = make_params(eb, eb_mode, radius, flags)
    rc = load().sz3g_regression_compress(
        ctypes.byref(g), ctypes.byref(p), _ptr(x), _ptr(d_minmax), _ptr(bufs.codes), _ptr(bufs.coef_codes),
        _ptr(bufs.coef_raw), _ptr(bufs.outlier_idx), _ptr(bufs.outlier_val), bufs.outlier_idx.numel(),
        _ptr(bufs.outlier_count), _ptr(bufs.hist if hist else None), _ptr(bufs.eb_abs), _ptr(bufs.status),
        _stream(stream))
    _check(rc, "sz3g_regression_compress")
    return Compressed(tuple(x.shape), x.dtype, radius, dim0_offset, bufs.codes, bufs.coef_codes, bufs.coef_raw,
                      bufs.outlier_idx, bufs.outlier_val, bufs.outlier_count, bufs.hist if hist else None,
                      bufs.eb_abs, bufs.status)


def regression_analyze(x: torch.Tensor, minmax: torch.Tensor | None = None, beta: torch.Tensor | None = None,
                       stream=None) -> tuple[torch.Tensor, torch.Tensor]:
    """sz3g_regression_analyze: one read of x -> (device double[2] {min, max}, float64 [NB, 4] beta)."""
    _require_cuda(x, minmax, beta)
    if minmax is None:
        minmax = torch.empty(2, dtype=torch.float64, device=x.device)
    if beta is None:
        beta = torch.empty((num_blocks(x.shape), 4), dtype=torch.float64, device=x.device)
    g = make_grid(x.shape, x.dtype)
    _check(load().sz3g_regression_analyze(ctypes.byref(g), _ptr(x), _ptr(minmax), _ptr(beta), _stream(stream)),
           "sz3g_regression_analyze")
    return minmax, beta


def regression_quantize(x: torch.Tensor, eb: float, eb_mode: str, radius: int, d_minmax: torch.Tensor | None,
                        beta: torch.Tensor, bufs: CompressBuffers | None = None, outlier_cap: int | None = None,
                        hist: bool = True, dim0_offset: int = 0, flags: int = 0, stream=None,
                        reset: bool = True) -> Compressed:
    """sz3g_regression_quantize: compression from the analyze pass's beta (asynchronous, like
    regression_compress; outputs bit-identical to it).  ``Compressed.coef_raw`` is ``beta``."""
    _require_cuda(x, d_minmax, beta)
    if bufs is None:
        bufs = CompressBuffers(x.shape, x.dtype, radius, outlier_cap, x.device, False, hist)
    elif reset:
        bufs.reset()
    if bufs.radius != radius:
        raise SZ3GError("buffer radius mismatch")
    g = make_grid(x.shape, x.dtype, dim0_offset)
    p = make_params(eb, eb_mode, radius, flags)
    rc = load().sz3g_regression_quantize(
        ctypes.byref(g), ctypes.byref(p), _ptr(x), _ptr(d_minmax), _ptr(beta), _ptr(bufs.codes),
        _ptr(bufs.coef_codes), _ptr(bufs.outlier_idx), _ptr(bufs.outlier_val), bufs.outlier_idx.numel(),
        _ptr(bufs.outlier_count), _ptr(bufs.hist if hist else None), _ptr(bufs.eb_abs), _ptr(bufs.status),
        _stream(stream))
    _check(rc, "sz3g_regression_quantize")
    return Compressed(tuple(x.shape), x.dtype, radius, dim0_offset, bufs.codes, bufs.coef_codes, beta,
                      bufs.outlier_idx, bufs.outlier_val, bufs.outlier_count, bufs.hist if hist else None,
                      bufs.eb_abs, bufs.status)


def compress_two_pass(x: torch.Tensor, eb: float, eb_mode: str = "rel", radius: int = 32768,
                      bufs: CompressBuffers | None = None, outlier_cap: int | None = None, hist: bool = True,
                      flags: int = 0, stream=None) -> Compressed:
    """analyze (range + beta, one read) -> quantize (one read): the REL-mode path (asynchronous)."""
    if bufs is None:
        bufs = CompressBuffers(x.shape, x.dtype, radius, outlier_cap, x.device, False, hist)
    minmax, beta = regression_analyze(x, bufs.minmax, bufs.beta_buffer(), stream)
    return regression_quantize(x, eb, eb_mode, radius, minmax, beta, bufs, hist=hist, flags=flags, stream=stream)


def regression_decompress(codes: torch.Tensor, coef_codes: torch.Tensor, outlier_idx: torch.Tensor,
                          outlier_val: torch.Tensor, n_outliers: int, eb: float, radius: int = 32768,
                          dtype: torch.dtype = torch.float32, dim0_offset: int = 0, out: torch.Tensor | None = None,
                          flags: int = 0, stream=None, d_outlier_count: torch.Tensor | None = None,
                          eb_mode: str = "abs", d_minmax: torch.Tensor | None = None) -> torch.Tensor:
    """sz3g_regression_decompress (recover) + outlier scatter.

    ``eb_mode="abs"``: ``eb`` is the eb_abs used at compression.  ``eb_mode="rel"``: ``eb`` is the
    relative bound and ``d_minmax`` the same device range compression used.  With ``d_outlier_count``
    (the device counter written by compress) ``n_outliers`` is only the capacity.  Neither form needs
    a host synchronisation.
    """
    _require_cuda(codes, coef_codes, outlier_idx, outlier_val, out, d_outlier_count, d_minmax)
    if out is None:
        out = torch.empty(codes.shape, dtype=dtype, device=codes.device)
    g = make_grid(codes.shape, out.dtype, dim0_offset)
    p = make_params(eb, eb_mode, radius, flags)
    rc = load().sz3g_regression_decompress(ctypes.byref(g), ctypes.byref(p), _ptr(d_minmax), _ptr(codes),
                                           _ptr(coef_codes), _ptr(outlier_idx), _ptr(outlier_val),
                                           int(n_outliers), _ptr(d_outlier_count), _ptr(out), _stream(stream))
    _check(rc, "sz3g_regression_decompress")
    return out


def lr_quantize(x: torch.Tensor, eb: float, eb_mode: str, radius: int, d_minmax: torch.Tensor | None,
                beta: torch.Tensor, bufs: CompressBuffers | None = None, outlier_cap: int | None = None,
                hist: bool = True, dim0_offset: int = 0, flags: int = 0, stream=None, reset: bool = True) -> Compressed:
    """sz3g_lr_quantize (SZ3-LR; DEFINITION.md L1-L6): per block the better of the regression and
    the prequantised Lorenzo predictor, from the analyze pass's beta (asynchronous).  The result's
    ``lr_flags`` marks the Lorenzo blocks; Lorenzo blocks' coefficient codes are 0."""
    _require_cuda(x, d_minmax, beta)
    if bufs is None:
        bufs = CompressBuffers(x.shape, x.dtype, radius, outlier_cap, x.device, False, hist)
    elif reset:
        bufs.reset()
    if bufs.radius != radius:
        raise SZ3GError("buffer radius mismatch")
    fl = bufs.flags_buffer()
    g = make_grid(x.shape, x.dtype, dim0_offset)
    p = make_params(eb, eb_mode, radius, flags)
    rc = load().sz3g_lr_quantize(
        ctypes.byref(g), ctypes.byref(p), _ptr(x), _ptr(d_minmax), _ptr(beta), _ptr(bufs.codes),
        _ptr(bufs.coef_codes), _ptr(fl), _ptr(bufs.outlier_idx), _ptr(bufs.outlier_val), bufs.outlier_idx.numel(),
        _ptr(bufs.outlier_count), _ptr(bufs.hist if hist else None), _ptr(bufs.eb_abs), _ptr(bufs.status),
        _stream(stream))
    _check(rc, "sz3g_lr_quantize")
    return Compressed(tuple(x.shape), x.dtype, radius, dim0_offset, bufs.codes, bufs.coef_codes, beta,
                      bufs.outlier_idx, bufs.outlier_val, bufs.outlier_count, bufs.hist if hist else None,
                      bufs.eb_abs, bufs.status, lr_flags=fl)


def lr_compress(x: torch.Tensor, eb: float, eb_mode: str = "rel", radius: int = 32768,
                bufs: CompressBuffers | None = None, outlier_cap: int | None = None, hist: bool = True,
                flags: int = 0, stream=None, finalize: bool = True) -> Compressed:
    """SZ3-LR compression: analyze (range + beta, one read) -> lr_quantize (one read)."""
    if bufs is None:
        bufs = CompressBuffers(x.shape, x.dtype, radius, outlier_cap, x.device, False, hist)
    minmax, beta = regression_analyze(x, bufs.minmax, bufs.beta_buffer(), stream)
    res = lr_quantize(x, eb, eb_mode, radius, minmax, beta, bufs, hist=hist, flags=flags, stream=stream)
    return res.finalize() if finalize else res


def lr_decompress(codes: torch.Tensor, coef_codes: torch.Tensor, lr_flags: torch.Tensor, outlier_idx: torch.Tensor,
                  outlier_val: torch.Tensor, n_outliers: int, eb: float, radius: int = 32768,
                  dtype: torch.dtype = torch.float32, dim0_offset: int = 0, out: torch.Tensor | None = None,
                  flags: int = 0, stream=None, d_outlier_count: torch.Tensor | None = None, eb_mode: str = "abs",
                  d_minmax: torch.Tensor | None = None) -> torch.Tensor:
    """sz3g_lr_decompress (L7): outlier scatter, then regression / Lorenzo blocks (asynchronous)."""
    _require_cuda(codes, coef_codes, lr_flags, outlier_idx, outlier_val, out, d_outlier_count, d_minmax)
    if out is None:
        out = torch.empty(codes.shape, dtype=dtype, device=codes.device)
    g = make_grid(codes.shape, out.dtype, dim0_offset)
    p = make_params(eb, eb_mode, radius, flags)
    rc = load().sz3g_lr_decompress(ctypes.byref(g), ctypes.byref(p), _ptr(d_minmax), _ptr(codes), _ptr(coef_codes),
                                   _ptr(lr_flags), _ptr(outlier_idx), _ptr(outlier_val), int(n_outliers),
                                   _ptr(d_outlier_count), _ptr(out), _stream(stream))
    _check(rc, "sz3g_lr_decompress")
    return out


def histogram(codes: torch.Tensor, radius: int = 32768, hist: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """sz3g_histogram: accumulate the 2R-bin int64 histogram of uint16 codes."""
    _require_cuda(codes, hist)
    if hist is None:
        hist = torch.zeros(2 * radius, dtype=torch.int64, device=codes.device)
    rc = load().sz3g_histogram(_ptr(codes), codes.numel(), radius, _ptr(hist), _stream(stream))
    _check(rc, "sz3g_histogram")
    return hist


def histogram_bins(codes: torch.Tensor, nbins: int, window_lo: int = 0, hist: torch.Tensor | None = None,
                   stream=None) -> torch.Tensor:
    """sz3g_histogram_bins: accumulate an nbins int64 histogram with the smem window at window_lo."""
    _require_cuda(codes, hist)
    if hist is None:
        hist = torch.zeros(nbins, dtype=torch.int64, device=codes.device)
    _check(load().sz3g_histogram_bins(_ptr(codes), codes.numel(), nbins, window_lo, _ptr(hist), _stream(stream)),
           "sz3g_histogram_bins")
    return hist


# ------------------------------------------------------------------------------------------- SZ3-Interp
@dataclass
class InterpCompressed:
    """sz3g_interp_compress outputs (device).  ``xprime`` is the compress-time reconstruction."""
    shape: tuple
    dtype: torch.dtype
    radius: int
    dim0_offset: int
    codes: torch.Tensor
    xprime: torch.Tensor
    outlier_idx: torch.Tensor
    outlier_val: torch.Tensor
    outlier_count: torch.Tensor
    hist: torch.Tensor | None
    eb_abs_dev: torch.Tensor
    status: torch.Tensor
    n_outliers: int | None = None
    eb_abs: float | None = None

    def finalize(self) -> "InterpCompressed":
        st = int(self.status.item())
        cnt = int(self.outlier_count.item())
        if st & STATUS_BAD_RANGE:
            raise SZ3GError("bad value range: eb_abs is not finite or <= 0")
        if st & STATUS_OUTLIER_OVERFLOW:
            raise SZ3GError(f"outlier capacity {self.outlier_idx.numel()} exceeded ({cnt} outliers)")
        self.n_outliers = cnt
        self.eb_abs = float(self.eb_abs_dev.item())
        return self


def interp_compress(x: torch.Tensor, eb: float, eb_mode: str = "rel", radius: int = 32768,
                    d_minmax: torch.Tensor | None = None, outlier_cap: int | None = None, hist: bool = True,
                    out: "InterpCompressed | None" = None, stream=None) -> InterpCompressed:
    """sz3g_interp_compress (SZ3-Interp; DEFINITION.md I1-I5), asynchronous.  REL mode without a
    given device range computes it with value_range.  ``out`` reuses a previous result's buffers."""
    _require_cuda(x, d_minmax)
    dev = x.device
    if out is None:
        N = x.numel()
        cap = outlier_cap if outlier_cap is not None else max(4096, N // 64)
        out = InterpCompressed(tuple(x.shape), x.dtype, radius, 0, torch.empty(tuple(x.shape), dtype=torch.uint16, device=dev),
                               torch.empty_like(x), torch.empty(cap, dtype=torch.int64, device=dev),
                               torch.empty(cap, dtype=x.dtype, device=dev), torch.zeros(1, dtype=torch.int64, device=dev),
                               torch.zeros(2 * radius, dtype=torch.int64, device=dev) if hist else None,
                               torch.zeros(1, dtype=torch.float64, device=dev), torch.zeros(1, dtype=torch.int32, device=dev))
    else:
        if out.shape != tuple(x.shape) or out.dtype != x.dtype or out.radius != radius or out.codes.device != dev:
            raise SZ3GError("interp_compress: `out` was made for another shape, dtype, radius or device")
        if (out.hist is None) == hist:
            raise SZ3GError("interp_compress: `out` was made with hist=" + str(out.hist is not None))
        out.outlier_count.zero_()
        out.status.zero_()
        if out.hist is not None:
            out.hist.zero_()
        out.n_outliers = out.eb_abs = None
    if eb_mode == "rel" and d_minmax is None:
        d_minmax = value_range(x, stream=stream)
    g = make_grid(x.shape, x.dtype)
    p = make_params(eb, eb_mode, radius)
    rc = load().sz3g_interp_compress(ctypes.byref(g), ctypes.byref(p), _ptr(x), _ptr(d_minmax), _ptr(out.codes),
                                     _ptr(out.xprime), _ptr(out.outlier_idx), _ptr(out.outlier_val),
                                     out.outlier_idx.numel(), _ptr(out.outlier_count), _ptr(out.hist), _ptr(out.eb_abs_dev),
                                     _ptr(out.status), _stream(stream))
    _check(rc, "sz3g_interp_compress")
    out._minmax = d_minmax
    return out


def interp_decompress(codes: torch.Tensor, outlier_idx: torch.Tensor, outlier_val: torch.Tensor, n_outliers: int,
                      eb: float, radius: int = 32768, dtype: torch.dtype = torch.float32, out: torch.Tensor | None = None,
                      d_outlier_count: torch.Tensor | None = None, eb_mode: str = "abs",
                      d_minmax: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """sz3g_interp_decompress (I6), asynchronous; arguments as regression_decompress."""
    _require_cuda(codes, outlier_idx, outlier_val, out, d_outlier_count, d_minmax)
    if out is None:
        out = torch.empty(codes.shape, dtype=dtype, device=codes.device)
    g = make_grid(codes.shape, out.dtype)
    p = make_params(eb, eb_mode, radius)
    rc = load().sz3g_interp_decompress(ctypes.byref(g), ctypes.byref(p), _ptr(d_minmax), _ptr(codes), _ptr(outlier_idx),
                                       _ptr(outlier_val), int(n_outliers), _ptr(d_outlier_count), _ptr(out),
                                       _stream(stream))
    _check(rc, "sz3g_interp_decompress")
    return out


TIE_COUNTER_NAMES = ("elem_near_ties", "elem_div_mismatch", "coef_near_ties", "coef_tie_blocks")


def tie_counts(x: torch.Tensor, eb: float, eb_mode: str, radius: int, d_minmax: torch.Tensor | None,
               coef_codes: torch.Tensor, beta: torch.Tensor | None = None, counts: torch.Tensor | None = None,
               stream=None) -> torch.Tensor:
    """sz3g_tie_counts: the parity rule's reported counters (i) element near-ties, (ii) division /
    reciprocal rounding mismatches, (iii) coefficient near-ties and their blocks, ACCUMULATED into a
    device int64 [4] (asynchronous).  ``beta`` None skips (iii)."""
    _require_cuda(x, d_minmax, coef_codes, beta, counts)
    if counts is None:
        counts = torch.zeros(4, dtype=torch.int64, device=x.device)
    g = make_grid(x.shape, x.dtype)
    p = make_params(eb, eb_mode, radius)
    _check(load().sz3g_tie_counts(ctypes.byref(g), ctypes.byref(p), _ptr(d_minmax), _ptr(x), _ptr(coef_codes),
                                  _ptr(beta), _ptr(counts), _stream(stream)), "sz3g_tie_counts")
    return counts


# ------------------------------------------------------------------------------------------- one-call API
def compress(x: torch.Tensor, eb: float, eb_mode: str = "rel", radius: int = 32768, two_pass: bool | None = None,
             **kw) -> Compressed:
    """Compress a CUDA field and check the device status (synchronises).  REL mode without a given
    range takes the two-pass path (analyze -> quantize, each one read of x); ABS mode or a given
    ``d_minmax`` the fused single-pass kernel.  Both give bit-identical outputs."""
    if two_pass is None:
        two_pass = eb_mode == "rel" and kw.get("d_minmax") is None and not kw.get("dim0_offset")
    if two_pass:
        kw.pop("coef_raw", None)
        kw.pop("d_minmax", None)
        res = compress_two_pass(x, eb, eb_mode, radius, **kw)
    else:
        res = regression_compress(x, eb, eb_mode, radius, **kw)
    res.finalize()
    return res


def decompress(res: Compressed, out: torch.Tensor | None = None, flags: int = 0) -> torch.Tensor:
    if res.n_outliers is None:
        res.finalize()
    if res.lr_flags is not None:
        return lr_decompress(res.codes, res.coef_codes, res.lr_flags, res.outlier_idx, res.outlier_val,
                             res.n_outliers, res.eb_abs, res.radius, res.dtype, res.dim0_offset, out, flags)
    return regression_decompress(res.codes, res.coef_codes, res.outlier_idx, res.outlier_val, res.n_outliers,
                                 res.eb_abs, res.radius, res.dtype, res.dim0_offset, out, flags)


# ------------------------------------------------------------------------------------------- Huffman
HUFF_MAX_LEN = 16     # DEFINITION.md H2 / G20
HUFF_CHUNK = 2048     # H4 / G21


@dataclass
class HuffmanTable:
    lengths: torch.Tensor     # uint8 [nsym]
    codewords: torch.Tensor   # int32 (uint32 bits) [nsym]: (length << 24) | canonical codeword
    dtable: torch.Tensor      # uint8 [sz3g_huffman_dtable_bytes]
    max_len: int
    status: torch.Tensor      # int32 [1]

    def stored_bytes(self) -> int:
        """A canonical code is rebuilt from its lengths alone (H3): 4 + 3 bytes per active symbol
        (u32 count, then u16 symbol + u8 length pairs)."""
        return 4 + 3 * int((self.lengths > 0).sum().item())

    def check(self) -> "HuffmanTable":
        if int(self.status.item()) & STATUS_BAD_HUFFMAN:
            raise SZ3GError("Huffman codebook: empty histogram, bad count, or too many symbols for max_len")
        return self


def huffman_codebook(hist: torch.Tensor, max_len: int = HUFF_MAX_LEN, stream=None) -> HuffmanTable:
    """sz3g_huffman_codebook (one CTA on the GPU) from a device int64 histogram (asynchronous)."""
    _require_cuda(hist)
    lib = load()
    nsym = hist.numel()
    dev = hist.device
    lens = torch.empty(nsym, dtype=torch.uint8, device=dev)
    cws = torch.empty(nsym, dtype=torch.int32, device=dev)
    dtab = torch.empty(int(lib.sz3g_huffman_dtable_bytes(nsym)), dtype=torch.uint8, device=dev)
    scratch = torch.empty(int(lib.sz3g_huffman_scratch_bytes(nsym, max_len)), dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    _check(lib.sz3g_huffman_codebook(_ptr(hist), nsym, max_len, _ptr(lens), _ptr(cws), _ptr(dtab), _ptr(scratch),
                                     _ptr(status), _stream(stream)), "sz3g_huffman_codebook")
    t = HuffmanTable(lens, cws, dtab, max_len, status)
    t._scratch = scratch   # keep alive until the stream has run
    return t


@dataclass
class HuffmanStream:
    n: int
    chunk: int
    offsets: torch.Tensor     # int64 [nchunks + 1] word offsets
    payload: torch.Tensor     # int32 (uint32 bits) [capacity]
    status: torch.Tensor

    def words(self) -> int:
        return int(self.offsets[-1].item())

    def check(self) -> "HuffmanStream":
        st = int(self.status.item())
        if st & STATUS_PAYLOAD_OVERFLOW:
            raise SZ3GError("Huffman payload capacity exceeded")
        if st & STATUS_BAD_HUFFMAN:
            raise SZ3GError("a code has no codeword in the Huffman table")
        return self


def huffman_encode(codes: torch.Tensor, table: HuffmanTable, chunk: int = HUFF_CHUNK,
                   payload: torch.Tensor | None = None, offsets: torch.Tensor | None = None,
                   scratch: torch.Tensor | None = None, stream=None) -> HuffmanStream:
    """sz3g_huffman_encode of a uint16 code array (asynchronous).  Without ``payload`` the capacity is
    the worst case (max_len bits per code + one word per chunk)."""
    _require_cuda(codes, payload, offsets, scratch)
    lib = load()
    n = codes.numel()
    nch = -(-n // chunk)
    dev = codes.device
    if offsets is None:
        offsets = torch.empty(nch + 1, dtype=torch.int64, device=dev)
    if payload is None:
        payload = torch.empty(max(1, -(-n * table.max_len // 32) + nch), dtype=torch.int32, device=dev)
    if scratch is None:
        scratch = torch.empty(int(lib.sz3g_huffman_encode_scratch_bytes(n, chunk)), dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    _check(lib.sz3g_huffman_encode(_ptr(codes), n, chunk, _ptr(table.codewords), table.codewords.numel(),
                                   _ptr(offsets), _ptr(payload), payload.numel(), _ptr(scratch), _ptr(status),
                                   _stream(stream)),
           "sz3g_huffman_encode")
    hs = HuffmanStream(n, chunk, offsets, payload, status)
    hs._scratch = scratch
    return hs


def huffman_decode(hs: HuffmanStream, table: HuffmanTable, out: torch.Tensor | None = None,
                   status: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """sz3g_huffman_decode -> uint16 codes (asynchronous; a corrupt stream sets STATUS_BAD_HUFFMAN)."""
    _require_cuda(out, status)
    lib = load()
    dev = hs.payload.device
    if out is None:
        out = torch.empty(hs.n, dtype=torch.uint16, device=dev)
    if status is None:
        status = hs.status
    _check(lib.sz3g_huffman_decode(_ptr(hs.payload), _ptr(hs.offsets), hs.n, hs.chunk, _ptr(table.dtable),
                                   table.max_len, _ptr(out), _ptr(status), _stream(stream)), "sz3g_huffman_decode")
    return out


# ------------------------------------------------------------------------------------------- Truncation
def truncation_compress(x: torch.Tensor, k: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """sz3g_truncation_compress: the k most-significant bytes of every element (uint8 [n * k])."""
    _require_cuda(x, out)
    if out is None:
        out = torch.empty(x.numel() * k, dtype=torch.uint8, device=x.device)
    g = make_grid((x.numel(),), x.dtype)
    _check(load().sz3g_truncation_compress(ctypes.byref(g), _ptr(x), k, _ptr(out), _stream(stream)),
           "sz3g_truncation_compress")
    return out


def truncation_decompress(b: torch.Tensor, n: int, k: int, dtype: torch.dtype = torch.float32,
                          out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """sz3g_truncation_decompress: zero-fill the discarded bytes."""
    _require_cuda(b, out)
    if out is None:
        out = torch.empty(n, dtype=dtype, device=b.device)
    g = make_grid((n,), dtype)
    _check(load().sz3g_truncation_decompress(ctypes.byref(g), _ptr(b), k, _ptr(out), _stream(stream)),
           "sz3g_truncation_decompress")
    return out


# ------------------------------------------------------------------------------------------- metrics
def error_stats(x: torch.Tensor, y: torch.Tensor, eb: float = float("inf"), stream=None) -> torch.Tensor:
    """sz3g_error_stats: device double[3] {max |x - y|, sum (x - y)^2, #(|x - y| > eb)} (asynchronous)."""
    _require_cuda(x, y)
    if x.shape != y.shape or x.dtype != y.dtype:
        raise SZ3GError("error_stats: x and y must have the same shape and dtype")
    lib = load()
    out = torch.empty(3, dtype=torch.float64, device=x.device)
    scratch = torch.empty(int(lib.sz3g_error_stats_scratch_bytes(x.numel())), dtype=torch.uint8, device=x.device)
    g = make_grid((x.numel(),), x.dtype)
    _check(lib.sz3g_error_stats(ctypes.byref(g), _ptr(x), _ptr(y), float(eb), _ptr(out), _ptr(scratch),
                                _stream(stream)), "sz3g_error_stats")
    out._scratch = scratch
    return out


def psnr(value_range: float, mse: float) -> float:
    """20 log10(range) - 10 log10(MSE); +inf when MSE = 0 ("infinity PSNR")."""
    import math
    return math.inf if mse == 0 else 20 * math.log10(value_range) - 10 * math.log10(mse)


def bit_rate(bits_per_sample: int, ratio: float) -> float:
    """bits / cr."""
    return bits_per_sample / ratio


# ------------------------------------------------------------------------------------------- coefficient codes
COEF_ESC = 65535


@dataclass
class CoefStream:
    nb: int
    table: HuffmanTable       # codebook of the delta symbols
    stream: HuffmanStream     # Huffman-coded symbols (4 * nb)
    escapes: torch.Tensor     # int64 (uint64 bits) [n_escapes]

    def nbytes(self) -> int:
        return 4 * self.stream.words() + 8 * self.stream.offsets.numel() + 8 * self.escapes.numel() + \
            self.table.stored_bytes()


def coef_delta_encode(coef_codes: torch.Tensor, stream=None, sync: bool = True, esc_cap: int | None = None):
    """sz3g_coef_delta_encode -> (sym uint16 [4 nb], escapes int64 [n]).  With ``sync=False`` no host
    synchronisation: returns (sym, escape buffer, device count) and the caller checks the count
    against the buffer (esc_cap entries, default nb)."""
    _require_cuda(coef_codes)
    lib = load()
    nb = coef_codes.numel() // 4
    dev = coef_codes.device
    sym = torch.empty(4 * nb, dtype=torch.uint16, device=dev)
    esc = torch.empty(max(1, esc_cap if esc_cap is not None else (4 * nb // 64 if sync else nb)), dtype=torch.int64,
                      device=dev)
    nesc = torch.zeros(1, dtype=torch.int64, device=dev)
    scratch = torch.empty(int(lib.sz3g_coef_delta_scratch_bytes(nb)), dtype=torch.uint8, device=dev)
    _check(lib.sz3g_coef_delta_encode(_ptr(coef_codes), nb, _ptr(sym), _ptr(esc), esc.numel(), _ptr(nesc),
                                      _ptr(scratch), _stream(stream)), "sz3g_coef_delta_encode")
    if not sync:
        sym._scratch = scratch
        return sym, esc, nesc
    n = int(nesc.item())
    if n > esc.numel():   # rare: more escapes than the first guess -> once more with room for all
        esc = torch.empty(n, dtype=torch.int64, device=dev)
        _check(lib.sz3g_coef_delta_encode(_ptr(coef_codes), nb, _ptr(sym), _ptr(esc), esc.numel(), _ptr(nesc),
                                          _ptr(scratch), _stream(stream)), "sz3g_coef_delta_encode")
    return sym, esc[:n]


def coef_delta_decode(sym: torch.Tensor, nb: int, escapes: torch.Tensor, out: torch.Tensor | None = None,
                      status: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """sz3g_coef_delta_decode -> int32 [nb, 4]."""
    _require_cuda(sym, escapes, out, status)
    lib = load()
    dev = sym.device
    if out is None:
        out = torch.empty((nb, 4), dtype=torch.int32, device=dev)
    if status is None:
        status = torch.zeros(1, dtype=torch.int32, device=dev)
    scratch = torch.empty(int(lib.sz3g_coef_delta_scratch_bytes(nb)), dtype=torch.uint8, device=dev)
    _check(lib.sz3g_coef_delta_decode(_ptr(sym), nb, _ptr(escapes if escapes.numel() else None), escapes.numel(),
                                      _ptr(out), _ptr(scratch), _ptr(status), _stream(stream)),
           "sz3g_coef_delta_decode")
    out._scratch = scratch
    return out


def encode_coefficients(coef_codes: torch.Tensor, stream=None, sync: bool = True) -> CoefStream:
    """Coefficient codes -> delta symbols -> their histogram -> Huffman codebook -> encoded stream.
    ``sync=False``: no host synchronisation; ``escapes`` is then the whole escape buffer and
    ``n_escapes`` a device count (the caller trims after its own synchronisation)."""
    nb = coef_codes.numel() // 4
    if sync:
        sym, esc = coef_delta_encode(coef_codes, stream)
        nesc = None
    else:
        sym, esc, nesc = coef_delta_encode(coef_codes, stream, sync=False)
    hist = histogram_bins(sym, 65536, 0, stream=stream)   # zigzag deltas: mass near 0
    table = huffman_codebook(hist, stream=stream)
    cs = CoefStream(nb, table, huffman_encode(sym, table, stream=stream), esc)
    cs.n_escapes = nesc
    return cs


def decode_coefficients(cs: CoefStream, stream=None) -> torch.Tensor:
    sym = huffman_decode(cs.stream, cs.table, stream=stream)
    return coef_delta_decode(sym, cs.nb, cs.escapes, stream=stream)


# ------------------------------------------------------------------------------------------- stream container
def _book_bytes(lengths: torch.Tensor):
    """Canonical codebook as stored: u32 n, then n x (u16 symbol, u8 length) (host bytes)."""
    import numpy as np
    L = lengths.cpu().numpy()
    sym = np.flatnonzero(L).astype(np.uint16)
    rec = np.zeros(sym.size, dtype=[("s", "<u2"), ("l", "u1")])
    rec["s"], rec["l"] = sym, L[sym]
    return np.uint32(sym.size).tobytes() + rec.tobytes()


def _book_lengths(b: bytes, nsym: int, device) -> torch.Tensor:
    import numpy as np
    n = int(np.frombuffer(b[:4], np.uint32)[0])
    rec = np.frombuffer(b[4:4 + 3 * n], dtype=[("s", "<u2"), ("l", "u1")])
    L = np.zeros(nsym, np.uint8)
    L[rec["s"]] = rec["l"]
    return torch.from_numpy(L).to(device)


def to_bytes(res: "Compressed", table: HuffmanTable | None = None, hs: HuffmanStream | None = None,
             coef: CoefStream | None = None, eb: float | None = None, eb_mode: str = "abs") -> bytes:
    """Serialise a finalized compression result: Huffman-coded codes, delta+Huffman-coded coefficient
    codes and the outliers, in the self-describing container (sz3g_stream_write).  Missing stages are
    run here (codebook from res.hist, encode, coefficient coding)."""
    if res.n_outliers is None:
        res.finalize()
    if table is None:
        table = huffman_codebook(res.hist).check()
    if hs is None:
        hs = huffman_encode(res.codes.view(-1), table).check()
    interp = isinstance(res, InterpCompressed)
    if coef is None and not interp:
        coef = encode_coefficients(res.coef_codes)
    n = res.n_outliers
    host = [
        (SEC_CODE_BOOK, _book_bytes(table.lengths)),
        (SEC_CODE_OFFS, hs.offsets.cpu().numpy().tobytes()),
        (SEC_CODE_DATA, hs.payload[:hs.words()].cpu().numpy().tobytes()),
    ]
    if not interp:
        host += [
            (SEC_COEF_BOOK, _book_bytes(coef.table.lengths)),
            (SEC_COEF_OFFS, coef.stream.offsets.cpu().numpy().tobytes()),
            (SEC_COEF_DATA, coef.stream.payload[:coef.stream.words()].cpu().numpy().tobytes()),
            (SEC_COEF_ESC, coef.escapes.cpu().numpy().tobytes()),
        ]
    host += [
        (SEC_OUT_IDX, res.outlier_idx[:n].cpu().numpy().tobytes()),
        (SEC_OUT_VAL, res.outlier_val[:n].cpu().numpy().tobytes()),
    ]
    if not interp and res.lr_flags is not None:   # SZ3-LR: the per-block predictor flags as a bitmap
        import numpy as np
        host.append((SEC_LR_FLAGS, np.packbits(res.lr_flags.cpu().numpy(), bitorder="little").tobytes()))
    secs = (Section * len(host))()
    keep = []
    for i, (tag, b) in enumerate(host):
        buf = ctypes.create_string_buffer(b, len(b)) if b else None
        keep.append(buf)
        secs[i] = Section(tag, ctypes.cast(buf, ctypes.c_void_p) if buf else None, len(b))
    s3 = _shape3(res.shape)
    hdr = StreamHeader(_dtype_id(res.dtype), len(res.shape), (ctypes.c_uint64 * 3)(*s3),
                       {"abs": SZ3G_EB_ABS, "rel": SZ3G_EB_REL_RANGE}[eb_mode],
                       float(res.eb_abs if eb is None else eb), float(res.eb_abs), res.radius, BLOCK, hs.chunk,
                       table.max_len, STREAM_INTERP if interp else (STREAM_LR if res.lr_flags is not None else 0), n,
                       0 if interp else res.coef_codes.shape[0], int(res.dim0_offset))
    lib = load()
    size = int(lib.sz3g_stream_size(secs, len(host)))
    out = ctypes.create_string_buffer(size)
    wr = ctypes.c_uint64(0)
    _check(lib.sz3g_stream_write(ctypes.byref(hdr), secs, len(host), out, size, ctypes.byref(wr)),
           "sz3g_stream_write")
    return out.raw[:wr.value]


def from_bytes(buf: bytes, device=None) -> torch.Tensor:
    """Parse and validate a container (sz3g_stream_read), then decode on the GPU: codebooks from their
    lengths, Huffman decode of codes and coefficient symbols, coefficient deltas, regression
    decompression and the outlier scatter."""
    import numpy as np
    lib = load()
    device = device or torch.device("cuda", torch.cuda.current_device())
    hdr = StreamHeader()
    secs = (Section * 16)()
    nsec, bad = ctypes.c_uint32(0), ctypes.c_uint32(0)
    rc = lib.sz3g_stream_read(buf, len(buf), ctypes.byref(hdr), secs, 16, ctypes.byref(nsec), ctypes.byref(bad))
    if rc != 0:
        raise SZ3GError(f"corrupt stream (section tag {bad.value})" if rc == -5 else f"sz3g_stream_read: {_ERR.get(rc, rc)}")
    # header / section consistency BEFORE anything is launched (sizes, offsets, codebooks, indices)
    rc = lib.sz3g_stream_validate(ctypes.byref(hdr), secs, nsec.value, ctypes.byref(bad))
    if rc != 0:
        raise SZ3GError(f"corrupt stream: inconsistent {'header' if bad.value == 0 else f'section {bad.value}'}")
    sec = {secs[i].tag: ctypes.string_at(secs[i].data, secs[i].bytes) if secs[i].bytes else b""
           for i in range(nsec.value)}
    dtype = {SZ3G_F32: torch.float32, SZ3G_F64: torch.float64}[hdr.dtype]
    shape = tuple(int(d) for d in hdr.dims)[3 - hdr.ndim:]
    N = int(np.prod(shape))
    R, ml, chunk, nb = hdr.radius, hdr.max_len, hdr.chunk, int(hdr.nblocks)

    def table_from(book: bytes, nsym: int) -> HuffmanTable:
        L = _book_lengths(book, nsym, device)
        cws = torch.empty(nsym, dtype=torch.int32, device=device)
        dt = torch.empty(int(lib.sz3g_huffman_dtable_bytes(nsym)), dtype=torch.uint8, device=device)
        st = torch.zeros(1, dtype=torch.int32, device=device)
        _check(lib.sz3g_huffman_codebook_from_lengths(_ptr(L), nsym, ml, _ptr(cws), _ptr(dt), _ptr(st),
                                                      _stream()), "sz3g_huffman_codebook_from_lengths")
        return HuffmanTable(L, cws, dt, ml, st).check()

    def stream_from(offs: bytes, data: bytes, n: int) -> HuffmanStream:
        o = torch.from_numpy(np.frombuffer(offs, np.int64).copy()).to(device)
        p = torch.from_numpy(np.frombuffer(data, np.int32).copy() if data else np.zeros(1, np.int32)).to(device)
        return HuffmanStream(n, chunk, o, p, torch.zeros(1, dtype=torch.int32, device=device))

    t_codes = table_from(sec[SEC_CODE_BOOK], 2 * R)
    hs = stream_from(sec[SEC_CODE_OFFS], sec[SEC_CODE_DATA], N)
    codes = huffman_decode(hs, t_codes).view(shape)
    if hdr.flags & STREAM_INTERP:   # SZ3-Interp: no coefficients
        oidx = torch.from_numpy(np.frombuffer(sec[SEC_OUT_IDX], np.int64).copy()).to(device)
        oval = torch.from_numpy(np.frombuffer(sec[SEC_OUT_VAL], np.float32 if dtype == torch.float32 else np.float64)
                                .copy()).to(device)
        out = interp_decompress(codes, oidx, oval, int(hdr.n_outliers), hdr.eb_abs, R, dtype)
        out = out.view(shape)
        torch.cuda.synchronize()
        if int(hs.status.item()):
            raise SZ3GError("corrupt Huffman stream")
        return out
    t_coef = table_from(sec[SEC_COEF_BOOK], 65536)
    cs = stream_from(sec[SEC_COEF_OFFS], sec[SEC_COEF_DATA], 4 * nb)
    esc = torch.from_numpy(np.frombuffer(sec[SEC_COEF_ESC], np.int64).copy()).to(device)
    coef_status = torch.zeros(1, dtype=torch.int32, device=device)
    coef = coef_delta_decode(huffman_decode(cs, t_coef), nb, esc, status=coef_status)
    oidx = torch.from_numpy(np.frombuffer(sec[SEC_OUT_IDX], np.int64).copy()).to(device)
    oval = torch.from_numpy(np.frombuffer(sec[SEC_OUT_VAL], np.float32 if dtype == torch.float32 else np.float64)
                            .copy()).to(device)
    oidx = oidx if oidx.numel() else torch.zeros(1, dtype=torch.int64, device=device)
    oval = oval if oval.numel() else torch.zeros(1, dtype=dtype, device=device)
    if hdr.flags & STREAM_LR:
        if SEC_LR_FLAGS not in sec:
            raise SZ3GError("corrupt stream: SZ3-LR stream without its flags section")
        bits = np.unpackbits(np.frombuffer(sec[SEC_LR_FLAGS], np.uint8), bitorder="little")[:nb]
        if bits.size != nb:
            raise SZ3GError("corrupt stream: short SZ3-LR flags section")
        fl = torch.from_numpy(bits.astype(np.uint8)).to(device)
        out = lr_decompress(codes, coef, fl, oidx, oval, int(hdr.n_outliers), hdr.eb_abs, R, dtype,
                            dim0_offset=int(hdr.dim0_offset))
    else:
        out = regression_decompress(codes, coef, oidx, oval, int(hdr.n_outliers), hdr.eb_abs, R, dtype,
                                    dim0_offset=int(hdr.dim0_offset))
    torch.cuda.synchronize()
    if int(hs.status.item()) or int(cs.status.item()):
        raise SZ3GError("corrupt Huffman stream")
    if int(coef_status.item()):
        raise SZ3GError("corrupt coefficient stream (escape list)")
    return out
