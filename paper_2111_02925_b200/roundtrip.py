"""One step of the hot path on device-resident data, exactly as ``bench.py`` times it (and as
``tests/test_gpu_c5.py`` checks it against the oracle).

Two-pass (REL eb, the default): ``regression_analyze`` (a0 value range + a2-a3 coefficients, one read of
x) -> MAX all-reduce of the range when sharded -> ``regression_quantize`` (a4-a7 from that beta, codes /
coefficient codes / outliers / histogram) -> SUM all-reduce of the histogram when sharded ->
``regression_decompress`` (a8 + outlier scatter, reading the device range and the device outlier
counter: no host synchronisation anywhere in the step).

Fused: ``value_range`` -> all-reduce -> ``regression_compress`` (a1-a7 in one kernel) -> all-reduce ->
``regression_decompress``.

Every kernel is a libsz3g kernel; this class only orders the calls and owns the buffers.
"""
from __future__ import annotations

import torch

from . import dist as pdist
from . import sz3g


def bench_outlier_cap(n: int) -> int:
    """Outlier capacity the bench allocates (>= 1/256 of the elements; overflow raises)."""
    return max(1 << 20, n // 256)


class RoundTrip:
    """compress -> decompress of one (slab of a) field, buffers preallocated; ``step()`` is async."""

    def __init__(self, x: torch.Tensor, eb: float, eb_mode: str = "rel", radius: int = 32768, dim0_offset: int = 0,
                 path: str = "two-pass", outlier_cap: int | None = None, group=None, stream=None):
        if path not in ("two-pass", "fused"):
            raise ValueError(path)
        self.x, self.eb, self.eb_mode, self.radius = x, eb, eb_mode, radius
        self.dim0_offset, self.path, self.group = dim0_offset, path, group
        self.stream = stream if stream is not None else torch.cuda.current_stream(x.device)
        self.cap = outlier_cap if outlier_cap is not None else bench_outlier_cap(x.numel())
        self.bufs = sz3g.CompressBuffers(x.shape, x.dtype, radius, outlier_cap=self.cap, device=x.device)
        self.beta = self.bufs.beta_buffer() if path == "two-pass" else None
        self.out = torch.empty_like(x)

    def step(self, record=None):
        """One pass of the whole hot path.  ``record``: 6 CUDA events recorded on the stream at
        [quantise start, quantise end, decompress start, decompress end, analyze start, analyze end]."""
        x, b, st = self.x, self.bufs, self.stream
        ev = (lambda i: record[i].record(st)) if record is not None else (lambda i: None)
        ev(4)
        if self.path == "two-pass":
            sz3g.regression_analyze(x, b.minmax, self.beta, stream=st)
        else:
            sz3g.value_range(x, b.minmax, stream=st)
        ev(5)
        with torch.cuda.stream(st):
            pdist.allreduce_range_(b.minmax, self.group)
            b.reset()
        ev(0)
        if self.path == "two-pass":
            sz3g.regression_quantize(x, self.eb, self.eb_mode, self.radius, b.minmax, self.beta, bufs=b, reset=False,
                                     dim0_offset=self.dim0_offset, stream=st)
        else:
            sz3g.regression_compress(x, self.eb, self.eb_mode, self.radius, d_minmax=b.minmax, bufs=b, reset=False,
                                     dim0_offset=self.dim0_offset, stream=st)
        ev(1)
        with torch.cuda.stream(st):
            pdist.allreduce_hist_(b.hist, self.group)
        ev(2)
        sz3g.regression_decompress(b.codes, b.coef_codes, b.outlier_idx, b.outlier_val, self.cap, self.eb,
                                   self.radius, x.dtype, dim0_offset=self.dim0_offset, out=self.out,
                                   d_outlier_count=b.outlier_count, eb_mode=self.eb_mode, d_minmax=b.minmax,
                                   stream=st)
        ev(3)

    def result(self) -> sz3g.Compressed:
        """The last step's compressed outputs (synchronises; raises on device status bits)."""
        b = self.bufs
        return sz3g.Compressed(tuple(self.x.shape), self.x.dtype, self.radius, self.dim0_offset, b.codes,
                               b.coef_codes, self.beta, b.outlier_idx, b.outlier_val, b.outlier_count, b.hist,
                               b.eb_abs, b.status).finalize()
