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
        # sharded: the histogram all-reduce (needed by the codebook, not by decompression) runs on a side
        # stream, overlapped with the decompression; the next step's reset and finish() wait for it
        self.side = torch.cuda.Stream(x.device)
        self._ev_q = torch.cuda.Event()
        self._ev_h = torch.cuda.Event()
        self._hist_pending = False

    # the step in five segments; every segment launches on the stream it is given
    def _analyze(self, st):
        if self.path == "two-pass":
            sz3g.regression_analyze(self.x, self.bufs.minmax, self.beta, stream=st)
        else:
            sz3g.value_range(self.x, self.bufs.minmax, stream=st)

    def _range_reset(self, st):
        with torch.cuda.stream(st):
            pdist.allreduce_range_(self.bufs.minmax, self.group)
            if self._hist_pending:        # the previous step's histogram all-reduce has finished
                st.wait_event(self._ev_h)
                self._hist_pending = False
            self.bufs.reset()

    def _quantize(self, st):
        x, b = self.x, self.bufs
        if self.path == "two-pass":
            sz3g.regression_quantize(x, self.eb, self.eb_mode, self.radius, b.minmax, self.beta, bufs=b, reset=False,
                                     dim0_offset=self.dim0_offset, stream=st)
        else:
            sz3g.regression_compress(x, self.eb, self.eb_mode, self.radius, d_minmax=b.minmax, bufs=b, reset=False,
                                     dim0_offset=self.dim0_offset, stream=st)

    def _hist(self, st):
        with torch.cuda.stream(st):
            pdist.allreduce_hist_(self.bufs.hist, self.group)

    def _decompress(self, st):
        b = self.bufs
        sz3g.regression_decompress(b.codes, b.coef_codes, b.outlier_idx, b.outlier_val, self.cap, self.eb,
                                   self.radius, self.x.dtype, dim0_offset=self.dim0_offset, out=self.out,
                                   d_outlier_count=b.outlier_count, eb_mode=self.eb_mode, d_minmax=b.minmax,
                                   stream=st)

    SEGMENTS = ("_analyze", "_range_reset", "_quantize", "_hist", "_decompress")
    # event index recorded after each segment (record[4] before the first): analyze end, quantise
    # start, quantise end, decompress start, decompress end
    _AFTER = (5, 0, 1, 2, 3)

    def step(self, record=None):
        """One pass of the whole hot path.  ``record``: 6 CUDA events recorded on the stream at
        [quantise start, quantise end, decompress start, decompress end, analyze start, analyze end].
        After ``capture()`` each segment is replayed from its CUDA graph (no host work per kernel)."""
        st = self.stream
        if record is not None:
            record[4].record(st)
        graphs = getattr(self, "graphs", None)
        sharded = torch.distributed.is_initialized() and torch.distributed.get_world_size(self.group) > 1
        for name, after in zip(self.SEGMENTS, self._AFTER):
            if name == "_hist" and graphs is None and sharded:   # overlapped with the decompression
                self._ev_q.record(st)
                self.side.wait_event(self._ev_q)
                self._hist(self.side)
                self._ev_h.record(self.side)
                self._hist_pending = True
                if record is not None:
                    record[after].record(st)
                continue
            if graphs is not None:
                if graphs[name] is not None:
                    with torch.cuda.stream(st):
                        graphs[name].replay()
            else:
                getattr(self, name)(st)
            if record is not None:
                record[after].record(st)

    def capture(self):
        """Capture every segment of the step in its own CUDA graph (single process or NCCL; gloo
        collectives cannot be captured).  Replays launch the same kernels with the same arguments:
        the buffers are fixed, and the kernels read the range / counters on the device."""
        if self.group is not None or (torch.distributed.is_initialized() and torch.distributed.get_world_size() > 1
                                      and torch.distributed.get_backend() != "nccl"):
            raise RuntimeError("CUDA graph capture needs a single process or NCCL")
        self.step()                      # warm: lazy attribute / descriptor setup outside the capture
        torch.cuda.synchronize()
        graphs = {}
        l0 = sz3g.launch_count()
        sharded = torch.distributed.is_initialized() and torch.distributed.get_world_size() > 1
        for name in self.SEGMENTS:
            if name == "_hist" and not sharded:   # no collective: nothing to launch
                graphs[name] = None
                continue
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                getattr(self, name)(torch.cuda.current_stream())
            graphs[name] = g
        torch.cuda.synchronize()
        self.graphs = graphs
        self.launches_per_step = sz3g.launch_count() - l0   # library kernels in one replayed step
        return self

    def capture_timed(self, record):
        """The whole step as ONE CUDA graph whose six timing events (``record``, created with
        ``external=True``) are nodes of the graph, recorded at the segment boundaries exactly as
        ``step(record)`` records them.  ``replay_timed()`` then runs the step with no host work and no
        graph-launch gap between segments (small fields: the per-segment graphs of ``capture()`` put a
        launch boundary inside every timed segment).  Single process only."""
        if torch.distributed.is_initialized() and torch.distributed.get_world_size(self.group) > 1:
            raise RuntimeError("capture_timed is single-process")
        self.step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            st = torch.cuda.current_stream()
            record[4].record(st)
            for name, after in zip(self.SEGMENTS, self._AFTER):
                if name != "_hist":           # single process: no collective
                    getattr(self, name)(st)
                record[after].record(st)
        torch.cuda.synchronize()
        self.timed_graph, self.timed_record = g, record
        return self

    def replay_timed(self):
        """One step from the ``capture_timed`` graph; its events hold this step's segment times."""
        with torch.cuda.stream(self.stream):
            self.timed_graph.replay()

    def finish(self):
        """Make the stream wait for the last step's histogram all-reduce (part of the step's output)."""
        if self._hist_pending:
            self.stream.wait_event(self._ev_h)
            self._hist_pending = False

    def result(self) -> sz3g.Compressed:
        """The last step's compressed outputs (synchronises; raises on device status bits)."""
        self.finish()
        b = self.bufs
        return sz3g.Compressed(tuple(self.x.shape), self.x.dtype, self.radius, self.dim0_offset, b.codes,
                               b.coef_codes, self.beta, b.outlier_idx, b.outlier_val, b.outlier_count, b.hist,
                               b.eb_abs, b.status).finalize()
