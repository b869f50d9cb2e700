"""Pipelined round trip of a sequence of fields held in host memory (a time series): for every field,
host->device copy, REL compression (analyze -> quantise), Huffman coding of the codes and of the
coefficient codes, decompression, and device->host copies of the compressed stream and of the
reconstruction -- with the copies of consecutive fields overlapped.

Three CUDA streams: `s_in` (host -> device), `s_comp` (all kernels, in order) and `s_out`
(device -> host).  Device inputs and outputs are double-buffered, so while field k is computed, field
k + 1 is copied in and field k - 1 is copied out on the other copy engine (PCIe is full duplex).  The
sizes of the variable-length sections (Huffman payload words, escapes, outliers) are read after field
k's compute has finished -- by then field k + 1's copy-in and compute are already enqueued -- and the
exact number of bytes is copied out.  Every kernel is a libsz3g kernel; this module only orders them
(streams and events are plumbing).  The per-field result is the compressed representation (payload,
chunk offsets, canonical code lengths, coefficient stream, outliers) in pinned host memory plus the
reconstruction x'.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from paper_2111_02925_b200 import dist as pdist
from paper_2111_02925_b200 import sz3g


@dataclass
class HostResult:
    """Compressed field in pinned host memory (views valid until the next use of the slot)."""
    payload: torch.Tensor        # int32 [words]
    offsets: torch.Tensor        # int64 [nchunks + 1]
    code_lengths: torch.Tensor   # uint8 [2R]
    coef_payload: torch.Tensor
    coef_offsets: torch.Tensor
    coef_lengths: torch.Tensor   # uint8 [65536]
    coef_escapes: torch.Tensor
    outlier_idx: torch.Tensor
    outlier_val: torch.Tensor
    eb_abs: float
    lr_flags: torch.Tensor | None = None   # SZ3-LR: uint8 [NB] predictor flags (1 = Lorenzo)

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (
            self.payload, self.offsets, self.coef_payload, self.coef_offsets, self.coef_escapes,
            self.outlier_idx, self.outlier_val)) + 4 + 3 * int((self.code_lengths > 0).sum()) + \
            4 + 3 * int((self.coef_lengths > 0).sum()) + \
            ((self.lr_flags.numel() + 7) // 8 if self.lr_flags is not None else 0)   # flags as a bitmap


class PipelinedCodec:
    def __init__(self, shape, dtype: torch.dtype, eb: float, eb_mode: str = "rel", radius: int = 32768,
                 device=None, outlier_cap: int | None = None, dim0_offset: int = 0, predictor: str = "regression"):
        """shape / dim0_offset: this rank's block-aligned slab when the field is sharded
        (torch.distributed initialised): the range and the histogram are then all-reduced.
        predictor: "regression" (the block regression predictor) or "lr" (SZ3-LR: per block the better of
        regression and the prequantised Lorenzo predictor)."""
        if predictor not in ("regression", "lr"):
            raise ValueError(f"unknown predictor {predictor!r}")
        self.predictor = predictor
        self.shape, self.dtype, self.eb, self.eb_mode, self.radius = tuple(shape), dtype, eb, eb_mode, radius
        self.dim0_offset = dim0_offset
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        n = 1
        for s_ in shape:
            n *= int(s_)
        self.n = n
        self.s_in, self.s_comp, self.s_out = (torch.cuda.Stream(dev) for _ in range(3))
        self.x = [torch.empty(self.shape, dtype=dtype, device=dev) for _ in range(2)]
        self.out = [torch.empty(self.shape, dtype=dtype, device=dev) for _ in range(2)]
        self.bufs = [sz3g.CompressBuffers(self.shape, dtype, radius, outlier_cap, dev) for _ in range(2)]
        for b in self.bufs:
            b.beta_buffer()
            if predictor == "lr":
                b.flags_buffer()
        nch = -(-n // sz3g.HUFF_CHUNK)
        cap = -(-n * sz3g.HUFF_MAX_LEN // 32) + nch
        self.payload = [torch.empty(cap, dtype=torch.int32, device=dev) for _ in range(2)]
        self.offsets = [torch.empty(nch + 1, dtype=torch.int64, device=dev) for _ in range(2)]
        lib = sz3g.load()
        self.enc_scratch = torch.empty(int(lib.sz3g_huffman_encode_scratch_bytes(n, sz3g.HUFF_CHUNK)),
                                       dtype=torch.uint8, device=dev)
        self.ev_in = [torch.cuda.Event() for _ in range(2)]
        self.ev_comp = [torch.cuda.Event() for _ in range(2)]
        self.ev_out = [torch.cuda.Event() for _ in range(2)]
        self.ev_xfree = [torch.cuda.Event() for _ in range(2)]
        self.state = [None, None]
        self.h_payload = torch.empty(cap, dtype=torch.int32, pin_memory=True)
        self.h_sizes = [torch.zeros(7, dtype=torch.int64, pin_memory=True) for _ in range(2)]
        self.h_offsets = torch.empty(nch + 1, dtype=torch.int64, pin_memory=True)
        # pinned host buffers of the small sections, sized for their maxima (no allocation per field:
        # a pinned allocation can synchronise the device)
        nb = self.bufs[0].coef_codes.shape[0]
        cnch = -(-4 * nb // sz3g.HUFF_CHUNK)
        ocap = self.bufs[0].outlier_idx.numel()
        self.h_small = [
            torch.empty(2 * radius, dtype=torch.uint8, pin_memory=True),                       # code lengths
            torch.empty(-(-4 * nb * sz3g.HUFF_MAX_LEN // 32) + cnch, dtype=torch.int32, pin_memory=True),
            torch.empty(cnch + 1, dtype=torch.int64, pin_memory=True),                         # coef offsets
            torch.empty(65536, dtype=torch.uint8, pin_memory=True),                            # coef lengths
            torch.empty(max(1, nb), dtype=torch.int64, pin_memory=True),                       # escapes
            torch.empty(ocap, dtype=torch.int64, pin_memory=True),                             # outlier idx
            torch.empty(ocap, dtype=dtype, pin_memory=True),                                   # outlier val
            torch.empty(max(1, nb), dtype=torch.uint8, pin_memory=True),                       # LR flags
        ]

    # ------------------------------------------------------------------ stages
    def _copy_in(self, k: int, host_x: torch.Tensor):
        b = k % 2
        with torch.cuda.stream(self.s_in):
            self.s_in.wait_event(self.ev_xfree[b])          # field k - 2 no longer reads x[b]
            self.x[b].copy_(host_x, non_blocking=True)
            self.ev_in[b].record(self.s_in)

    def _compute(self, k: int):
        b = k % 2
        x, bufs, st = self.x[b], self.bufs[b], self.s_comp
        with torch.cuda.stream(st):
            st.wait_event(self.ev_in[b])
            st.wait_event(self.ev_out[b])                    # field k - 2's outputs have left slot b
            bufs.reset()
            sz3g.regression_analyze(x, bufs.minmax, bufs.beta, stream=st)
            pdist.allreduce_range_(bufs.minmax)    # sharded: the global range (no-op on one rank)
            quantize = sz3g.lr_quantize if self.predictor == "lr" else sz3g.regression_quantize
            quantize(x, self.eb, self.eb_mode, self.radius, bufs.minmax, bufs.beta, bufs=bufs, reset=False,
                     dim0_offset=self.dim0_offset, stream=st)
            pdist.allreduce_hist_(bufs.hist)       # sharded: one codebook for every slab
            table = sz3g.huffman_codebook(bufs.hist, stream=st)
            hs = sz3g.huffman_encode(bufs.codes.view(-1), table, payload=self.payload[b], offsets=self.offsets[b],
                                     scratch=self.enc_scratch, stream=st)
            coef = sz3g.encode_coefficients(bufs.coef_codes, stream=st, sync=False)
            if self.predictor == "lr":
                sz3g.lr_decompress(bufs.codes, bufs.coef_codes, bufs.lr_flags, bufs.outlier_idx, bufs.outlier_val,
                                   bufs.outlier_idx.numel(), self.eb, self.radius, self.dtype,
                                   dim0_offset=self.dim0_offset, out=self.out[b],
                                   d_outlier_count=bufs.outlier_count, eb_mode=self.eb_mode,
                                   d_minmax=bufs.minmax, stream=st)
            else:
                sz3g.regression_decompress(bufs.codes, bufs.coef_codes, bufs.outlier_idx, bufs.outlier_val,
                                           bufs.outlier_idx.numel(), self.eb, self.radius, self.dtype,
                                           dim0_offset=self.dim0_offset, out=self.out[b],
                                           d_outlier_count=bufs.outlier_count, eb_mode=self.eb_mode,
                                           d_minmax=bufs.minmax, stream=st)
            # the sizes the copy-out needs, gathered on this stream into pinned host memory: no
            # operation on the legacy default stream (it would wait for every other stream's work)
            sizes = torch.stack([bufs.status.to(torch.int64)[0], bufs.outlier_count[0],
                                 bufs.eb_abs.view(torch.int64)[0], self.offsets[b][-1], coef.stream.offsets[-1],
                                 coef.n_escapes[0], table.status.to(torch.int64)[0] | hs.status.to(torch.int64)[0]])
            self.h_sizes[b].copy_(sizes, non_blocking=True)
            self.ev_xfree[b].record(st)
            self.ev_comp[b].record(st)
        self.state[b] = (table, hs, coef)

    def _copy_out(self, k: int, host_out: torch.Tensor) -> HostResult:
        b = k % 2
        bufs = self.bufs[b]
        table, hs, coef = self.state[b]
        self.ev_comp[b].synchronize()                        # sizes of the variable-length sections
        status, n_out, eb_bits, words, cw, nesc, hstat = (int(v) for v in self.h_sizes[b].tolist())
        if status & sz3g.STATUS_BAD_RANGE:
            raise sz3g.SZ3GError("bad value range")
        if status & sz3g.STATUS_OUTLIER_OVERFLOW:
            raise sz3g.SZ3GError("outlier capacity exceeded")
        if hstat or nesc > coef.escapes.numel():
            raise sz3g.SZ3GError("Huffman stage failed (status or escape capacity)")
        import struct
        eb_abs = struct.unpack("<d", struct.pack("<q", eb_bits))[0]
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.ev_comp[b])
            hp = self.h_payload[:words]
            hp.copy_(self.payload[b][:words], non_blocking=True)
            self.h_offsets.copy_(self.offsets[b], non_blocking=True)
            host_out.copy_(self.out[b], non_blocking=True)
            small = []
            srcs = [table.lengths, coef.stream.payload[:cw], coef.stream.offsets, coef.table.lengths,
                    coef.escapes[:nesc], bufs.outlier_idx[:n_out], bufs.outlier_val[:n_out]]
            if self.predictor == "lr":
                srcs.append(bufs.lr_flags)
            for h, t in zip(self.h_small, srcs):
                hv = h[:t.numel()]
                hv.copy_(t, non_blocking=True)
                small.append(hv)
            self.ev_out[b].record(self.s_out)
        return HostResult(hp, self.h_offsets, small[0], small[1], small[2], small[3], small[4], small[5], small[6],
                          eb_abs, small[7] if self.predictor == "lr" else None)

    # ------------------------------------------------------------------ driver
    def run(self, host_fields, host_out: torch.Tensor, on_result=None) -> list:
        """Round trip every field of `host_fields` (pinned host tensors of the codec's shape); every
        reconstruction is written to `host_out` (pinned), in order.  Returns the host results' sizes
        (the payload buffers are reused: consume them in `on_result(k, HostResult)`)."""
        sizes = []
        nf = len(host_fields)
        for k in range(nf + 1):
            if k < nf:
                self._copy_in(k, host_fields[k])
                self._compute(k)
            if k >= 1:
                r = self._copy_out(k - 1, host_out)
                if on_result is not None:
                    self.s_out.synchronize()
                    on_result(k - 1, r)
                sizes.append(r)
        self.s_out.synchronize()
        return sizes
