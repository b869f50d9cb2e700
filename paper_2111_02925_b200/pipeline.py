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

from . import dist as pdist
from . import sz3g


@dataclass
class HostResult:
    """Compressed field in pinned host memory.  Each of the two slots has its own pinned buffers, so a
    result stays valid until its slot is reused two fields later (consume it in ``on_result``)."""
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
            (4 + 3 * int((self.coef_lengths > 0).sum()) if self.coef_lengths.numel() else 0) + \
            ((self.lr_flags.numel() + 7) // 8 if self.lr_flags is not None else 0)   # flags as a bitmap


class PipelinedCodec:
    def __init__(self, shape, dtype: torch.dtype, eb: float, eb_mode: str = "rel", radius: int = 32768,
                 device=None, outlier_cap: int | None = None, dim0_offset: int = 0, predictor: str = "regression"):
        """shape / dim0_offset: this rank's block-aligned slab when the field is sharded
        (torch.distributed initialised): the range and the histogram are then all-reduced.
        predictor: "regression" (the block regression predictor), "lr" (SZ3-LR: per block the better of
        regression and the prequantised Lorenzo predictor) or "interp" (SZ3-Interp, level-serial: not
        shardable, one process per field)."""
        if predictor not in ("regression", "lr", "interp"):
            raise ValueError(f"unknown predictor {predictor!r}")
        if predictor == "interp" and torch.distributed.is_initialized() and torch.distributed.get_world_size() > 1:
            raise ValueError("SZ3-Interp is not sharded: its donors cross every slab boundary")
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
        # SZ3-Interp: per-slot outputs of sz3g_interp_compress (codes, its reconstruction buffer, outliers,
        # histogram); the coefficient sections are empty
        self.ires = [None, None]
        if predictor == "interp":
            self.ires = [sz3g.InterpCompressed(self.shape, dtype, radius, 0, bf.codes, torch.empty_like(self.x[0]),
                                               bf.outlier_idx, bf.outlier_val, bf.outlier_count, bf.hist, bf.eb_abs,
                                               bf.status) for bf in self.bufs]
            self._none16 = torch.empty(0, dtype=torch.uint8, device=dev)
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
        # pinned host buffers PER SLOT (a slot's result is not overwritten by the other slot's field).
        # The payload buffer grows on demand to the payload actually produced (a pinned allocation can
        # synchronise the device, so it happens at most a few times, on the first fields).
        self.h_payload = [None, None]
        self.h_sizes = [torch.zeros(9, dtype=torch.int64, pin_memory=True) for _ in range(2)]
        self.h_offsets = [torch.empty(nch + 1, dtype=torch.int64, pin_memory=True) for _ in range(2)]
        # pinned host buffers of the small sections, sized for their maxima (no allocation per field)
        nb = self.bufs[0].coef_codes.shape[0]
        self.nb = nb
        cnch = -(-4 * nb // sz3g.HUFF_CHUNK)
        ocap = self.bufs[0].outlier_idx.numel()
        self.h_small = [[
            torch.empty(2 * radius, dtype=torch.uint8, pin_memory=True),                       # code lengths
            torch.empty(-(-4 * nb * sz3g.HUFF_MAX_LEN // 32) + cnch, dtype=torch.int32, pin_memory=True),
            torch.empty(cnch + 1, dtype=torch.int64, pin_memory=True),                         # coef offsets
            torch.empty(65536, dtype=torch.uint8, pin_memory=True),                            # coef lengths
            torch.empty(max(1, nb), dtype=torch.int64, pin_memory=True),                       # escapes
            torch.empty(ocap, dtype=torch.int64, pin_memory=True),                             # outlier idx
            torch.empty(ocap, dtype=dtype, pin_memory=True),                                   # outlier val
            torch.empty(max(1, nb), dtype=torch.uint8, pin_memory=True),                       # LR flags
        ] for _ in range(2)]

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
            if self.predictor == "interp":
                self._compute_interp(b, x, bufs, st)
                return
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
                                 coef.n_escapes[0], table.status.to(torch.int64)[0] | hs.status.to(torch.int64)[0],
                                 (table.lengths > 0).sum(), (coef.table.lengths > 0).sum()])
            self.h_sizes[b].copy_(sizes, non_blocking=True)
            self.ev_xfree[b].record(st)
            self.ev_comp[b].record(st)
        self.state[b] = (table, hs, coef)

    def _compute_interp(self, b: int, x: torch.Tensor, bufs, st):
        """SZ3-Interp for slot b (inside _compute's stream context): range, level passes, codebook, encode,
        decompression from the codes (the round trip, not the compress-time reconstruction)."""
        res = self.ires[b]
        mm = sz3g.value_range(x, bufs.minmax, stream=st) if self.eb_mode == "rel" else None
        sz3g.interp_compress(x, self.eb, self.eb_mode, self.radius, d_minmax=mm, out=res, stream=st)
        table = sz3g.huffman_codebook(res.hist, stream=st)
        hs = sz3g.huffman_encode(res.codes.view(-1), table, payload=self.payload[b], offsets=self.offsets[b],
                                 scratch=self.enc_scratch, stream=st)
        sz3g.interp_decompress(res.codes, res.outlier_idx, res.outlier_val, res.outlier_idx.numel(), self.eb,
                               self.radius, self.dtype, out=self.out[b], d_outlier_count=res.outlier_count,
                               eb_mode=self.eb_mode, d_minmax=mm, stream=st)
        z = torch.zeros((), dtype=torch.int64, device=self.dev)
        sizes = torch.stack([res.status.to(torch.int64)[0], res.outlier_count[0], res.eb_abs_dev.view(torch.int64)[0],
                             self.offsets[b][-1], z, z, table.status.to(torch.int64)[0] | hs.status.to(torch.int64)[0],
                             (table.lengths > 0).sum(), z])
        self.h_sizes[b].copy_(sizes, non_blocking=True)
        self.ev_xfree[b].record(st)
        self.ev_comp[b].record(st)
        self.state[b] = (table, hs, None)

    def _copy_out(self, k: int, host_out: torch.Tensor) -> tuple[HostResult, int]:
        b = k % 2
        bufs = self.bufs[b]
        table, hs, coef = self.state[b]
        self.ev_comp[b].synchronize()                        # sizes of the variable-length sections
        status, n_out, eb_bits, words, cw, nesc, hstat, nact, ncact = (int(v) for v in self.h_sizes[b].tolist())
        if status & sz3g.STATUS_BAD_RANGE:
            raise sz3g.SZ3GError("bad value range")
        if status & sz3g.STATUS_OUTLIER_OVERFLOW:
            raise sz3g.SZ3GError("outlier capacity exceeded")
        if hstat or (coef is not None and nesc > coef.escapes.numel()):
            raise sz3g.SZ3GError("Huffman stage failed (status or escape capacity)")
        import struct
        eb_abs = struct.unpack("<d", struct.pack("<q", eb_bits))[0]
        # the slot's pinned buffers were last read by field k - 2's consumer (on_result ran before
        # this call); the payload buffer grows if this field's payload is larger
        if self.h_payload[b] is None or self.h_payload[b].numel() < words:
            self.s_out.synchronize()
            self.h_payload[b] = torch.empty(max(1, words + words // 4), dtype=torch.int32, pin_memory=True)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.ev_comp[b])
            hp = self.h_payload[b][:words]
            hp.copy_(self.payload[b][:words], non_blocking=True)
            self.h_offsets[b].copy_(self.offsets[b], non_blocking=True)
            host_out.copy_(self.out[b], non_blocking=True)
            small = []
            if coef is None:   # SZ3-Interp: no coefficient sections
                e = self._none16
                srcs = [table.lengths, e, e, e, e, bufs.outlier_idx[:n_out], bufs.outlier_val[:n_out]]
            else:
                srcs = [table.lengths, coef.stream.payload[:cw], coef.stream.offsets, coef.table.lengths,
                        coef.escapes[:nesc], bufs.outlier_idx[:n_out], bufs.outlier_val[:n_out]]
            if self.predictor == "lr":
                srcs.append(bufs.lr_flags)
            for h, t in zip(self.h_small[b], srcs):
                hv = h[:t.numel()]
                hv.copy_(t, non_blocking=True)
                small.append(hv)
            self.ev_out[b].record(self.s_out)
        # compressed bytes of this field, from the device-side sizes (no read of the pinned data):
        # the same sum as HostResult.nbytes()
        es = torch.empty((), dtype=self.dtype).element_size()
        coef_b = 0 if coef is None else 4 * cw + 8 * coef.stream.offsets.numel() + 8 * nesc + 4 + 3 * ncact
        nbytes = 4 * words + 8 * self.offsets[b].numel() + coef_b + (8 + es) * n_out + 4 + 3 * nact + \
            ((self.nb + 7) // 8 if self.predictor == "lr" else 0)
        return HostResult(hp, self.h_offsets[b], small[0], small[1], small[2], small[3], small[4], small[5], small[6],
                          eb_abs, small[7] if self.predictor == "lr" else None), nbytes

    # ------------------------------------------------------------------ driver
    def run(self, host_fields, host_out: torch.Tensor, on_result=None) -> list[int]:
        """Round trip every field of `host_fields` (pinned host tensors of the codec's shape); every
        reconstruction is written to `host_out` (pinned), in order.  Returns each field's compressed
        size in bytes.  The compressed sections live in per-slot pinned buffers that are reused two
        fields later: consume them in `on_result(k, HostResult)` (called once field k is on the host)."""
        sizes = []
        nf = len(host_fields)
        for k in range(nf + 1):
            if k < nf:
                self._copy_in(k, host_fields[k])
                self._compute(k)
            if k >= 1:
                r, nbytes = self._copy_out(k - 1, host_out)
                if on_result is not None:
                    self.s_out.synchronize()
                    on_result(k - 1, r)
                sizes.append(nbytes)
        self.s_out.synchronize()
        return sizes
