"""PipelinedCodec (copy / compute overlap over a sequence of host fields): every field's host results
equal the direct path -- reconstruction bit-identical to decompress(compress(x)), Huffman payload and
offsets equal to huffman_encode of the same codes, the coefficient stream decodes to the coefficient
codes."""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def test_pipeline_matches_direct():
    from paper_2111_02925_b200 import sz3g
    from paper_2111_02925_b200.pipeline import PipelinedCodec
    from synth import config_by_name, make_field
    cfg = config_by_name("c2")
    fields = [make_field(cfg, device="cuda", shape=(48, 96, 120)) * (1.0 + 0.5 * k) for k in range(3)]
    hosts = [f.cpu().pin_memory() for f in fields]
    h_out = torch.empty_like(hosts[0]).pin_memory()
    codec = PipelinedCodec(tuple(fields[0].shape), fields[0].dtype, cfg.eb, cfg.eb_mode, cfg.radius)
    got = {}

    def keep(k, r):
        got[k] = (h_out.clone(), r.payload.clone(), r.offsets.clone(), r.coef_payload.clone(), r.coef_offsets.clone(),
                  r.coef_lengths.clone(), r.coef_escapes.clone(), r.code_lengths.clone())

    codec.run(hosts, h_out, on_result=keep)
    for k, x in enumerate(fields):
        res = sz3g.compress(x, cfg.eb, cfg.eb_mode, cfg.radius)
        direct = sz3g.decompress(res).cpu()
        xo, pay, offs, cpay, coffs, clen, cesc, lens = got[k]
        assert torch.equal(xo.view(torch.int32), direct.view(torch.int32))
        table = sz3g.huffman_codebook(res.hist).check()
        hs = sz3g.huffman_encode(res.codes.view(-1), table).check()
        assert torch.equal(lens, table.lengths.cpu())
        assert torch.equal(offs, hs.offsets.cpu()) and torch.equal(pay, hs.payload[:hs.words()].cpu())
        cs = sz3g.encode_coefficients(res.coef_codes)
        assert torch.equal(cpay, cs.stream.payload[:cs.stream.words()].cpu())
        assert torch.equal(cesc, cs.escapes.cpu()) and torch.equal(clen, cs.table.lengths.cpu())


def test_pipeline_lr_matches_direct():
    """predictor="lr": every field's reconstruction equals decompress(lr_compress(x)) bit for bit, and the
    flags reach the host."""
    from paper_2111_02925_b200 import sz3g
    from paper_2111_02925_b200.pipeline import PipelinedCodec
    from synth import config_by_name, make_field
    cfg = config_by_name("c2")
    fields = [make_field(cfg, device="cuda", shape=(48, 96, 120)) * (1.0 + 0.5 * k) for k in range(3)]
    hosts = [f.cpu().pin_memory() for f in fields]
    h_out = torch.empty_like(hosts[0]).pin_memory()
    codec = PipelinedCodec(tuple(fields[0].shape), fields[0].dtype, cfg.eb, cfg.eb_mode, cfg.radius, predictor="lr")
    got = {}
    codec.run(hosts, h_out, on_result=lambda k, r: got.__setitem__(k, (h_out.clone(), r.lr_flags.clone())))
    for k, x in enumerate(fields):
        res = sz3g.lr_compress(x, cfg.eb, cfg.eb_mode, cfg.radius)
        direct = sz3g.decompress(res).cpu()
        xo, fl = got[k]
        assert torch.equal(xo.view(torch.int32), direct.view(torch.int32))
        assert torch.equal(fl, res.lr_flags.cpu()) and int(fl.sum()) > 0


def test_pipeline_slots_do_not_alias_and_sizes():
    """The two slots own separate pinned buffers (r1: HostResults of consecutive fields aliased): when
    field k + 1 is on the host, field k's result is still intact; run() returns each field's
    compressed size, equal to HostResult.nbytes()."""
    from paper_2111_02925_b200.pipeline import PipelinedCodec
    from synth import config_by_name, make_field
    cfg = config_by_name("c2")
    fields = [make_field(cfg, device="cuda", shape=(48, 96, 120)) * (1.0 + 0.5 * k) for k in range(4)]
    hosts = [f.cpu().pin_memory() for f in fields]
    h_out = torch.empty_like(hosts[0]).pin_memory()
    codec = PipelinedCodec(tuple(fields[0].shape), fields[0].dtype, cfg.eb, cfg.eb_mode, cfg.radius)
    live, snap, nb = {}, {}, {}

    def on(k, r):
        live[k], snap[k], nb[k] = r, (r.payload.clone(), r.code_lengths.clone(), r.outlier_idx.clone()), r.nbytes()
        if k >= 1:   # the previous field's result is untouched by this one
            p, lens, oi = snap[k - 1]
            assert live[k - 1].payload.data_ptr() != r.payload.data_ptr()
            assert torch.equal(live[k - 1].payload, p) and torch.equal(live[k - 1].code_lengths, lens)
            assert torch.equal(live[k - 1].outlier_idx, oi)

    sizes = codec.run(hosts, h_out, on_result=on)
    assert sizes == [nb[k] for k in range(4)]


def test_pipeline_interp_matches_direct():
    """predictor="interp": every field's reconstruction equals interp_decompress(interp_compress(x)) bit
    for bit, its Huffman payload equals huffman_encode of the same codes, there are no coefficient
    sections, and run()'s sizes equal HostResult.nbytes()."""
    from paper_2111_02925_b200 import sz3g
    from paper_2111_02925_b200.pipeline import PipelinedCodec
    from synth import config_by_name, make_field
    cfg = config_by_name("c2")
    fields = [make_field(cfg, device="cuda", shape=(40, 72, 130)) * (1.0 + 0.5 * k) for k in range(3)]
    hosts = [f.cpu().pin_memory() for f in fields]
    h_out = torch.empty_like(hosts[0]).pin_memory()
    R = 512
    n = fields[0].numel()
    codec = PipelinedCodec(tuple(fields[0].shape), fields[0].dtype, cfg.eb, cfg.eb_mode, R, outlier_cap=n,
                           predictor="interp")
    got = {}
    codec.run(hosts, h_out, on_result=lambda k, r: got.__setitem__(
        k, (h_out.clone(), r.payload.clone(), r.offsets.clone(), r.coef_payload.numel(), r.outlier_idx.numel(),
            r.nbytes())))
    for k, x in enumerate(fields):
        res = sz3g.interp_compress(x, cfg.eb, cfg.eb_mode, R, outlier_cap=n).finalize()
        direct = sz3g.interp_decompress(res.codes, res.outlier_idx, res.outlier_val, res.n_outliers, res.eb_abs, R,
                                        x.dtype).cpu()
        xo, pay, offs, ncp, nout, _ = got[k]
        assert torch.equal(xo.view(torch.int32), direct.view(torch.int32))
        table = sz3g.huffman_codebook(res.hist).check()
        hs = sz3g.huffman_encode(res.codes.view(-1), table).check()
        assert torch.equal(offs, hs.offsets.cpu()) and torch.equal(pay, hs.payload[:hs.words()].cpu())
        assert ncp == 0 and nout == res.n_outliers > 0
    sizes = codec.run(hosts, h_out, on_result=lambda k, r: got.__setitem__(k, r.nbytes()))
    assert sizes == [got[k] for k in range(3)]

