"""The multi-rank GPU path rehearsed on ONE GPU: two processes, each with its
block-aligned slab on cuda:0, the range MAX all-reduce and the histogram SUM all-reduce through a gloo
process group (CUDA tensors staged through the host; nothing waits inside a kernel on another rank).

* RoundTrip (the bench's step) on 2 ranks == the 1-rank run: concatenated codes, coefficient codes,
  outlier sets (global indices), merged histogram, eb_abs and x' bit-identical (slab invariance, P8).
* PipelinedCodec sharded: x' identical and one shared codebook (the merged histogram's) on both ranks.
* bench.py under torchrun with --dist-backend gloo prints a valid N = 2 line.
"""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPE = (100, 130, 256)     # 17 block rows: ranks get 9 + 8, the last slab ragged (4 planes)
EB, R = 1e-3, 8             # R = 8: ~0.5% radius outliers on this lognormal field, so the outlier path is sharded too


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tmp):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2111_02925_b200 import sz3g
    from paper_2111_02925_b200.dist import slab_bounds
    from paper_2111_02925_b200.pipeline import PipelinedCodec
    from paper_2111_02925_b200.roundtrip import RoundTrip
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sz3g.load()
    full = np.load(os.path.join(tmp, "field.npy"))
    a, b = slab_bounds(full.shape[0], world, rank)
    x = torch.from_numpy(full[a:b].copy()).cuda()
    rt = RoundTrip(x, EB, "rel", R, dim0_offset=a, outlier_cap=x.numel())
    rt.step()
    rt.step()
    res = rt.result()
    n = res.n_outliers
    out = dict(a=a, codes=res.codes.cpu().numpy(), coef=res.coef_codes.cpu().numpy(),
               oidx=res.outlier_idx[:n].cpu().numpy(), oval=res.outlier_val[:n].cpu().numpy(),
               hist=res.hist.cpu().numpy(), eb_abs=np.float64(res.eb_abs), minmax=rt.bufs.minmax.cpu().numpy(),
               xo=rt.out.cpu().numpy())
    # the pipelined codec, sharded: host field -> ... -> host x' and compressed sections
    h_x = x.cpu().pin_memory()
    h_out = torch.empty_like(h_x).pin_memory()
    codec = PipelinedCodec(tuple(x.shape), x.dtype, EB, "rel", R, outlier_cap=x.numel(), dim0_offset=a)
    got = {}
    codec.run([h_x], h_out, on_result=lambda k, r: got.update(lens=r.code_lengths.clone(), xo=h_out.clone()))
    out["pipe_xo"] = got["xo"].numpy()
    out["pipe_lens"] = got["lens"].numpy()
    np.savez(os.path.join(tmp, f"rank{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_single_rank():
    import torch.multiprocessing as mp
    from paper_2111_02925_b200 import sz3g
    from paper_2111_02925_b200.roundtrip import RoundTrip
    from synth import make_field
    sz3g.load()
    x = make_field("c3", device="cuda", shape=SHAPE)
    with tempfile.TemporaryDirectory() as tmp:
        np.save(os.path.join(tmp, "field.npy"), x.cpu().numpy())
        ctx = mp.get_context("spawn")
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, 2, port, tmp)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=600)
            assert p.exitcode == 0
        outs = [dict(np.load(os.path.join(tmp, f"rank{r}.npz"))) for r in range(2)]
    # the single-rank run (no process group: the all-reduces are no-ops)
    rt = RoundTrip(x, EB, "rel", R, outlier_cap=x.numel())
    rt.step()
    res = rt.result()
    n = res.n_outliers
    assert n > 1000
    assert np.array_equal(np.concatenate([o["codes"] for o in outs]), res.codes.cpu().numpy())
    assert np.array_equal(np.concatenate([o["coef"] for o in outs]), res.coef_codes.cpu().numpy())
    xo = rt.out.cpu().numpy()
    assert np.array_equal(np.concatenate([o["xo"] for o in outs]).view(np.uint32), xo.view(np.uint32))
    gi = np.concatenate([o["oidx"] for o in outs])
    gv = np.concatenate([o["oval"] for o in outs])
    oi, ov = res.outlier_idx[:n].cpu().numpy(), res.outlier_val[:n].cpu().numpy()
    g, w = np.argsort(gi), np.argsort(oi)
    assert np.array_equal(gi[g], oi[w]) and np.array_equal(gv[g].view(np.uint32), ov[w].view(np.uint32))
    for o in outs:
        assert np.array_equal(o["hist"], res.hist.cpu().numpy())        # merged histogram
        assert float(o["eb_abs"]) == res.eb_abs                          # global range -> same eb
        assert np.array_equal(o["minmax"], rt.bufs.minmax.cpu().numpy())
    # sharded pipelined codec: same reconstruction, one codebook (from the merged histogram)
    assert np.array_equal(np.concatenate([o["pipe_xo"] for o in outs]).view(np.uint32), xo.view(np.uint32))
    table = sz3g.huffman_codebook(res.hist).check()
    for o in outs:
        assert np.array_equal(o["pipe_lens"], table.lengths.cpu().numpy())


def test_bench_two_ranks_gloo():
    """bench.py's N > 1 branch (torchrun, slabs, all-reduces, max-over-ranks timing, sharded e2e)
    rehearsed with gloo on one GPU at a cropped c5 shape."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--dist-backend", "gloo", "--shape", "96,1024,1024", "--steps", "3", "--warmup", "3",
           "--e2e-steps", "2", "--huffman-reps", "2", "--configs", ""]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "slabs2" and d["config"]["dist_backend"] == "gloo"
    assert d["quality"]["above_eb"] == 0 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["roofline"]["ranks"] == "max over ranks"
    print(json.dumps({k: d[k] for k in ("value", "ms_per_step", "compress_gbs", "decompress_gbs")}))


def test_roundtrip_cuda_graph_replay_bit_identical():
    """RoundTrip.capture(): the step replayed from CUDA graphs (the bench's per-config legs) gives the
    eager step's outputs bit for bit, replay after replay."""
    from paper_2111_02925_b200 import sz3g
    from paper_2111_02925_b200.roundtrip import RoundTrip
    from synth import make_field
    sz3g.load()
    for name, shape, R in (("c3", (60, 96, 200), 8), ("c4", (30, 64, 96), 32768), ("c2", (24, 50, 50), 32768)):
        x = make_field(name, device="cuda", shape=shape)
        eager = RoundTrip(x, 1e-3, "rel", R, outlier_cap=x.numel())
        eager.step()
        e = eager.result()
        g = RoundTrip(x, 1e-3, "rel", R, outlier_cap=x.numel()).capture()
        for _ in range(3):
            g.out.zero_()
            g.step()
            r = g.result()
            assert torch.equal(r.codes, e.codes) and torch.equal(r.coef_codes, e.coef_codes)
            assert torch.equal(r.hist, e.hist) and r.n_outliers == e.n_outliers
            assert torch.equal(g.out.view(torch.uint8), eager.out.view(torch.uint8)), name
