"""Multi-rank host logic on CPU (gloo, world size 2): slab partition, the range MAX all-reduce and the
histogram SUM all-reduce.  Each rank compresses its block-aligned slab with the ORACLE (test code) and the
merged results must equal the single-process output."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2111_02925_b200.dist import all_slabs, allreduce_hist_, allreduce_range_, slab_bounds


def test_slab_bounds_cover_block_aligned():
    for n0 in (1, 5, 6, 7, 100, 1024):
        for world in (1, 2, 3, 4, 8):
            sl = all_slabs(n0, world)
            assert sl[0][0] == 0 and sl[-1][1] == n0
            for (a, b), (c, d) in zip(sl, sl[1:]):
                assert b == c
            for a, b in sl:
                assert a <= b and (a == b or a % 6 == 0)   # empty slabs when ranks > block rows
    # c5 at G=8: 171 block rows -> 22,22,22,21,21,21,21,21
    rows = [(b - a + 5) // 6 for a, b in all_slabs(1024, 8)]
    assert rows == [22, 22, 22, 21, 21, 21, 21, 21]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(42)
    f = np.cumsum(rng.normal(size=(31, 13, 20)), axis=0).astype(np.float32)
    a, b = slab_bounds(f.shape[0], world, rank)
    part = f[a:b]
    lo, hi = oracle.value_range(part)
    mm = torch.tensor([lo, hi], dtype=torch.float64)
    allreduce_range_(mm)
    res = oracle.compress(part, 1e-3, "rel", radius=64, dim0_offset=a, value_range_override=(float(mm[0]), float(mm[1])))
    h = torch.from_numpy(res.hist.copy())
    allreduce_hist_(h)
    q.put((rank, a, res.codes, res.outlier_idx, float(mm[0]), float(mm[1]), h.numpy(), res.eb_abs))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_two_ranks_match_single_process(world):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(42)
    f = np.cumsum(rng.normal(size=(31, 13, 20)), axis=0).astype(np.float32)
    whole = oracle.compress(f, 1e-3, "rel", radius=64)
    assert outs[0][4] == float(f.min()) and outs[0][5] == float(f.max())
    assert all(o[7] == whole.eb_abs for o in outs)
    assert np.array_equal(np.concatenate([o[2] for o in outs]), whole.codes)
    assert np.array_equal(np.concatenate([o[3] for o in outs]), whole.outlier_idx)
    for o in outs:
        assert np.array_equal(o[6], whole.hist)
