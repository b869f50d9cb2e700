"""Multi-GPU plumbing: block-aligned slab sharding of a field along dim 0 and the two collectives of the
path.

* Slabs: rank r owns block-rows [sum_{r'<r} s_r', ...) with s_r = floor(NB0/G) + [r < NB0 mod G], i.e.
  planes [6*start, min(6*end, n0)).  Blocks never straddle ranks, so every rank's codes / coefficient
  codes are contiguous slices of the single-GPU output and outlier indices are global (dim0_offset).
* a0 (REL eb only): all-reduce MAX of (-min, max) so every rank uses the global value range.
* a7: all-reduce SUM of the int64 code histogram -> one shared codebook histogram.
No halo exchange: regression reads only its own block's original values.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

BLOCK = 6


def slab_bounds(n0: int, world: int, rank: int, B: int = BLOCK) -> tuple[int, int]:
    """[start, stop) planes of rank's block-aligned slab."""
    nb0 = math.ceil(n0 / B)
    base, extra = divmod(nb0, world)
    start_blk = rank * base + min(rank, extra)
    nblk = base + (1 if rank < extra else 0)
    return min(start_blk * B, n0), min((start_blk + nblk) * B, n0)


def all_slabs(n0: int, world: int, B: int = BLOCK) -> list[tuple[int, int]]:
    return [slab_bounds(n0, world, r, B) for r in range(world)]


def allreduce_range_(minmax: torch.Tensor, group=None) -> torch.Tensor:
    """In place: minmax = [global min, global max] (one MAX all-reduce of [-min, max], 16 B)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return minmax
    t = torch.stack([-minmax[0], minmax[1]])
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    minmax[0] = -t[0]
    minmax[1] = t[1]
    return minmax


def allreduce_hist_(hist: torch.Tensor, group=None) -> torch.Tensor:
    """In place SUM of the int64 histogram over ranks (2R x 8 B = 512 KiB at R = 32768)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    return hist
