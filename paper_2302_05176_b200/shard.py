"""Multi-GPU partitioning (one process per GPU, torch.distributed plumbing).

Two shapes, SURVEY.md section 8(e):
  * a batch of independent vectors (configs 2-3): contiguous vector ranges
    balanced by element count; no data-path collective.
  * one huge vector or stream (configs 4-5): contiguous element ranges, a
    sketch per rank, then ONE exchange: every rank all-gathers the k
    registers (k x 16 B) and min-merges them in rank order with the device
    merge kernel, which reproduces merge([sketch_rank0, sketch_rank1, ...])
    exactly (estimate.py:103-125; partition law test_estimate.py:174-199).
    `allreduce_min_registers` is the collective-only alternative: two
    all-reduces with MIN (y, then the ids of the registers that hold the
    minimum), the register-wise lexicographic (y, id) minimum -- the whole
    element set's sketch (sketch_naive's smaller-id tie rule, sketch.py:196-205).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def element_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of n elements for `rank`."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def vector_ranges(offsets, world: int) -> list[tuple[int, int]]:
    """Split CSR vectors into `world` contiguous ranges with near-equal
    element counts (sizes are LogNormal in config 3, so balance elements,
    not vectors).  Returns [(v_lo, v_hi)] per rank."""
    off = np.asarray(offsets, dtype=np.int64)
    n_vec = off.size - 1
    total = int(off[-1])
    cuts = [0]
    for r in range(1, world):
        target = total * r // world
        v = int(np.searchsorted(off, target, side="left"))
        cuts.append(min(max(v, cuts[-1]), n_vec))
    cuts.append(n_vec)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def gather_registers(y: torch.Tensor, s: torch.Tensor, group=None) -> tuple[torch.Tensor, torch.Tensor]:
    """All-gather one sketch's registers from every rank: ([world, k], [world, k])."""
    world = dist.get_world_size(group)
    ys = [torch.empty_like(y) for _ in range(world)]
    ss = [torch.empty_like(s) for _ in range(world)]
    dist.all_gather(ys, y.contiguous(), group=group)
    dist.all_gather(ss, s.contiguous(), group=group)
    return torch.stack(ys), torch.stack(ss)


def merge_across_ranks(y: torch.Tensor, s: torch.Tensor, group=None) -> tuple[torch.Tensor, torch.Tensor]:
    """Exchange + device min-merge: every rank ends with the merged sketch."""
    from .estimate import merge_arrays

    ya, sa = gather_registers(y, s, group)
    return merge_arrays(ya, sa)


_SIGN = 1 << 63


def allreduce_min_registers(y: torch.Tensor, s: torch.Tensor, group=None) -> tuple[torch.Tensor, torch.Tensor]:
    """Every rank ends with the register-wise lexicographic minimum of
    (y, s) over the ranks: all-reduce(MIN) of y, then all-reduce(MIN) of the
    ids of the ranks that hold that minimum (others contribute the largest
    id).  Ids are unsigned 64-bit values carried in int64: the sign bit is
    flipped so that signed MIN orders them as unsigned.  Equal to the
    rank-order merge unless two ranks hold different elements with the very
    same y bits in one register (then the smaller id wins, as in
    sketch_naive over the whole set)."""
    ym = y.clone()
    dist.all_reduce(ym, op=dist.ReduceOp.MIN, group=group)
    sign = torch.tensor(-_SIGN, dtype=torch.int64, device=s.device)  # bit pattern 1 << 63
    key = torch.where(y == ym, s ^ sign, torch.full_like(s, (1 << 63) - 1))
    dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
    return ym, key ^ sign
