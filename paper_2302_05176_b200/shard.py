"""Multi-GPU partitioning (one process per GPU; torch.distributed only for
the rendezvous, the register exchange is NCCL inside the C ABI).

Two shapes, SURVEY.md section 8(e):
  * a batch of independent vectors (configs 2-3): contiguous vector ranges
    balanced by element count; no data-path collective.
  * one huge vector or stream (configs 4-5): contiguous element ranges, a
    sketch per rank, then ONE exchange of the k registers (k x 16 B) over
    NCCL, in place on every rank (RegisterExchange; gm_comm.cuh):
      - allreduce_min: two all-reduces with MIN (y, then the ids of the
        ranks holding the minimum) -- the register-wise lexicographic (y, id)
        minimum, sketch_naive's smaller-id tie rule (sketch.py:196-205);
      - allgather_merge: all-gather + the device merge in rank order --
        merge([sketch_rank0, sketch_rank1, ...]) exactly (estimate.py:103-125).
    Both reproduce the whole set's sketch (partition law,
    test_estimate.py:174-199; the reference's "sketch per site, merge
    centrally").
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _device, _lib


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


class RegisterExchange:
    """An NCCL communicator owned by the C ABI (gm_comm_init) for the ranks
    of `group`; torch.distributed carries only its unique id from rank 0.
    Exchanges run in place on (y float64 [k], s int64 [k] holding uint64
    ids) device tensors, on the current CUDA stream."""

    def __init__(self, group=None):
        L = _lib.load()
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        nbytes = L.gm_comm_id_bytes()
        uid = (ctypes.c_char * nbytes)()
        if self.rank == 0:
            _device.call("gm_comm_unique_id", ctypes.addressof(uid))
        box = [bytes(uid) if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (ctypes.c_char * nbytes).from_buffer_copy(box[0])
        self._comm = ctypes.c_void_p()
        _device.call("gm_comm_init", ctypes.addressof(uid), self.world, self.rank, ctypes.byref(self._comm))

    def allreduce_min(self, y: torch.Tensor, s: torch.Tensor):
        _device.call("gm_allreduce_min_registers", self._comm, y.data_ptr(), s.data_ptr(), y.numel(),
                     _device.stream_ptr())
        return y, s

    def allgather_merge(self, y: torch.Tensor, s: torch.Tensor):
        _device.call("gm_allgather_merge_registers", self._comm, y.data_ptr(), s.data_ptr(), y.numel(),
                     _device.stream_ptr())
        return y, s

    def close(self) -> None:
        if self._comm:
            _device.call("gm_comm_destroy", self._comm)
            self._comm = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
