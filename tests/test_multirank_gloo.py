"""world_size-2 gloo runs of the multi-GPU host logic on CPU.

Per-rank sketches come from the CPU oracle (this container has no GPU);
what is under test is the sharding (paper_2302_05176_b200/shard.py:
contiguous element shards, element-balanced vector ranges) and the two
register-exchange protocols the C ABI runs over NCCL
(csrc/gm_comm.cuh: gm_allreduce_min_registers, gm_allgather_merge_registers),
restated here with torch.distributed collectives over gloo -- all-reduce MIN
of y, then MIN of the ids of the ranks holding the minimum; all-gather and
the rank-order merge -- both reproducing the whole-stream sketch (partition
law, test_estimate.py:174-199).  The NCCL build of the same protocol runs
on the GPU (tests/test_gpu_parity.py::test_nccl_exchange_world1).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2302_05176_b200 import shard, workloads

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


_SIGN = 1 << 63


def model_allreduce_min(y: torch.Tensor, s: torch.Tensor):
    """gm_allreduce_min_registers' protocol: MIN of y; ids of the ranks that
    hold the minimum (UINT64_MAX elsewhere); MIN of those ids.  Unsigned ids
    ride in int64 with the sign bit flipped so signed MIN orders them."""
    ym = y.clone()
    dist.all_reduce(ym, op=dist.ReduceOp.MIN)
    sign = torch.tensor(-_SIGN, dtype=torch.int64)
    key = torch.where(y == ym, s ^ sign, torch.full_like(s, _SIGN - 1))
    dist.all_reduce(key, op=dist.ReduceOp.MIN)
    return ym, key ^ sign


def model_allgather_merge(y: torch.Tensor, s: torch.Tensor):
    """gm_allgather_merge_registers' protocol: all-gather, merge in rank order."""
    world = dist.get_world_size()
    ys = [torch.empty_like(y) for _ in range(world)]
    ss = [torch.empty_like(s) for _ in range(world)]
    dist.all_gather(ys, y)
    dist.all_gather(ss, s)
    return O.merge(torch.stack(ys).numpy(), torch.stack(ss).numpy().view(np.uint64))


def _stream_worker(rank, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    ids, w, k, seed = workloads.config4(n_pairs=200_000, n_keys=50_000)
    k = 256
    lo, hi = shard.element_range(ids.size, WORLD, rank)
    rc, y, s, _, _ = O.sketch_stream(ids[lo:hi], w[lo:hi].astype(np.float64), k, seed)
    assert rc == 0
    ym, sm = model_allgather_merge(torch.from_numpy(y), torch.from_numpy(s.view(np.int64)))
    yr, sr = model_allreduce_min(torch.from_numpy(y.copy()), torch.from_numpy(s.view(np.int64).copy()))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), y=ym, s=sm, yr=yr.numpy(), sr=sr.numpy().view(np.uint64))
    dist.destroy_process_group()


def _csr_worker(rank, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    ids, w, off, k, seed = workloads.config3(n_vectors=300)
    v0, v1 = shard.vector_ranges(off, WORLD)[rank]
    lo, hi = off[v0], off[v1]
    rc, y, s, _ = O.sketch_csr(ids[lo:hi].astype(np.uint64), w[lo:hi].astype(np.float64), off[v0:v1 + 1] - lo,
                               k, seed, mode=0)
    assert rc == 0
    # no data-path collective: only the element count is all-reduced for the report
    n = torch.tensor([int(hi - lo)], dtype=torch.int64)
    dist.all_reduce(n)
    np.savez(os.path.join(out_dir, f"csr{rank}.npz"), y=y, s=s, n=n.numpy(), v0=v0, v1=v1)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_stream_shards_merge_to_whole(tmp_path):
    mp.spawn(_stream_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    ids, w, _, seed = workloads.config4(n_pairs=200_000, n_keys=50_000)
    rc, yw, sw, _, _ = O.sketch_stream(ids, w.astype(np.float64), 256, seed)
    assert rc == 0
    for r in range(WORLD):
        d = np.load(tmp_path / f"rank{r}.npz")
        assert np.array_equal(d["s"], sw)
        assert d["y"].tolist() == yw.tolist()
        # the MIN all-reduce variant gives the same registers
        assert np.array_equal(d["sr"], sw)
        assert d["yr"].tolist() == yw.tolist()


@pytest.mark.timeout(300)
def test_vector_shards_cover_batch(tmp_path):
    mp.spawn(_csr_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    ids, w, off, k, seed = workloads.config3(n_vectors=300)
    rc, yw, sw, _ = O.sketch_csr(ids.astype(np.uint64), w.astype(np.float64), off, k, seed, mode=0)
    parts = [np.load(tmp_path / f"csr{r}.npz") for r in range(WORLD)]
    assert int(parts[0]["n"][0]) == int(off[-1])
    y = np.concatenate([p["y"] for p in parts])
    s = np.concatenate([p["s"] for p in parts])
    assert np.array_equal(s, sw) and y.tolist() == yw.tolist()


def _minreduce_worker(rank, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    # hand-made registers: ids above 2**63 (negative as int64), exact y ties
    # between ranks (smaller id wins), unset registers (inf, id 2**64-1)
    inf = float("inf")
    y = [[1.0, 2.0, inf, 3.0, 5.0], [1.0, 1.5, inf, 3.0, inf]][rank]
    s = [[(1 << 64) - 2, 7, (1 << 64) - 1, (1 << 63) + 5, 9], [(1 << 63), 8, (1 << 64) - 1, (1 << 63) + 4, (1 << 64) - 1]][rank]
    yr, sr = model_allreduce_min(torch.tensor(y, dtype=torch.float64),
                                 torch.from_numpy(np.array(s, dtype=np.uint64).view(np.int64)))
    np.savez(os.path.join(out_dir, f"mr{rank}.npz"), y=yr.numpy(), s=sr.numpy().view(np.uint64))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_allreduce_min_unsigned_ids_and_ties(tmp_path):
    mp.spawn(_minreduce_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    for r in range(WORLD):
        d = np.load(tmp_path / f"mr{r}.npz")
        assert d["y"].tolist() == [1.0, 1.5, float("inf"), 3.0, 5.0]
        assert d["s"].tolist() == [1 << 63, 8, (1 << 64) - 1, (1 << 63) + 4, 9]
