"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference measures on no public dataset; these generators stand in for
the configs named in BASELINE.json (SURVEY.md section 8(d) fixes the
distributions, seeds and id layouts; choices marked there with a dagger are
the survey's, not BASELINE.json's).  All generators are numpy-seeded and
deterministic, return host arrays in the device layouts the C-ABI takes
(ids u32 or u64, weights f32 or f64, CSR offsets i64), and never touch
/root/reference.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

K_ELEM = 0x9E3779B97F4A7C15
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def mix64_np(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finalizer (randgen.py:64-69) over uint64."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = (x ^ (x >> np.uint64(30))) * M1
        x = (x ^ (x >> np.uint64(27))) * M2
        return x ^ (x >> np.uint64(31))


def config1():
    """Config 1: one dense vector, ids 0..9999, fp64 weights Uniform(0,1]
    (= 1 - default_rng(1).random), k=256, seed 1.  Returns (ids u32, w f64, k, seed)."""
    n = 10_000
    ids = np.arange(n, dtype=np.uint32)
    w = 1.0 - np.random.default_rng(1).random(n)
    return ids, w, 256, 1


def config2(n_vectors: int = 1000):
    """Config 2: vectors paired (2i, 2i+1).  A: 1000 distinct ids uniform
    without replacement from [1, 10**6]; B: A's first 500 ids with identical
    weights plus 500 fresh ids not in A.  Weights fp32 Exponential(1) with
    zeros resampled; k=1024; seed 1.  Returns (ids u32, w f32, offsets i64, k, seed)."""
    rng = np.random.default_rng(2)
    n_pairs = (n_vectors + 1) // 2
    ids_out, w_out = [], []
    for _ in range(n_pairs):
        pool = rng.choice(10**6, size=1500, replace=False).astype(np.uint32) + 1
        wt = rng.standard_exponential(1500, dtype=np.float32)
        while np.any(wt == 0):
            z = wt == 0
            wt[z] = rng.standard_exponential(int(z.sum()), dtype=np.float32)
        ids_out.append(pool[:1000])
        w_out.append(wt[:1000])
        ids_out.append(np.concatenate([pool[:500], pool[1000:]]))
        w_out.append(np.concatenate([wt[:500], wt[1000:]]))
    ids_out, w_out = ids_out[:n_vectors], w_out[:n_vectors]
    offsets = np.zeros(n_vectors + 1, dtype=np.int64)
    offsets[1:] = np.cumsum([a.size for a in ids_out])
    return np.concatenate(ids_out), np.concatenate(w_out), offsets, 1024, 1


def config3(n_vectors: int = 100_000):
    """Config 3: CSR vectors over dimension 2**32; n_i = clip(round(LogNormal(6,1)),
    1, 50000); ids distinct per vector, uniform in [1, 2**32); weights fp32
    classical Pareto(alpha=1.5, x_m=1) = 1 + rng.pareto(1.5); k=512; seed 1.
    Returns (ids u32, w f32, offsets i64, k, seed)."""
    rng = np.random.default_rng(3)
    sizes = np.clip(np.rint(rng.lognormal(6.0, 1.0, n_vectors)), 1, 50_000).astype(np.int64)
    offsets = np.zeros(n_vectors + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(sizes)
    total = int(offsets[-1])
    ids = rng.integers(1, 1 << 32, size=total, dtype=np.uint64)
    vec = np.repeat(np.arange(n_vectors, dtype=np.uint64), sizes)
    while True:  # make ids distinct within each vector
        key = (vec << np.uint64(32)) | ids
        order = np.argsort(key, kind="stable")
        ks = key[order]
        dup = np.zeros(total, dtype=bool)
        dup[order[1:][ks[1:] == ks[:-1]]] = True
        nd = int(dup.sum())
        if nd == 0:
            break
        ids[dup] = rng.integers(1, 1 << 32, size=nd, dtype=np.uint64)
    w = (1.0 + rng.pareto(1.5, size=total)).astype(np.float32)
    return ids.astype(np.uint32), w, offsets, 512, 1


def _parallel(fn, items) -> None:
    items = list(items)
    if len(items) <= 1:
        for c in items:
            fn(c)
        return
    with ThreadPoolExecutor(min(len(items), os.cpu_count() or 1)) as ex:
        list(ex.map(fn, items))


PAIR_CHUNK = 1 << 22   # config 4: pairs per keyed chunk
ELEM_CHUNK = 1 << 26   # config 5: elements per keyed chunk


def _config4_chunk(c: int, size: int, n_keys: int) -> np.ndarray:
    """Zipf(1.1) ranks <= n_keys (truncated by rejection) of pair chunk c,
    from its own generator default_rng([4, c]): any range of the stream can
    be generated alone (a rank of an N-GPU job makes only its shard)."""
    rng = np.random.default_rng([4, c])
    out = np.empty(size, dtype=np.int64)
    filled = 0
    while filled < size:
        need = size - filled
        draw = rng.zipf(1.1, size=int(need * 1.45) + 1024)
        draw = draw[draw <= n_keys][:need]
        out[filled:filled + draw.size] = draw
        filled += draw.size
    return out


def config4(n_pairs: int = 10**8, n_keys: int = 10**7, lo: int = 0, hi: int | None = None):
    """Config 4: weighted-cardinality stream of (u64 id, f32 weight) pairs.
    10**7 key weights fp32 U(0.1, 10) (default_rng(4)); ranks ~ Zipf(1.1)
    truncated to <= n_keys by rejection, drawn in keyed chunks of PAIR_CHUNK
    pairs (default_rng([4, chunk])); id = mix64(rank); stream order = draw
    order; k=4096; seed 1.  ``lo:hi`` selects a contiguous range of the
    stream (generated alone).  Returns (ids u64, w f32, k, seed)."""
    hi = n_pairs if hi is None else min(hi, n_pairs)
    lo = max(0, min(lo, hi))
    key_w = np.random.default_rng(4).uniform(0.1, 10.0, size=n_keys).astype(np.float32)
    ranks = np.empty(hi - lo, dtype=np.int64)

    def fill(c):  # chunks are independent: generated on all host threads
        c0 = c * PAIR_CHUNK
        c1 = min(c0 + PAIR_CHUNK, n_pairs)
        r = _config4_chunk(c, c1 - c0, n_keys)
        a, b = max(lo, c0), min(hi, c1)
        ranks[a - lo:b - lo] = r[a - c0:b - c0]

    _parallel(fill, range(lo // PAIR_CHUNK, (hi + PAIR_CHUNK - 1) // PAIR_CHUNK))
    ids = mix64_np(ranks.astype(np.uint64))
    return ids, key_w[ranks - 1], 4096, 1


def config5(n: int = 10**9, lo: int = 0, hi: int | None = None):
    """Config 5: one huge vector, ids 0..n-1 (u32), weights fp32
    LogNormal(0, 2), drawn in keyed chunks of ELEM_CHUNK elements
    (default_rng([5, chunk])); k=8192; seed 1.  ``lo:hi`` selects a
    contiguous element range (generated alone).  Returns (ids u32, w f32,
    k, seed)."""
    hi = n if hi is None else min(hi, n)
    lo = max(0, min(lo, hi))
    w = np.empty(hi - lo, dtype=np.float32)

    def fill(c):
        c0 = c * ELEM_CHUNK
        c1 = min(c0 + ELEM_CHUNK, n)
        a, b = max(lo, c0), min(hi, c1)
        rng = np.random.default_rng([5, c])
        if a > c0:
            rng.lognormal(0.0, 2.0, a - c0)  # advance to a (same stream as the whole chunk)
        w[a - lo:b - lo] = rng.lognormal(0.0, 2.0, b - a)

    _parallel(fill, range(lo // ELEM_CHUNK, (hi + ELEM_CHUNK - 1) // ELEM_CHUNK))
    ids = np.arange(lo, hi, dtype=np.uint32)
    return ids, w, 8192, 1
