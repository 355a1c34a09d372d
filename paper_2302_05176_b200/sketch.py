"""Sketch types and generators (reference sketch.py), backed by the CUDA
engine.

Types keep the reference's names, fields and validation (WeightedVector
sketch.py:40-115, GumbelMaxSketch :118-136, GenerationParams :139-157).
Generators run on the device:
  sketch_fast / sketch_fast_counted   -> gm_sketch_csr (K1), or
                                         gm_sketch_elements (K2) for vectors
                                         above LARGE_VECTOR elements
  sketch_naive / sketch_naive_counted -> the same kernels with every queue
                                         run to k (GM_FLAG_EXHAUSTIVE)
  sketch_csr / sketch_many            -> batched K1 over CSR arrays (new; the
                                         reference callers loop per vector)
Registers equal the reference's bit for bit, s and y: the device log is a
clone of glibc's (the reference's math.log; csrc/gm_glibc_log.cuh), so
GumbelMaxSketch equality holds against the reference's own sketches with no
host pass.  (exact_y_host, the host re-derivation of y from the winners, is
kept as a cross-check.)
The *_counted work counters count arrivals the device computed, which is
schedule-dependent and differs from the reference's FastSearch count.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import Iterator, Mapping, Sequence

import numpy as np
import torch

from . import _device, _lib
from .errors import (
    EmptyVectorError,
    IncompleteSketchError,
    InvalidParameterError,
    InvalidWeightError,
    MismatchedSketchError,
    MissingElementError,
)
from .randgen import MIN_WEIGHT, SeedScheme

SKETCH_FORMAT = "gmsketch/1"
LARGE_VECTOR = 1 << 20  # above this a single vector uses the grid-wide kernel
UINT64_MAX = (1 << 64) - 1


class WeightedVector:
    """Sparse map element index (>= 1) -> weight > 0 (sketch.py:40-115)."""

    __slots__ = ("_items", "_index", "_weight_sum", "_ids", "_w")

    def __init__(self, entries: Mapping[int, float]):
        items = []
        for element, weight in entries.items():
            element = int(element)
            if element < 1:
                raise InvalidWeightError(f"element indices must be >= 1, got {element}")
            weight = float(weight)
            if not math.isfinite(weight) or weight <= 0.0:
                raise InvalidWeightError(
                    f"element {element}: weight must be positive and finite, got {weight}")
            if weight < MIN_WEIGHT:
                raise InvalidWeightError(
                    f"element {element}: weight {weight} below minimum {MIN_WEIGHT}")
            items.append((element, weight))
        items.sort()
        self._items = tuple(items)
        self._index = dict(items)
        self._weight_sum = math.fsum(w for _, w in items)
        self._ids = None
        self._w = None

    @classmethod
    def from_arrays(cls, ids, weights) -> "WeightedVector":
        return cls(dict(zip((int(e) for e in ids), (float(w) for w in weights))))

    @property
    def n_plus(self) -> int:
        return len(self._items)

    @property
    def weight_sum(self) -> float:
        return self._weight_sum

    def items(self):
        return self._items

    def arrays(self) -> tuple[np.ndarray, np.ndarray]:
        """(ids uint64, weights float64) in ascending id order."""
        if self._ids is None:
            self._ids = np.array([e for e, _ in self._items], dtype=np.uint64)
            self._w = np.array([w for _, w in self._items], dtype=np.float64)
        return self._ids, self._w

    def get(self, element: int, default: float = 0.0) -> float:
        return self._index.get(element, default)

    def __getitem__(self, element: int) -> float:
        try:
            return self._index[element]
        except KeyError:
            raise MissingElementError(f"element {element} not in vector") from None

    def __contains__(self, element: int) -> bool:
        return element in self._index

    def __len__(self) -> int:
        return len(self._items)

    def __iter__(self) -> Iterator[int]:
        return iter(self._index)

    def __eq__(self, other) -> bool:
        if not isinstance(other, WeightedVector):
            return NotImplemented
        return self._items == other._items

    def __repr__(self) -> str:
        return f"WeightedVector(n_plus={self.n_plus}, weight_sum={self._weight_sum!r})"

    def as_dict(self) -> dict[int, float]:
        return dict(self._items)

    def scaled(self, factor: float) -> "WeightedVector":
        if not (factor > 0.0) or not math.isfinite(factor):
            raise InvalidWeightError(f"scale factor must be positive, got {factor}")
        return WeightedVector({e: w * factor for e, w in self._items})


@dataclass(frozen=True)
class GumbelMaxSketch:
    """k registers: winning element s[j] and value y[j] (sketch.py:118-136)."""

    k: int
    s: tuple
    y: tuple
    fingerprint: int

    def __post_init__(self):
        if len(self.s) != self.k or len(self.y) != self.k:
            raise InvalidParameterError(
                f"register arrays must have length k={self.k}, got {len(self.s)} and {len(self.y)}")


@dataclass(frozen=True)
class GenerationParams:
    """k and the search increment delta (sketch.py:139-157).  delta only
    shaped the reference's FastSearch schedule; the device schedule ignores
    it (output is schedule-independent)."""

    k: int
    scheme: SeedScheme
    delta: int | None = None

    def __post_init__(self):
        if self.k < 1:
            raise InvalidParameterError(f"k must be >= 1, got {self.k}")
        if self.delta is None:
            object.__setattr__(self, "delta", self.k)
        elif self.delta < 1:
            raise InvalidParameterError(f"delta must be >= 1, got {self.delta}")


def compute_ri(R: int, v: WeightedVector, element: int) -> int:
    """ceil(R * w / W) (sketch.py:160-169), the reference's release budget."""
    if R < 0:
        raise InvalidParameterError(f"R must be >= 0, got {R}")
    weight = v[element]
    return math.ceil(R * weight / v.weight_sum)


@dataclass
class SketchBatch:
    """n sketches as device tensors: y [n, k] float64, s [n, k] int64 holding
    uint64 element ids (two's complement view), emitted [n] int64 or None."""

    k: int
    y: torch.Tensor
    s: torch.Tensor
    fingerprint: int | None
    emitted: torch.Tensor | None = None
    fingerprints: list[int] | None = None  # per sketch (sketch_csr_seeded), else None

    def __len__(self) -> int:
        return self.y.shape[0]

    def to_sketches(self) -> list[GumbelMaxSketch]:
        y = self.y.cpu().numpy()
        s = self.s.cpu().numpy().view(np.uint64)
        fps = self.fingerprints or [self.fingerprint] * y.shape[0]
        return [GumbelMaxSketch(self.k, tuple(int(x) for x in s[i]), tuple(y[i].tolist()),
                                fps[i]) for i in range(y.shape[0])]


def _check_k(k: int) -> None:
    if k < 1:
        raise InvalidParameterError(f"k must be >= 1, got {k}")


def sketch_csr(ids, weights, offsets, k: int, scheme: SeedScheme, *, exhaustive: bool = False,
               counted: bool = False, asynchronous: bool = False,
               exact_y: bool = False) -> SketchBatch:
    """Sketch every CSR vector ids[offsets[v]:offsets[v+1]] on the device.

    ids: uint32/uint64 (or int32/int64 viewed as unsigned) tensor or array;
    weights: float32/float64; offsets: int64 [n_vec + 1].  Ids must be
    distinct within a vector (WeightedVector keys).  Device tensors are used
    in place; host arrays are copied in.
    ``exact_y=True`` re-derives y on the host with the reference's
    arithmetic (exact_y_host; a cross-check -- the device y is already
    bit-identical)."""
    _check_k(k)
    dev = _device.require_cuda()
    ids_t = ids if isinstance(ids, torch.Tensor) else torch.from_numpy(_as_id_np(ids))
    w_t = weights if isinstance(weights, torch.Tensor) else torch.from_numpy(_device.weight_array(weights)[0])
    off_t = offsets if isinstance(offsets, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(offsets, dtype=np.int64)))
    ids_t = ids_t.to(dev).contiguous()
    w_t = w_t.to(dev).contiguous()
    off_t = off_t.to(dev, dtype=torch.int64).contiguous()
    n_vec = off_t.numel() - 1
    y = torch.empty((n_vec, k), dtype=torch.float64, device=dev)
    s = torch.empty((n_vec, k), dtype=torch.int64, device=dev)
    em = torch.empty(n_vec, dtype=torch.int64, device=dev) if counted else None
    flags = (_lib.GM_FLAG_EXHAUSTIVE if exhaustive else 0) | (_lib.GM_FLAG_ASYNC if asynchronous else 0)
    _device.call("gm_sketch_csr", ids_t.data_ptr(), _device.id_bits_of(ids_t), w_t.data_ptr(),
                 _device.w_bits_of(w_t), off_t.data_ptr(), n_vec, k, scheme.global_seed,
                 scheme.stream_salt, flags, y.data_ptr(), s.data_ptr(), _device.ptr(em),
                 _device.stream_ptr())
    if exact_y:
        y_h = y.cpu()
        exact_y_host(ids_t.cpu(), w_t.cpu(), off_t.cpu(), k, scheme, s.cpu(), y_h)
        y.copy_(y_h)
    return SketchBatch(k, y, s, scheme.fingerprint, em)


def sketch_vector_seeds(ids, weights, k: int, schemes: Sequence[SeedScheme], *, exhaustive: bool = False,
                        counted: bool = False) -> SketchBatch:
    """R sketches of ONE vector, one per SeedScheme, in one launch
    (gm_sketch_csr_seeded + GM_FLAG_ONE_VECTOR: the vector is stored once).
    Row r equals sketch_csr of the vector under schemes[r]."""
    n = len(ids)
    return sketch_csr_seeded(ids, weights, np.array([0, n], np.int64), k, schemes, exhaustive=exhaustive,
                             counted=counted, one_vector=True)


def sketch_csr_seeded(ids, weights, offsets, k: int, schemes: Sequence[SeedScheme], *,
                      exhaustive: bool = False, counted: bool = False, one_vector: bool = False) -> SketchBatch:
    """sketch_csr with one SeedScheme per vector (gm_sketch_csr_seeded).  All
    schemes must share the stream salt (the permutation seed is
    global_seed ^ salt, randgen.py:72-95).  ``one_vector``: offsets is
    [lo, hi] of a single vector and len(schemes) sketches of it are made."""
    _check_k(k)
    dev = _device.require_cuda()
    salts = {sc.stream_salt for sc in schemes}
    if len(salts) != 1:
        raise InvalidParameterError("sketch_csr_seeded: every scheme must have the same stream salt")
    ids_t = ids if isinstance(ids, torch.Tensor) else torch.from_numpy(_as_id_np(ids))
    w_t = weights if isinstance(weights, torch.Tensor) else torch.from_numpy(_device.weight_array(weights)[0])
    off_t = offsets if isinstance(offsets, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(offsets, dtype=np.int64)))
    ids_t, w_t = ids_t.to(dev).contiguous(), w_t.to(dev).contiguous()
    off_t = off_t.to(dev, dtype=torch.int64).contiguous()
    n_vec = len(schemes) if one_vector else off_t.numel() - 1
    if one_vector and off_t.numel() != 2:
        raise InvalidParameterError("one_vector: offsets must be [lo, hi]")
    if len(schemes) != n_vec:
        raise InvalidParameterError(f"{len(schemes)} schemes for {n_vec} vectors")
    seeds = torch.from_numpy(np.array([sc.global_seed for sc in schemes], dtype=np.uint64).view(np.int64)).to(dev)
    y = torch.empty((n_vec, k), dtype=torch.float64, device=dev)
    s = torch.empty((n_vec, k), dtype=torch.int64, device=dev)
    em = torch.empty(n_vec, dtype=torch.int64, device=dev) if counted else None
    _device.call("gm_sketch_csr_seeded", ids_t.data_ptr(), _device.id_bits_of(ids_t), w_t.data_ptr(),
                 _device.w_bits_of(w_t), off_t.data_ptr(), n_vec, k, seeds.data_ptr(), salts.pop(),
                 (_lib.GM_FLAG_EXHAUSTIVE if exhaustive else 0) | (_lib.GM_FLAG_ONE_VECTOR if one_vector else 0),
                 y.data_ptr(), s.data_ptr(), _device.ptr(em),
                 _device.stream_ptr())
    return SketchBatch(k, y, s, None, em, [sc.fingerprint for sc in schemes])


def sketch_csr_host(ids, weights, offsets, k: int, scheme: SeedScheme, *, out=None,
                    counted: bool = False, exhaustive: bool = False, exact_y: bool = False, s32: bool = False):
    """Host-buffer batch: ``sketch_csr`` for CPU-resident CSR arrays, through
    gm_sketch_csr_host (input copies pipelined with the sketch; results
    stored straight into page-locked outputs).  ``out=(y, s)`` supplies
    output arrays or CPU tensors (float64 / uint64-or-int64, shape
    [n_vec, k]); pin them for the zero-copy store.  Returns (y, s, emitted
    or None) as given/allocated (numpy when allocated here).  ``exact_y``:
    see sketch_csr.  ``s32`` (32-bit ids only): s comes back as uint32
    (GM_FLAG_S32; 12 instead of 16 bytes per register over the bus)."""
    _check_k(k)
    _device.require_cuda()

    def host(a, dt):
        if isinstance(a, torch.Tensor):
            assert a.device.type == "cpu" and a.is_contiguous(), "host tensors must be contiguous CPU tensors"
            return a, a.data_ptr()
        a = np.ascontiguousarray(a, dtype=dt) if dt is not None else np.ascontiguousarray(a)
        return a, a.ctypes.data

    if isinstance(ids, torch.Tensor):
        id_bits = _device.id_bits_of(ids)
        ids_h, ip = host(ids, None)
    else:
        a, id_bits = _device.id_array(ids)
        ids_h, ip = host(a, None)
    if isinstance(weights, torch.Tensor):
        w_bits = _device.w_bits_of(weights)
        w_h, wp = host(weights, None)
    else:
        a, w_bits = _device.weight_array(weights)
        w_h, wp = host(a, None)
    off_h, op = host(offsets, None) if isinstance(offsets, torch.Tensor) else host(offsets, np.int64)
    n_vec = int(off_h.shape[0]) - 1
    if out is None:
        y, s = np.empty((n_vec, k), np.float64), np.empty((n_vec, k), np.uint32 if s32 else np.uint64)
    else:
        y, s = out
    _, yp = host(y, None)
    _, sp = host(s, None)
    em = np.zeros(max(n_vec, 1), np.int64) if counted else None
    flags = (_lib.GM_FLAG_EXHAUSTIVE if exhaustive else 0) | (_lib.GM_FLAG_S32 if s32 else 0)
    _device.call("gm_sketch_csr_host", ip, id_bits, wp, w_bits, op, n_vec, k, scheme.global_seed,
                 scheme.stream_salt, flags, yp, sp, em.ctypes.data if em is not None else None,
                 _device.stream_ptr())
    if exact_y:
        s64 = (s.numpy() if isinstance(s, torch.Tensor) else s).astype(np.uint64) if s32 else s
        exact_y_host(ids_h, w_h, off_h, k, scheme, s64, y)
    return y, s, (em[:n_vec] if em is not None else None)


def exact_y_host(ids, weights, offsets, k: int, scheme: SeedScheme, s, y, threads: int = 0):
    """Re-derive registers' values with the reference's arithmetic (glibc log,
    randgen.py:158-207) from their winning elements, in place (gm_exact_y;
    host arrays, no device work).  A cross-check of the device registers,
    which already carry these bits; no generator calls it.  s: uint64/int64 [n_vec, k] (or [k]), y: float64 of the same
    shape; CPU tensors or numpy arrays."""
    def np_of(a):
        return a.numpy() if isinstance(a, torch.Tensor) else a

    a_ids, id_bits = _device.id_array(np_of(ids).view(np.uint32) if np_of(ids).dtype == np.int32 else np_of(ids))
    a_w, w_bits = _device.weight_array(np_of(weights))
    off = np.ascontiguousarray(np.asarray(np_of(offsets), dtype=np.int64))
    s_np = np.ascontiguousarray(np_of(s)).view(np.uint64)
    y_np = np_of(y)
    assert y_np.dtype == np.float64 and y_np.flags.c_contiguous, "y must be a contiguous float64 array"
    assert s_np.size == y_np.size == (off.size - 1) * k, "s, y must hold k registers per vector"
    rc = _lib.load().gm_exact_y(a_ids.ctypes.data, id_bits, a_w.ctypes.data, w_bits, off.ctypes.data,
                                off.size - 1, k, scheme.global_seed, scheme.stream_salt, s_np.ctypes.data,
                                y_np.ctypes.data, threads)
    if rc == _lib.GM_ERR_MISMATCHED:
        raise MismatchedSketchError("a register names an element that is not in its vector")
    if rc:
        raise InvalidParameterError(f"gm_exact_y failed with code {rc}")
    return y


def sketch_csr_host_many(batches, k: int, scheme: SeedScheme, *, streams: int = 6, s32: bool = False):
    """A stream of host-buffer CSR batches (the serving loop): yields (y, s)
    per batch, in order, with batches issued over ``streams`` CUDA streams so
    one batch's copies and first CTAs overlap the previous batches' kernels
    (GM_FLAG_ASYNC).  ``batches`` yields (ids, weights,
    offsets) numpy arrays or CPU tensors (u32/u64 ids, f32/f64 weights;
    page-locked tensors are used in place, anything else is copied into a
    reused page-locked staging buffer per stream); each result is a pair of
    page-locked CPU tensors that stay valid while ``streams`` more results
    are taken from the generator (copy them to keep them longer)."""
    _check_k(k)
    dev = _device.require_cuda()
    pool = _device.stream_pool(dev, max(1, streams))
    inflight = []  # (stream index, y, s, keep-alive inputs)
    outs = {}  # output set -> page-locked (y, s) flat buffers, grown when a batch needs more

    staging = {}  # per stream: page-locked input buffers, reused (grown when needed)

    def pinned(j, name, a):
        t = torch.from_numpy(a) if isinstance(a, np.ndarray) else a
        if t.is_pinned():
            return t
        buf = staging.get((j, name))
        if buf is None or buf.numel() < t.numel() or buf.dtype != t.dtype:
            buf = torch.empty(max(t.numel(), 1), dtype=t.dtype).pin_memory()
            staging[(j, name)] = buf
        view = buf[: t.numel()]
        view.copy_(t.reshape(-1))
        return view

    def issue(i, b):
        ids, w, off = b
        j = i % len(pool)
        if isinstance(ids, torch.Tensor):
            id_bits, t_ids = _device.id_bits_of(ids), ids
        else:
            a_ids, id_bits = _device.id_array(ids)
            t_ids = a_ids.view(np.int32 if id_bits == 32 else np.int64)
        if isinstance(w, torch.Tensor):
            w_bits, t_w = _device.w_bits_of(w), w
        else:
            t_w, w_bits = _device.weight_array(w)
        t_off = off if isinstance(off, torch.Tensor) else np.ascontiguousarray(np.asarray(off, dtype=np.int64))
        t_ids, t_w, t_off = pinned(j, "ids", t_ids), pinned(j, "w", t_w), pinned(j, "off", t_off)
        n_vec = t_off.numel() - 1
        key = i % (2 * len(pool))  # two output sets per stream: a result outlives `streams` more yields
        yb, sb = outs.get(key, (None, None))
        if yb is None or yb.numel() < n_vec * k:
            yb = torch.empty(max(n_vec * k, 1), dtype=torch.float64).pin_memory()
            sb = torch.empty(max(n_vec * k, 1), dtype=torch.int32 if s32 else torch.int64).pin_memory()
            outs[key] = (yb, sb)
        y, s = yb[: n_vec * k].view(n_vec, k), sb[: n_vec * k].view(n_vec, k)
        flags = _lib.GM_FLAG_ASYNC | (_lib.GM_FLAG_S32 if s32 else 0)
        _device.call("gm_sketch_csr_host", t_ids.data_ptr(), id_bits, t_w.data_ptr(), w_bits, t_off.data_ptr(), n_vec,
                     k, scheme.global_seed, scheme.stream_salt, flags, y.data_ptr(), s.data_ptr(), None,
                     pool[j].cuda_stream)
        inflight.append((j, y, s, (t_ids, t_w, t_off)))

    def retire():
        j, y, s, _ = inflight.pop(0)
        pool[j].synchronize()
        _device.call("gm_stream_status", pool[j].cuda_stream)
        return y, s

    for i, b in enumerate(batches):
        if len(inflight) == len(pool):
            yield retire()
        issue(i, b)
    while inflight:
        yield retire()


def _as_id_np(ids) -> np.ndarray:
    a, bits = _device.id_array(ids)
    return a.view(np.int32 if bits == 32 else np.int64)


def sketch_elements(ids, weights, k: int, scheme: SeedScheme, *, exhaustive: bool = False,
                    into: tuple[torch.Tensor, torch.Tensor] | None = None):
    """One sketch over a large element set on the device (grid-wide kernel).
    Ids may repeat only with identical weights.  With ``into=(y, s)`` the
    elements are folded into an existing device sketch.  Returns
    (y [k] float64, s [k] int64 view of uint64, emitted)."""
    _check_k(k)
    dev = _device.require_cuda()
    ids_t = ids if isinstance(ids, torch.Tensor) else torch.from_numpy(_as_id_np(ids))
    w_t = weights if isinstance(weights, torch.Tensor) else torch.from_numpy(_device.weight_array(weights)[0])
    ids_t = ids_t.to(dev).contiguous()
    w_t = w_t.to(dev).contiguous()
    flags = _lib.GM_FLAG_EXHAUSTIVE if exhaustive else 0
    if into is not None:
        y, s = into
        flags |= _lib.GM_FLAG_ACCUMULATE
    else:
        y = torch.empty(k, dtype=torch.float64, device=dev)
        s = torch.empty(k, dtype=torch.int64, device=dev)
    em = np.zeros(1, dtype=np.int64)
    _device.call("gm_sketch_elements", ids_t.data_ptr(), _device.id_bits_of(ids_t), w_t.data_ptr(),
                 _device.w_bits_of(w_t), ids_t.numel(), k, scheme.global_seed, scheme.stream_salt,
                 flags, y.data_ptr(), s.data_ptr(), em.ctypes.data, _device.stream_ptr())
    return y, s, int(em[0])


def sketch_elements_many(sets, k: int, scheme: SeedScheme):
    """One sketch per (ids, weights) element set, enqueued back to back on the
    current stream without host synchronisation between them
    (gm_sketch_elements_async: one pass at the list bound each); one
    synchronisation at the end reads the unset-register counts, and a sketch
    that needs it is finished with the synchronous call (GM_FLAG_ACCUMULATE).
    Returns [(y [k] float64, s [k] int64 view of uint64)] in order, equal to
    sketch_elements per set."""
    _check_k(k)
    dev = _device.require_cuda()
    sets = [(ids if isinstance(ids, torch.Tensor) else torch.from_numpy(_as_id_np(ids)),
             w if isinstance(w, torch.Tensor) else torch.from_numpy(_device.weight_array(w)[0])) for ids, w in sets]
    sets = [(i.to(dev).contiguous(), w.to(dev).contiguous()) for i, w in sets]
    out = [(torch.empty(k, dtype=torch.float64, device=dev), torch.empty(k, dtype=torch.int64, device=dev))
           for _ in sets]
    unset = torch.zeros(max(1, len(sets)), dtype=torch.int32, device=dev)
    sp = _device.stream_ptr()
    for j, ((i, w), (y, s)) in enumerate(zip(sets, out)):
        if i.numel() == 0:
            raise IncompleteSketchError([])
        _device.call("gm_sketch_elements_async", i.data_ptr(), _device.id_bits_of(i), w.data_ptr(),
                     _device.w_bits_of(w), i.numel(), k, scheme.global_seed, scheme.stream_salt, 0,
                     y.data_ptr(), s.data_ptr(), unset[j].data_ptr(), sp)
    counts = unset.cpu().numpy()  # the one synchronisation
    _device.call("gm_stream_status", sp)
    for j, ((i, w), (y, s)) in enumerate(zip(sets, out)):
        if counts[j] > 0:
            sketch_elements(i, w, k, scheme, into=(y, s))
    return out


def _to_sketch(k, y: np.ndarray, s: np.ndarray, fp: int) -> GumbelMaxSketch:
    return GumbelMaxSketch(k, tuple(int(x) for x in s.view(np.uint64)), tuple(y.tolist()), fp)


def _sketch_vector(v: WeightedVector, params: GenerationParams, exhaustive: bool):
    if v.n_plus == 0:
        raise EmptyVectorError("cannot sketch a vector with no positive entries")
    ids, w = v.arrays()
    k = params.k
    off = np.array([0, ids.size], dtype=np.int64)
    if v.n_plus > LARGE_VECTOR:
        y, s, em = sketch_elements(ids, w, k, params.scheme, exhaustive=exhaustive)
        return _to_sketch(k, y.cpu().numpy(), s.cpu().numpy(), params.scheme.fingerprint), em
    _device.require_cuda()
    bits = 32 if (ids.size and int(ids.max()) < (1 << 32)) else 64
    ids_h = ids.astype(np.uint32) if bits == 32 else ids
    y = np.empty(k, np.float64)
    s = np.empty(k, np.uint64)
    em = np.zeros(1, np.int64)
    flags = _lib.GM_FLAG_EXHAUSTIVE if exhaustive else 0
    _device.call("gm_sketch_csr_host", ids_h.ctypes.data, bits, w.ctypes.data, 64, off.ctypes.data, 1,
                 k, params.scheme.global_seed, params.scheme.stream_salt, flags, y.ctypes.data,
                 s.ctypes.data, em.ctypes.data, _device.stream_ptr())
    return _to_sketch(k, y, s, params.scheme.fingerprint), int(em[0])


def sketch_naive(v: WeightedVector, params: GenerationParams) -> GumbelMaxSketch:
    """Exhaustive generator: every queue run to k (sketch.py:177-180)."""
    return sketch_naive_counted(v, params)[0]


def sketch_naive_counted(v: WeightedVector, params: GenerationParams):
    """(sketch, emitted) with emitted = n_plus * k (sketch.py:183-209)."""
    return _sketch_vector(v, params, exhaustive=True)


def sketch_fast(v: WeightedVector, params: GenerationParams) -> GumbelMaxSketch:
    """Pruned generator; equal to sketch_naive (sketch.py:212-215)."""
    return sketch_fast_counted(v, params)[0]


def sketch_fast_counted(v: WeightedVector, params: GenerationParams):
    """(sketch, arrivals computed on the device) (sketch.py:218-311)."""
    return _sketch_vector(v, params, exhaustive=False)


def sketch_many(vectors: Sequence[WeightedVector], params: GenerationParams,
                exact_y: bool = False) -> list[GumbelMaxSketch]:
    """Sketch a list of vectors in one batched launch (``exact_y``: see
    sketch_csr)."""
    if not vectors:
        return []
    for v in vectors:
        if v.n_plus == 0:
            raise EmptyVectorError("cannot sketch a vector with no positive entries")
    ids = np.concatenate([v.arrays()[0] for v in vectors])
    w = np.concatenate([v.arrays()[1] for v in vectors])
    off = np.zeros(len(vectors) + 1, dtype=np.int64)
    off[1:] = np.cumsum([v.n_plus for v in vectors])
    return sketch_csr(ids, w, off, params.k, params.scheme, exact_y=exact_y).to_sketches()


def check_compatible(a: GumbelMaxSketch, b: GumbelMaxSketch) -> None:
    """sketch.py:314-322"""
    if a.k != b.k:
        raise MismatchedSketchError(f"register counts differ: {a.k} != {b.k}")
    if a.fingerprint != b.fingerprint:
        raise MismatchedSketchError(
            f"seed-scheme fingerprints differ: {a.fingerprint:#018x} != {b.fingerprint:#018x}")


def sketch_to_json(sk: GumbelMaxSketch) -> str:
    """Versioned record with hex-float registers (sketch.py:325-339)."""
    record = {"format": SKETCH_FORMAT, "k": sk.k, "fingerprint": f"{sk.fingerprint:#018x}",
              "s": list(sk.s), "y": [float(value).hex() for value in sk.y]}
    return json.dumps(record, separators=(",", ":"))


def sketch_from_json(text: str) -> GumbelMaxSketch:
    """sketch.py:342-357"""
    try:
        record = json.loads(text)
    except json.JSONDecodeError as exc:
        raise MismatchedSketchError(f"not a sketch record: {exc}") from exc
    if not isinstance(record, dict) or record.get("format") != SKETCH_FORMAT:
        raise MismatchedSketchError(
            f"unsupported sketch format {record.get('format') if isinstance(record, dict) else None!r}; "
            f"expected {SKETCH_FORMAT!r}")
    k = int(record["k"])
    s = tuple(int(e) for e in record["s"])
    y = tuple(float.fromhex(value) for value in record["y"])
    return GumbelMaxSketch(k, s, y, int(record["fingerprint"], 16))
