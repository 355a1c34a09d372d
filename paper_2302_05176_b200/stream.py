"""Streaming construction (reference stream.py), device-backed.

StreamSketchState keeps the k registers on the device.  stream_update does
the reference's per-item checks on the host (weight validation, the
id -> weight dict that raises InconsistentWeightError, duplicate skipping;
stream.py:58-78) and buffers new items; buffered items are folded into the
device registers by the grid-wide kernel (gm_sketch_elements with
GM_FLAG_ACCUMULATE) when the buffer fills or when state is observed.
Because the registers are a per-register minimum, the result equals the
reference's one-item-at-a-time walk (stream order only changes work,
stream.py:1-12); exact ties go to the smaller id (measure zero).
"""

from __future__ import annotations

import math
from typing import Iterable, TextIO

import numpy as np
import torch

from . import _device
from .errors import IncompleteSketchError, InconsistentWeightError, InvalidParameterError, InvalidWeightError
from .randgen import MIN_WEIGHT, SeedScheme
from .sketch import GumbelMaxSketch, exact_y_host, sketch_elements

StreamItem = tuple[int, float]
_MASK64 = (1 << 64) - 1
FLUSH_ITEMS = 1 << 16


class StreamSketchState:
    """Mutable per-stream sketch under construction (stream.py:30-55)."""

    def __init__(self, k: int, scheme: SeedScheme, skip_duplicates: bool = True):
        if k < 1:
            raise InvalidParameterError(f"k must be >= 1, got {k}")
        self.k = k
        self.scheme = scheme
        self.skip_duplicates = skip_duplicates
        self.weights: dict[int, float] = {}
        self.emitted = 0
        self.last_item_emitted = 0
        self._pending_ids: list[int] = []
        self._pending_w: list[float] = []
        self._alias: dict[int, int] = {}  # u64 key -> original id when id not in [0, 2**64)
        dev = _device.require_cuda()
        self._y = torch.full((k,), math.inf, dtype=torch.float64, device=dev)
        self._s = torch.full((k,), -1, dtype=torch.int64, device=dev)
        self._unset = k

    def _flush(self) -> None:
        if not self._pending_ids:
            return
        ids = np.array([e & _MASK64 for e in self._pending_ids], dtype=np.uint64)
        w = np.array(self._pending_w, dtype=np.float64)
        self._pending_ids, self._pending_w = [], []
        try:
            _, _, em = sketch_elements(ids, w, self.k, self.scheme, into=(self._y, self._s))
        except IncompleteSketchError:
            em = 0
        self.emitted += em
        self.last_item_emitted = em
        self._unset = int(torch.isinf(self._y).sum().item())

    @property
    def unset_count(self) -> int:
        self._flush()
        return self._unset

    @property
    def prune_enabled(self) -> bool:
        return self.unset_count == 0


def stream_update(state: StreamSketchState, item: StreamItem) -> StreamSketchState:
    """Fold one (element, weight) item into the sketch (stream.py:58-122)."""
    element, weight = item
    element = int(element)
    weight = float(weight)
    if not math.isfinite(weight) or weight <= 0.0 or weight < MIN_WEIGHT:
        raise InvalidWeightError(f"element {element}: weight must be positive and finite, got {weight}")
    known = state.weights.get(element)
    if known is not None:
        if known != weight:
            raise InconsistentWeightError(
                f"element {element} reappeared with weight {weight}, previously {known}")
        if state.skip_duplicates:
            state.last_item_emitted = 0
            return state
    else:
        state.weights[element] = weight
    if not 0 <= element <= _MASK64:
        state._alias[element & _MASK64] = element
    state._pending_ids.append(element)
    state._pending_w.append(weight)
    if len(state._pending_ids) >= FLUSH_ITEMS:
        state._flush()
    return state


def stream_finalize(state: StreamSketchState) -> GumbelMaxSketch:
    """Freeze the state; IncompleteSketchError if a register is unset (stream.py:125-140)."""
    state._flush()
    y = state._y.cpu().numpy()
    if state._unset > 0:
        raise IncompleteSketchError([j for j in range(state.k) if math.isinf(y[j])])
    s = state._s.cpu().numpy().view(np.uint64)
    alias = state._alias
    s_out = tuple(alias.get(int(x), int(x)) for x in s)
    return GumbelMaxSketch(state.k, s_out, tuple(y.tolist()), state.scheme.fingerprint)


def sketch_stream(items: Iterable[StreamItem], k: int, scheme: SeedScheme,
                  skip_duplicates: bool = True) -> GumbelMaxSketch:
    """One-pass sketch of an item iterable (stream.py:143-153)."""
    state = StreamSketchState(k, scheme, skip_duplicates=skip_duplicates)
    for item in items:
        stream_update(state, item)
    return stream_finalize(state)


def sketch_pairs(ids, weights, k: int, scheme: SeedScheme, check: bool = True, exact_y: bool = False,
                 skip_duplicates: bool = True):
    """Bulk stream of (id, weight) arrays, checked and sketched on the device.

    With ``check`` the reference's stream rules run on the device for every
    item at once (gm_check_pairs): InvalidWeightError for a bad weight and
    InconsistentWeightError for an id that reappears with another weight,
    raised for the first offending item like stream_update.  With
    ``skip_duplicates`` only first occurrences are sketched (duplicates are
    register no-ops; stream.py:74-78).  ``exact_y`` re-derives y on the host
    (sketch.exact_y_host, a cross-check: the device y is already the
    reference's).  Returns a GumbelMaxSketch."""
    a_ids, id_bits = _device.id_array(ids)
    a_w, w_bits = _device.weight_array(weights)
    dev = _device.require_cuda()
    ids_t = torch.from_numpy(a_ids.view(np.int32 if id_bits == 32 else np.int64)).to(dev)
    w_t = torch.from_numpy(a_w).to(dev)
    if a_ids.size and (check or skip_duplicates):
        ui = torch.empty_like(ids_t) if skip_duplicates else None
        uw = torch.empty_like(w_t) if skip_duplicates else None
        out = np.zeros(3, np.int64)
        _device.call("gm_check_pairs", ids_t.data_ptr(), id_bits, w_t.data_ptr(), w_bits, a_ids.size,
                     out[0:].ctypes.data, out[1:].ctypes.data, _device.ptr(ui), _device.ptr(uw),
                     out[2:].ctypes.data, _device.stream_ptr())
        first_bad, first_conf, n_uniq = (int(x) for x in out)
        if check and first_bad >= 0 and (first_conf < 0 or first_bad <= first_conf):
            raise InvalidWeightError(f"item {first_bad}: weight must be positive and finite, got {a_w[first_bad]}")
        if check and first_conf >= 0:
            raise InconsistentWeightError(
                f"item {first_conf}: element {int(a_ids[first_conf])} reappeared with another weight")
        if skip_duplicates:
            ids_t, w_t = ui[:n_uniq], uw[:n_uniq]
    y, s, _ = sketch_elements(ids_t, w_t, k, scheme)
    y, s = y.cpu().numpy(), s.cpu().numpy().view(np.uint64)
    if exact_y:  # only the winners' (id, weight) pairs are scanned by the host walk
        keep = np.isin(a_ids, np.unique(s))
        exact_y_host(a_ids[keep], a_w[keep], np.array([0, int(keep.sum())], np.int64), k, scheme, s, y)
    return GumbelMaxSketch(k, tuple(int(x) for x in s), tuple(y.tolist()), scheme.fingerprint)


def parse_stream_items(lines: Iterable[str] | TextIO) -> Iterable[StreamItem]:
    """``element_id weight`` lines (stream.py:156-175)."""
    for number, raw in enumerate(lines, start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        if len(parts) != 2:
            raise InvalidParameterError(f"line {number}: expected 'element_id weight', got {line!r}")
        try:
            element = int(parts[0])
            weight = float(parts[1])
        except ValueError as exc:
            raise InvalidParameterError(f"line {number}: {exc}") from exc
        yield element, weight
