"""Seed schemes and the keyed random streams (reference randgen.py).

SeedScheme / derive_seed / mix64 are the reference's 64-bit key algebra
(randgen.py:64-104) on two host integers.  The streams themselves
(uniform_open, the permutation draw) are evaluated by the CUDA library:
uniform_open_batch and perm_draw_batch run the device K0 functions that
every sketch kernel uses, so tests can pin them bit-for-bit against the
reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device

MASK64 = (1 << 64) - 1

# randgen.py:46-61 (must never change: every sketch depends on them)
K_ELEM = 0x9E3779B97F4A7C15
K_STEP = 0xC2B2AE3D27D4EB4F
K_RETRY = 0xD6E8FEB86659FD93
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
DEFAULT_STREAM_SALT = 0x6A09E667F3BCC909
MIN_WEIGHT = 1e-300


def mix64(x: int) -> int:
    """splitmix64 finalizer (randgen.py:64-69)."""
    x &= MASK64
    x = ((x ^ (x >> 30)) * _M1) & MASK64
    x = ((x ^ (x >> 27)) * _M2) & MASK64
    return x ^ (x >> 31)


@dataclass(frozen=True)
class SeedScheme:
    """(global_seed, stream_salt), both masked to 64 bits (randgen.py:72-95)."""

    global_seed: int
    stream_salt: int = DEFAULT_STREAM_SALT

    def __post_init__(self):
        object.__setattr__(self, "global_seed", self.global_seed & MASK64)
        object.__setattr__(self, "stream_salt", self.stream_salt & MASK64)

    @property
    def perm_seed(self) -> int:
        return self.global_seed ^ self.stream_salt

    @property
    def fingerprint(self) -> int:
        return mix64(self.global_seed + mix64(self.stream_salt))


def derive_seed(master: int, index: int) -> int:
    """Child seed for trial ``index`` (randgen.py:98-104)."""
    return mix64((master + (index + 1) * K_ELEM) & MASK64)


class LazyPermutation(dict):
    """Sparse Fisher-Yates array of 1..k (randgen.py:146-155)."""

    def __missing__(self, index):
        return index + 1


def _u64_tensor(values, dev) -> torch.Tensor:
    a = np.asarray([int(v) & MASK64 for v in values], dtype=np.uint64) if not isinstance(
        values, np.ndarray) else np.ascontiguousarray(values.astype(np.uint64))
    return torch.from_numpy(a.view(np.int64)).to(dev)


def uniform_open_batch(seeds, elements, steps) -> np.ndarray:
    """uniform_open (randgen.py:107-119) for arrays of (seed, element, step),
    evaluated on the device by the K0 stream the kernels use."""
    dev = _device.require_cuda()
    s = _u64_tensor(seeds, dev)
    e = _u64_tensor(elements, dev)
    z = _u64_tensor(steps, dev)
    n = s.numel()
    if np.any(np.asarray(steps, dtype=np.int64) < 1):
        raise ValueError("step must be >= 1")
    out = torch.empty(n, dtype=torch.float64, device=dev)
    _device.call("gm_uniform_open_batch", s.data_ptr(), e.data_ptr(), z.data_ptr(), n,
                 out.data_ptr(), _device.stream_ptr())
    return out.cpu().numpy()


def uniform_open(scheme: SeedScheme, element: int, step: int) -> float:
    if step < 1:
        raise ValueError(f"step must be >= 1, got {step}")
    return float(uniform_open_batch([scheme.global_seed], [element], [step])[0])


def perm_draw_batch(perm_seeds, elements, steps, ks) -> np.ndarray:
    """j in [z, k] = rand_int_between(scheme, e, z, z, k) (randgen.py:122-143)
    on the device, for k - z + 1 <= 65536."""
    dev = _device.require_cuda()
    p = _u64_tensor(perm_seeds, dev)
    e = _u64_tensor(elements, dev)
    z = _u64_tensor(steps, dev)
    kk = torch.as_tensor(np.asarray(ks, dtype=np.int64).astype(np.int32), device=dev)
    n = p.numel()
    out = torch.empty(n, dtype=torch.int32, device=dev)
    _device.call("gm_perm_draw_batch", p.data_ptr(), e.data_ptr(), z.data_ptr(), kk.data_ptr(), n,
                 out.data_ptr(), _device.stream_ptr())
    return out.cpu().numpy().astype(np.int64)


def rand_int_between(scheme: SeedScheme, element: int, step: int, lo: int, hi: int) -> int:
    """Unbiased integer in [lo, hi] (randgen.py:122-143), any range up to
    2**64 wide, drawn on the device (gm_rand_int_between_batch)."""
    if step < 1:
        raise ValueError(f"step must be >= 1, got {step}")
    if hi < lo:
        raise ValueError(f"empty range [{lo}, {hi}]")
    m = hi - lo + 1
    if m > 1 << 64:
        # the reference's rejection bound 2**64 - 2**64 % m is 0 here: it never returns
        raise ValueError("ranges wider than 2**64 have no accepted draw")
    dev = _device.require_cuda()
    # the four key arrays stay referenced until the call returns (it synchronises)
    keys = [_u64_tensor([v & MASK64], dev) for v in (scheme.perm_seed, element, step, m - 1)]
    out = torch.empty(1, dtype=torch.int64, device=dev)
    _device.call("gm_rand_int_between_batch", *(a.data_ptr() for a in keys), 1, out.data_ptr(), _device.stream_ptr())
    return lo + (int(out.cpu().item()) & ((1 << 64) - 1))


class ElementQueueState:
    """Generation cursor for one element's queue of k customers
    (randgen.py:210-242): emitted count z, last emitted value b, and the
    Fisher-Yates array perm (values 1..k, a uint32 array).  Advanced on the
    device (gm_queue_advance_batch: the reference's _run_queue arithmetic,
    glibc log included)."""

    def __init__(self, element_id: int, weight: float, k: int, z: int = 0, b: float = 0.0, perm=None):
        from .errors import InvalidWeightError

        weight = float(weight)
        if not (weight > 0.0) or not math.isfinite(weight):
            raise InvalidWeightError(f"element {element_id}: weight must be positive and finite, got {weight}")
        if weight < MIN_WEIGHT:
            raise InvalidWeightError(f"element {element_id}: weight {weight} below {MIN_WEIGHT}")
        self.element_id = int(element_id)
        self.weight = weight
        self.k = int(k)
        self.z = int(z)
        self.b = float(b)
        self.perm = (np.arange(1, self.k + 1, dtype=np.uint32) if perm is None or len(perm) == 0
                     else np.ascontiguousarray(np.asarray(perm, dtype=np.uint32)))

    @property
    def exhausted(self) -> bool:
        return self.z >= self.k


def advance_queues(states, scheme: SeedScheme, steps: int = 1):
    """Advance every ElementQueueState of `states` (same k) by `steps`
    emissions in one device launch (gm_queue_advance_batch); returns
    (times [n, steps] float64, servers [n, steps] int64) and updates the
    states (z, b, perm) in place."""
    from .errors import QueueExhaustedError

    states = list(states)
    if not states:
        return np.zeros((0, steps)), np.zeros((0, steps), np.int64)
    k = states[0].k
    if any(st.k != k for st in states):
        raise ValueError("advance_queues: every queue must have the same k")
    for st in states:
        if st.z + steps > k:
            raise QueueExhaustedError(f"element {st.element_id}: all {st.k} order statistics emitted")
    dev = _device.require_cuda()
    n = len(states)
    el = _u64_tensor([st.element_id for st in states], dev)
    w = torch.tensor([st.weight for st in states], dtype=torch.float64, device=dev)
    z0 = torch.tensor([st.z for st in states], dtype=torch.int32, device=dev)
    b0 = torch.tensor([st.b for st in states], dtype=torch.float64, device=dev)
    perm = torch.from_numpy(np.stack([st.perm for st in states]).view(np.int32)).to(dev)
    t = torch.empty((n, steps), dtype=torch.float64, device=dev)
    s = torch.empty((n, steps), dtype=torch.int32, device=dev)
    bo = torch.empty(n, dtype=torch.float64, device=dev)
    _device.call("gm_queue_advance_batch", el.data_ptr(), w.data_ptr(), z0.data_ptr(), b0.data_ptr(), n, k, steps,
                 scheme.global_seed, scheme.stream_salt, perm.data_ptr(), t.data_ptr(), s.data_ptr(), bo.data_ptr(),
                 _device.stream_ptr())
    perm_h = perm.cpu().numpy().view(np.uint32)
    b_h = bo.cpu().numpy()
    for i, st in enumerate(states):
        st.perm = np.ascontiguousarray(perm_h[i])
        st.z += steps
        st.b = float(b_h[i])
    return t.cpu().numpy(), s.cpu().numpy().astype(np.int64)


def next_order_statistic(state: ElementQueueState, scheme: SeedScheme) -> tuple[float, int]:
    """Advance a queue by one emission; (arrival time, server) (randgen.py:245-271)."""
    t, s = advance_queues([state], scheme, 1)
    return float(t[0, 0]), int(s[0, 0])
