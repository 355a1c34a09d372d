"""Device plumbing: torch tensors as I/O buffers, the current CUDA stream,
and C-ABI calls that raise the reference exception classes.  PyTorch is
used only for device memory and streams; all compute is in the CUDA
library."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import DeviceError, raise_for

MASK64 = (1 << 64) - 1


def require_cuda() -> torch.device:
    lib = _lib.load()  # raises LibraryMissingError when not built
    del lib
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the FastGM engine runs only on sm_100 GPUs "
                          "(there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


_POOLS: dict[tuple[int, int], list] = {}


def stream_pool(dev: torch.device, n: int) -> list:
    """n CUDA streams of `dev`, created once per process and reused: the
    library keeps scratch per (device, stream), so fresh streams per call
    would each leave a workspace behind (gm_release_stream frees one)."""
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), n)
    pool = _POOLS.get(key)
    if pool is None:
        pool = [torch.cuda.Stream(device=dev) for _ in range(n)]
        _POOLS[key] = pool
    return pool


def call(name: str, *args) -> int:
    rc = getattr(_lib.load(), name)(*args)
    if rc:
        raise_for(rc, _lib.last_error())
    return rc


def ptr(t) -> int:
    if t is None:
        return 0
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    raise TypeError(type(t))


def id_array(ids) -> tuple[np.ndarray, int]:
    """Element ids as a contiguous uint32/uint64 numpy array (ids are keyed
    modulo 2**64 like randgen.py:115); returns (array, id_bits)."""
    if isinstance(ids, np.ndarray) and ids.dtype in (np.uint32, np.uint64):
        a = np.ascontiguousarray(ids)
        return a, 32 if a.dtype == np.uint32 else 64
    if isinstance(ids, np.ndarray) and ids.dtype.kind == "i":
        return np.ascontiguousarray(ids.astype(np.int64).view(np.uint64)), 64
    return np.array([int(e) & MASK64 for e in ids], dtype=np.uint64), 64


def weight_array(w) -> tuple[np.ndarray, int]:
    if isinstance(w, np.ndarray) and w.dtype == np.float32:
        return np.ascontiguousarray(w), 32
    return np.ascontiguousarray(np.asarray(w, dtype=np.float64)), 64


def id_bits_of(t: torch.Tensor) -> int:
    if t.dtype in (torch.int32, torch.uint32):
        return 32
    if t.dtype in (torch.int64, torch.uint64):
        return 64
    raise TypeError(f"ids must be a 32/64-bit integer tensor, got {t.dtype}")


def w_bits_of(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return 32
    if t.dtype == torch.float64:
        return 64
    raise TypeError(f"weights must be float32/float64, got {t.dtype}")
