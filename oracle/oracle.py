"""ctypes wrapper over the CPU restatement ``libgm_oracle.so``.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, ``__graft_entry__.smoke()``
and ``bench.py`` (cpu_baseline and ``--impl reference``) as the checker or
the timed CPU reference; never by the product package.  Each wrapper names
the reference function (``/root/reference/pkg/src/gmsketch``) it restates.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgm_oracle.so")
_lib = None

MASK64 = (1 << 64) - 1
DEFAULT_STREAM_SALT = 0x6A09E667F3BCC909

OK, EMPTY_VECTOR, INVALID_WEIGHT, INVALID_PARAMETER, INCONSISTENT_WEIGHT, INCOMPLETE, NO_MEMORY = range(7)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        u64, i64, i32, dbl = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        vp = ctypes.c_void_p
        L.gmo_mix64.restype = u64
        L.gmo_mix64.argtypes = [u64]
        L.gmo_fingerprint.restype = u64
        L.gmo_fingerprint.argtypes = [u64, u64]
        L.gmo_derive_seed.restype = u64
        L.gmo_derive_seed.argtypes = [u64, u64]
        L.gmo_uniform_open.restype = dbl
        L.gmo_uniform_open.argtypes = [u64, u64, u64]
        L.gmo_rand_int_between.restype = u64
        L.gmo_rand_int_between.argtypes = [u64, u64, u64, u64, u64]
        L.gmo_run_queue_full.restype = None
        L.gmo_run_queue_full.argtypes = [u64, u64, u64, dbl, i32, vp, vp]
        L.gmo_fsum.restype = dbl
        L.gmo_fsum.argtypes = [vp, i64]
        L.gmo_sketch_naive.restype = ctypes.c_int
        L.gmo_sketch_naive.argtypes = [vp, vp, i64, i32, u64, u64, vp, vp, vp]
        L.gmo_sketch_fast.restype = ctypes.c_int
        L.gmo_sketch_fast.argtypes = [vp, vp, i64, i32, i64, u64, u64, vp, vp, vp]
        L.gmo_sketch_stream.restype = ctypes.c_int
        L.gmo_sketch_stream.argtypes = [vp, vp, i64, i32, u64, u64, ctypes.c_int, vp, vp, vp, vp]
        L.gmo_sketch_csr.restype = ctypes.c_int
        L.gmo_sketch_csr.argtypes = [vp, vp, vp, i64, i32, u64, u64, ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.gmo_log_uniforms.restype = None
        L.gmo_log_uniforms.argtypes = [u64, i64, i64, vp, vp]
        L.gmo_merge.restype = None
        L.gmo_merge.argtypes = [vp, vp, i64, i32, vp, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _ids(ids) -> np.ndarray:
    """Element ids as uint64, wrapping negatives mod 2**64 like the reference
    key arithmetic (randgen.py:115, ``& MASK64``)."""
    if isinstance(ids, np.ndarray) and ids.dtype == np.uint64:
        return np.ascontiguousarray(ids)
    if isinstance(ids, np.ndarray) and ids.dtype.kind in "iu":
        return np.ascontiguousarray(ids.astype(np.int64).view(np.uint64) if ids.dtype.kind == "i" else ids.astype(np.uint64))
    return np.array([int(e) & MASK64 for e in ids], dtype=np.uint64)


def _w(w) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(w, dtype=np.float64))


def mix64(x: int) -> int:
    return lib().gmo_mix64(x & MASK64)


def fingerprint(seed: int, salt: int = DEFAULT_STREAM_SALT) -> int:
    return lib().gmo_fingerprint(seed & MASK64, salt & MASK64)


def uniform_open(seed: int, element: int, step: int) -> float:
    return lib().gmo_uniform_open(seed & MASK64, element & MASK64, step)


def rand_int_between(perm_seed: int, element: int, step: int, lo: int, hi: int) -> int:
    return lib().gmo_rand_int_between(perm_seed & MASK64, element & MASK64, step, lo, hi)


def run_queue_full(seed: int, salt: int, element: int, weight: float, k: int):
    t = np.empty(k, np.float64)
    s = np.empty(k, np.int32)
    lib().gmo_run_queue_full(seed & MASK64, (seed ^ salt) & MASK64, element & MASK64, weight, k, _p(t), _p(s))
    return t, s


def fsum(x) -> float:
    a = _w(x)
    return lib().gmo_fsum(_p(a), a.size)


def _sketch_call(fn, ids, w, k, seed, salt, *extra):
    i = _ids(ids)
    ww = _w(w)
    y = np.empty(k, np.float64)
    s = np.empty(k, np.uint64)
    em = np.zeros(1, np.int64)
    rc = fn(_p(i), _p(ww), i.size, k, *extra[:1], seed & MASK64, salt & MASK64, *extra[1:], _p(y), _p(s), _p(em))
    return rc, y, s, int(em[0])


def sketch_naive(ids, w, k, seed, salt=DEFAULT_STREAM_SALT):
    """sketch.py:183-209 over elements in the given order; returns (rc, y, s, emitted)."""
    return _sketch_call(lib().gmo_sketch_naive, ids, w, k, seed, salt)


def sketch_fast(ids, w, k, seed, salt=DEFAULT_STREAM_SALT, delta=0):
    """sketch.py:218-311 over elements in the given order; returns (rc, y, s, emitted)."""
    L = lib()
    i = _ids(ids)
    ww = _w(w)
    y = np.empty(k, np.float64)
    s = np.empty(k, np.uint64)
    em = np.zeros(1, np.int64)
    rc = L.gmo_sketch_fast(_p(i), _p(ww), i.size, k, delta, seed & MASK64, salt & MASK64, _p(y), _p(s), _p(em))
    return rc, y, s, int(em[0])


def sketch_stream(ids, w, k, seed, salt=DEFAULT_STREAM_SALT, skip_duplicates=True):
    """stream.py:143-153; returns (rc, y, s, emitted, err_index)."""
    L = lib()
    i = _ids(ids)
    ww = _w(w)
    y = np.empty(k, np.float64)
    s = np.empty(k, np.uint64)
    em = np.zeros(1, np.int64)
    ei = np.full(1, -1, np.int64)
    rc = L.gmo_sketch_stream(_p(i), _p(ww), i.size, k, seed & MASK64, salt & MASK64, int(bool(skip_duplicates)), _p(y), _p(s), _p(em), _p(ei))
    return rc, y, s, int(em[0]), int(ei[0])


def sketch_csr(ids, w, offsets, k, seed, salt=DEFAULT_STREAM_SALT, mode=0, threads=1):
    """Batch of CSR vectors; mode 0 = sketch_fast per vector (sorted by id),
    mode 1 = sketch_stream per vector.  Returns (rc, y[n_vec,k], s[n_vec,k], emitted[n_vec])."""
    L = lib()
    i = _ids(ids)
    ww = _w(w)
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    nv = off.size - 1
    y = np.empty((nv, k), np.float64)
    s = np.empty((nv, k), np.uint64)
    em = np.zeros(nv, np.int64)
    rc = L.gmo_sketch_csr(_p(i), _p(ww), _p(off), nv, k, seed & MASK64, salt & MASK64, mode, threads, _p(y), _p(s), _p(em))
    return rc, y, s, em


def merge(y, s):
    """estimate.py:103-125 over rows of y[n_sk,k], s[n_sk,k]."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    s = np.ascontiguousarray(s, dtype=np.uint64)
    n, k = y.shape
    yo = np.empty(k, np.float64)
    so = np.empty(k, np.uint64)
    lib().gmo_merge(_p(y), _p(s), n, k, _p(yo), _p(so))
    return yo, so


def log_uniforms(seed: int, i0: int, n: int):
    """(u, log u) for the keyed uniforms uniform_open(seed, i0 + i, 1),
    i < n, with glibc's log (math.log; randgen.py:107-119, :186)."""
    u = np.empty(n, np.float64)
    lg = np.empty(n, np.float64)
    lib().gmo_log_uniforms(seed & MASK64, i0, n, _p(u), _p(lg))
    return u, lg


def sketch_stream_chunked(ids, w, k, seed, salt=DEFAULT_STREAM_SALT, threads=0, chunk=1 << 23):
    """sketch_stream (stream.py:143-153) of a large element set, run as
    contiguous chunks of `chunk` items sketched on all host threads (ctypes
    releases the GIL) and merged in chunk order -- the partition law
    (estimate.py:103-125, test_estimate.py:174-199): equal to one
    sketch_stream of the whole when duplicates carry equal weights.  Each
    worker widens its own chunk to u64 ids / f64 weights, so the whole set is
    never copied.  Returns (rc, y, s)."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    n = len(ids)
    bounds = list(range(0, n, chunk)) + [n]
    threads = threads or min(32, os.cpu_count() or 1)

    def one(c):
        a, b = bounds[c], bounds[c + 1]
        rc, y, s, _, _ = sketch_stream(ids[a:b], w[a:b], k, seed, salt)
        return rc, y, s

    with ThreadPoolExecutor(threads) as ex:
        parts = list(ex.map(one, range(len(bounds) - 1)))
    rc = next((p[0] for p in parts if p[0] not in (OK, INCOMPLETE)), OK)
    if rc != OK:
        return rc, None, None
    y, s = merge(np.stack([p[1] for p in parts]), np.stack([p[2] for p in parts]))
    return (INCOMPLETE if np.isinf(y).any() else OK), y, s


def digest(y, s) -> str:
    """sha256 of the registers: y as IEEE doubles then s as uint64, little-endian."""
    import hashlib

    h = hashlib.sha256()
    h.update(np.ascontiguousarray(y, dtype="<f8").tobytes())
    h.update(np.ascontiguousarray(s, dtype="<u8").tobytes())
    return h.hexdigest()
