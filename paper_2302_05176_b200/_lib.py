"""ctypes binding of libgmsketch_b200.so (include/gmsketch_b200.h).

The CUDA library is the only compute path: if it is missing or no sm_100
device is visible, every sketch call raises instead of falling back to a
CPU implementation.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GM_LIB_PATH") or os.path.join(_HERE, "libgmsketch_b200.so")

GM_OK = 0
GM_ERR_EMPTY_VECTOR = 1
GM_ERR_INVALID_WEIGHT = 2
GM_ERR_INVALID_PARAMETER = 3
GM_ERR_INCONSISTENT_WEIGHT = 4
GM_ERR_INCOMPLETE = 5
GM_ERR_MISMATCHED = 6
GM_ERR_CUDA = 100
GM_ERR_NO_DEVICE = 101
GM_ERR_COMM = 102

GM_FLAG_ASYNC = 0x1
GM_FLAG_EXHAUSTIVE = 0x2
GM_FLAG_ACCUMULATE = 0x4
GM_FLAG_S32 = 0x10
GM_FLAG_ONE_VECTOR = 0x20

# every symbol include/gmsketch_b200.h declares: (name, restype, argtypes)
_u64, _i64, _i32, _u32, _int, _vp, _dbl = (ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32,
                                           ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p,
                                           ctypes.c_double)
SIGNATURES = {
    "gm_version": (_int, []),
    "gm_debug_error": (_int, [_vp]),
    "gm_last_error": (ctypes.c_char_p, []),
    "gm_stats_read": (_int, [_vp]),
    "gm_trace_read": (_int, [_vp, _vp]),
    "gm_stream_status": (_int, [_vp]),
    "gm_comm_id_bytes": (_int, []),
    "gm_comm_unique_id": (_int, [_vp]),
    "gm_comm_init": (_int, [_vp, _int, _int, _vp]),
    "gm_comm_destroy": (_int, [_vp]),
    "gm_allreduce_min_registers": (_int, [_vp, _vp, _vp, _i32, _vp]),
    "gm_allgather_merge_registers": (_int, [_vp, _vp, _vp, _i32, _vp]),
    "gm_release_stream": (_int, [_vp]),
    "gm_finalize": (_int, []),
    "gm_workspace_count": (_int, []),
    "gm_sketch_csr": (_int, [_vp, _int, _vp, _int, _vp, _i64, _i32, _u64, _u64, _u32, _vp, _vp, _vp, _vp]),
    "gm_sketch_csr_seeded": (_int, [_vp, _int, _vp, _int, _vp, _i64, _i32, _vp, _u64, _u32, _vp, _vp, _vp, _vp]),
    "gm_sketch_csr_host": (_int, [_vp, _int, _vp, _int, _vp, _i64, _i32, _u64, _u64, _u32, _vp, _vp, _vp, _vp]),
    "gm_sketch_elements": (_int, [_vp, _int, _vp, _int, _i64, _i32, _u64, _u64, _u32, _vp, _vp, _vp, _vp]),
    "gm_sketch_elements_host": (_int, [_vp, _int, _vp, _int, _i64, _i32, _u64, _u64, _u32, _vp, _vp, _vp, _vp]),
    "gm_sketch_elements_async": (_int, [_vp, _int, _vp, _int, _i64, _i32, _u64, _u64, _u32, _vp, _vp, _vp, _vp]),
    "gm_merge": (_int, [_vp, _vp, _i64, _i32, _vp, _vp, _vp]),
    "gm_match_count": (_int, [_vp, _vp, _i64, _i32, _vp, _vp]),
    "gm_cardinality": (_int, [_vp, _i64, _i32, _vp, _vp, _vp]),
    "gm_uniform_open_batch": (_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "gm_perm_draw_batch": (_int, [_vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "gm_rand_int_between_batch": (_int, [_vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "gm_arith_check": (_int, [_i64, _u64, _vp, _vp]),
    "gm_log_batch": (_int, [_vp, _i64, _vp, _vp]),
    "gm_check_pairs": (_int, [_vp, _int, _vp, _int, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "gm_queue_advance_batch": (_int, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _u64, _u64, _vp, _vp, _vp, _vp, _vp]),
    "gm_exact_y": (_int, [_vp, _int, _vp, _int, _vp, _i64, _i32, _u64, _u64, _vp, _vp, _i32]),
    "gm_probe_arrival_rate": (_int, [_i64, _i32, _i32, _vp, _vp]),
    "gm_count_arrivals_csr": (_int, [_vp, _int, _vp, _int, _vp, _i64, _i32, _u64, _vp, _vp, _vp]),
}

_lib = None
_lock = threading.Lock()


class LibraryMissingError(RuntimeError):
    """libgmsketch_b200.so is absent or unloadable (no CPU fallback exists)."""


def load():
    """Load the CUDA library (does not need a GPU to load)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissingError(
                    f"{LIB_PATH} not built; run __graft_entry__.build() (there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def last_error() -> str:
    msg = load().gm_last_error()
    return msg.decode() if msg else ""
