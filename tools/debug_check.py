"""Run K1 over stress inputs with a -DGM_DEBUG build of the library (bounds and
invariant checks compiled in; GM_LIB_PATH=gpu_scratch/lib_dbg.so) and print the
first failed check, if any (line << 32 | code; 0 = none)."""
import ctypes
import math
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2302_05176_b200 as gm  # noqa: E402
from paper_2302_05176_b200 import _lib, workloads  # noqa: E402

L = _lib.load()


def err():
    out = ctypes.c_ulonglong(0)
    L.gm_debug_error(ctypes.byref(out))
    return out.value


for k, depth in [(1024, 36.0), (1024, 44.0), (600, 40.0), (512, 36.0), (300, 30.0), (129, 20.0), (40, 12.0), (8, 3.0), (1, 1.0)]:
    rng = np.random.default_rng(k)
    n0 = max(2, int(k * (math.log(k) + 2.5) / depth))
    sizes = rng.integers(max(1, int(n0 * 0.8)), int(n0 * 1.2) + 2, size=64)
    off = np.zeros(sizes.size + 1, np.int64)
    off[1:] = np.cumsum(sizes)
    ids = np.concatenate([rng.choice(1 << 31, size=int(m), replace=False) + 1 for m in sizes]).astype(np.uint32)
    w = rng.uniform(0.7, 1.3, size=int(off[-1]))
    gm.sketch_csr(ids, w, off, k, gm.SeedScheme(5))
    gm.sketch_csr(ids, w, off, k, gm.SeedScheme(5), counted=True)
    if k <= 512:
        gm.sketch_vector_seeds(ids[:off[1]], w[:off[1]], k, [gm.SeedScheme(9 + r) for r in range(40)])
    e = err()
    print(f"k={k} depth~{depth}: debug word {e:#x} (line {e >> 32}, code {e & 0xFFFFFFFF})")
ids, w, off, k, seed = workloads.config2()
gm.sketch_csr(ids, w, off, k, gm.SeedScheme(seed))
print(f"config 2: debug word {err():#x}")
ids, w, off, k, seed = workloads.config3(n_vectors=5000)
gm.sketch_csr(ids, w, off, k, gm.SeedScheme(seed))
print(f"config 3 (5000 vectors): debug word {err():#x}")
