"""End-to-end stream of config-2 batches through gm_sketch_csr_host over S
streams: u64 vs u32 (GM_FLAG_S32) s, wall clock per batch (GPU box).
  python tools/e2e_variants.py [steps] [streams]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05176_b200 as gm  # noqa: E402
from paper_2302_05176_b200 import _lib, workloads  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 3
L = _lib.load()
ids, w, off, k, seed = workloads.config2()
sc = gm.SeedScheme(seed)
n_vec = off.size - 1
streams = [torch.cuda.Stream() for _ in range(ns)]
h_ids = torch.from_numpy(ids.view(np.int32)).pin_memory()
h_w = torch.from_numpy(w).pin_memory()
h_off = torch.from_numpy(off).pin_memory()
for s32 in (False, True):
    h_y = [torch.empty((n_vec, k), dtype=torch.float64).pin_memory() for _ in range(ns)]
    h_s = [torch.empty((n_vec, k), dtype=torch.int32 if s32 else torch.int64).pin_memory() for _ in range(ns)]
    flags = _lib.GM_FLAG_ASYNC | (_lib.GM_FLAG_S32 if s32 else 0)

    def call(i):
        assert L.gm_sketch_csr_host(h_ids.data_ptr(), 32, h_w.data_ptr(), 32, h_off.data_ptr(), n_vec, k,
                                    sc.global_seed, sc.stream_salt, flags, h_y[i % ns].data_ptr(),
                                    h_s[i % ns].data_ptr(), 0, streams[i % ns].cuda_stream) == 0

    for i in range(3 * ns):
        call(i)
    torch.cuda.synchronize()
    for rep in range(3):
        t0 = time.perf_counter()
        for i in range(steps):
            call(i)
        for st in streams:
            st.synchronize()
        dt = (time.perf_counter() - t0) / steps
        print(f"s32={s32} streams={ns}: {1e3 * dt:.3f} ms/batch")
