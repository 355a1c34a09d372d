"""Throughput of the Python serving loop sketch_csr_host_many on config-2
batches (page-locked tensors in place vs numpy inputs staged), GPU box.
  python tools/host_many.py [batches] [streams]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05176_b200 as gm  # noqa: E402
from paper_2302_05176_b200 import workloads  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
nb = int(args[0]) if args else 64
ns = int(args[1]) if len(args) > 1 else 6
ids, w, off, k, seed = workloads.config2()
sc = gm.SeedScheme(seed)
pinned = (torch.from_numpy(ids.view(np.int32)).pin_memory(), torch.from_numpy(w).pin_memory(),
          torch.from_numpy(off).pin_memory())
for name, b in (("page-locked tensors", pinned), ("numpy arrays", (ids, w, off))):
    for s32 in (False, True):
        for _ in gm.sketch_csr_host_many([b] * (2 * ns), k, sc, streams=ns, s32=s32):
            pass
        t0 = time.perf_counter()
        n = 0
        for y, s in gm.sketch_csr_host_many([b] * nb, k, sc, streams=ns, s32=s32):
            n += 1
        dt = (time.perf_counter() - t0) / n
        print(f"{name:20s} s32={s32}: {1e3 * dt:.3f} ms/batch  {int(off[-1]) / dt / 1e9:.2f} Gelem/s")

if "--profile" in sys.argv:
    import cProfile
    import pstats
    b = pinned
    pr = cProfile.Profile()
    pr.enable()
    for y, s in gm.sketch_csr_host_many([b] * nb, k, sc, streams=ns, s32=True):
        pass
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
