"""Timing of the element-set path (configs 4 and 5) on the device.

  python tools/bench_elements.py [n5] [n4]
Config 5: weights LogNormal(0,2) generated on the device (torch, seeded), ids
0..n-1, k=8192.  Config 4: the seeded Zipf stream prefix (workloads.config4),
k=4096.  Prints elements/s and ms per sketch (CUDA events, median of 5)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05176_b200 as gm  # noqa: E402
from paper_2302_05176_b200 import workloads  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


n5 = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**8
n4 = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10**7
g = torch.Generator(device="cuda").manual_seed(5)
w5 = torch.empty(n5, device="cuda", dtype=torch.float32).log_normal_(0.0, 2.0, generator=g)
ids5 = torch.arange(n5, device="cuda", dtype=torch.int32)
sc = gm.SeedScheme(1)
ms = timeit(lambda: gm.sketch_elements(ids5, w5, 8192, sc))
print(f"config5 n={n5:.3g}: {ms:.3f} ms  {n5 / ms / 1e6:.3g} Gelem/s")
ids4, w4, k4, seed = workloads.config4(n_pairs=n4, n_keys=10**7)
i4 = torch.from_numpy(ids4.view(np.int64)).cuda()
ww4 = torch.from_numpy(w4).cuda()
ms = timeit(lambda: gm.sketch_elements(i4, ww4, k4, gm.SeedScheme(seed)))
print(f"config4 n={n4:.3g}: {ms:.3f} ms  {n4 / ms / 1e6:.3g} Gpairs/s")
