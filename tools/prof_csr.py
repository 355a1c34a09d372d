"""Run the config-2 batch sketch a few times (profiling target for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05176_b200 as gm  # noqa: E402
from paper_2302_05176_b200 import workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if cfg == 2:
    ids, w, off, k, seed = workloads.config2()
else:
    ids, w, off, k, seed = workloads.config3(n_vectors=20000)
d_ids = torch.from_numpy(ids.view(np.int32)).cuda()
d_w = torch.from_numpy(w).cuda()
d_off = torch.from_numpy(off).cuda()
for _ in range(reps):
    b = gm.sketch_csr(d_ids, d_w, d_off, k, gm.SeedScheme(seed))
torch.cuda.synchronize()
print("ok", float(b.y.sum()))
