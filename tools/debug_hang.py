import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2302_05176_b200 as gm
from paper_2302_05176_b200 import workloads
nv = int(sys.argv[1])
ids, w, off, k, seed = workloads.config3(n_vectors=nv)
t = time.time()
b = gm.sketch_csr(ids, w, off, k, gm.SeedScheme(seed))
torch.cuda.synchronize()
print(nv, 'ok', time.time() - t, flush=True)
