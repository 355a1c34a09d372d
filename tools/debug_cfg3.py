"""Debug: config-3 subset on the device vs the oracle; per failing vector report."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05176_b200 as gm  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2302_05176_b200 import workloads  # noqa: E402

nv = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
ids, w, off, k, seed = workloads.config3(n_vectors=nv)
rc, yo, so, _ = O.sketch_csr(ids.astype(np.uint64), w.astype(np.float64), off, k, seed, mode=0, threads=8)
for rep in range(3):
    b = gm.sketch_csr(ids, w, off, k, gm.SeedScheme(seed), counted=True)
    y = b.y.cpu().numpy()
    s = b.s.cpu().numpy().view(np.uint64)
    bad = np.nonzero(np.any(s != so, axis=1))[0]
    print(f"rep {rep}: {len(bad)} bad vectors {bad[:20]}")
    for v in bad[:5]:
        a, e = off[v], off[v + 1]
        ww = w[a:e].astype(np.float64)
        tau = (np.log(k) + 2.5) / ww.sum()
        nd = int(((s[v] != so[v])).sum())
        ninf = int(np.isinf(y[v]).sum())
        rel = np.abs(y[v] - yo[v]) / yo[v]
        print(f"  v={v} n={e - a} maxdepth={k * tau * ww.max():.1f} diff_regs={nd} inf={ninf} "
              f"ybigger={int((y[v] > yo[v]).sum())} ysmaller={int((y[v] < yo[v]).sum())} maxrel={np.nanmax(rel):.3g}")

# provenance of wrong registers of the first bad vectors (last rep)
idset = {}
for v in bad[:8]:
    a, e = off[v], off[v + 1]
    mine = set(ids[a:e].tolist())
    wrong = np.nonzero(s[v] != so[v])[0]
    foreign = [int(s[v][j]) for j in wrong if int(s[v][j]) not in mine]
    # which vector do the foreign ids come from?
    src = []
    for f in foreign[:5]:
        hit = np.nonzero(ids == f)[0]
        src.append([int(np.searchsorted(off, h, side="right") - 1) for h in hit[:3]])
    print(f"v={v}: wrong={len(wrong)} foreign={len(foreign)} from vectors {src}")
