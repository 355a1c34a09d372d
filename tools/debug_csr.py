"""Debug: one config-2 CSR batch on the device against the oracle, per-register diff report (GPU box)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05176_b200 as gm
from paper_2302_05176_b200 import workloads, _lib
from oracle import oracle as O
L = _lib.load()
def dbg(tag):
    torch.cuda.synchronize()
    e = ctypes.c_ulonglong(0); L.gm_debug_error(ctypes.byref(e)); v = e.value
    print(tag, "dbg line", v >> 32, "code", v & 0xffffffff, flush=True)
for cfg in (3, 2):
    if cfg == 3: ids, w, off, k, seed = workloads.config3(n_vectors=3000)
    else: ids, w, off, k, seed = workloads.config2()
    for rep in range(3):
        try:
            b = gm.sketch_csr(ids, w, off, k, gm.SeedScheme(seed))
            dbg(f"cfg{cfg} rep{rep}")
        except Exception as ex:
            print("EXC", cfg, rep, ex); dbg("after exc"); sys.exit(1)
    y = b.y.cpu().numpy(); s = b.s.cpu().numpy().view(np.uint64)
    rc, yo, so, _ = O.sketch_csr(ids.astype(np.uint64), w.astype(np.float64), off, k, seed, mode=0, threads=8)
    print("cfg", cfg, "s mismatches", int((s != so).sum()), "max rel", float(np.max(np.abs(y - yo) / yo)))
