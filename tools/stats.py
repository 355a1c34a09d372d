"""Work counters of the CSR kernel (a -DGM_STATS build of the library).

  python tools/stats.py [2|3]         builds paper_2302_05176_b200/libgmsketch_b200_stats.so
                                      (if missing) and runs one batch of config 2 or 3 through it."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.environ.get("GM_STATS_SO") or os.path.join(ROOT, "paper_2302_05176_b200", "libgmsketch_b200_stats.so")
sys.path.insert(0, ROOT)
if "--build" in sys.argv or not os.path.exists(SO):
    from paper_2302_05176_b200 import build as b  # noqa: E402
    extra = ["-DGM_STATS_WALK"] if os.environ.get("GM_STATS_WALK") else []
    cmd = ["nvcc", *b.NVCC_FLAGS, "-DGM_STATS", *extra, "-o", SO, *b.SOURCES, "-lcudart", "-ldl"]
    subprocess.run(cmd, check=True, capture_output=True)
    if "--build" in sys.argv:
        sys.exit(0)
os.environ["GM_LIB_PATH"] = SO
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_05176_b200 as gm  # noqa: E402
from paper_2302_05176_b200 import _lib, workloads  # noqa: E402

L = _lib.load()
cfg = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 2
ids, w, off, k, seed = workloads.config2() if cfg == 2 else workloads.config3()
d_ids = torch.from_numpy(ids.view(np.int32)).cuda()
d_w = torch.from_numpy(w).cuda()
d_off = torch.from_numpy(off).cuda()
gm.sketch_csr(d_ids, d_w, d_off, k, gm.SeedScheme(seed))
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
L.gm_stats_read(buf)
gm.sketch_csr(d_ids, d_w, d_off, k, gm.SeedScheme(seed))
torch.cuda.synchronize()
L.gm_stats_read(buf)
names = ["idle iters", "step iters", "live lane-steps", "warp walks", "warp-walk arrivals", "deep lanes at steps",
         "idle lanes at steps", "  of which no slot had tickets"]
if os.environ.get("GM_STATS_WALK"):  # walk phases (cycles) instead of the lane categories
    names = ["walk iterations", "step iters", "live lane-steps", "warp walks", "warp-walk arrivals",
             "walk cycles: draws, dense reads, spacings", "walk cycles: prefix", "walk cycles: resolve, stores, CAS"]
for i, nme in enumerate(names):
    print(f"{nme:22s} {buf[i]:>14,d}")
sec = {8: "finalise", 9: "warp walks", 10: "refill", 12: "exit/idle", 13: "lane steps", 14: "completions"}  # section after each marker
tot = sum(buf[i] for i in sec) or 1
print(f"  cycles in slot loads (within finalise) {100 * buf[11] / tot:5.1f}%")
for i, nme in sec.items():
    print(f"  cycles {nme:12s} {100 * buf[i] / tot:5.1f}%")
it = max(buf[1], 1)
print(f"per step iteration (of 32 lanes): live {buf[2] / it:.2f}, deep (waiting for the warp walk) {buf[5] / it:.2f}, "
      f"without an element {buf[6] / it:.2f}")
