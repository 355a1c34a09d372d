"""Sketch time vs batch size on config-2-shaped vectors (1000 ids, fp32
Exp(1), k=1024): exposes the tail of the persistent CSR kernel (GPU box).

  python tools/batch_scaling.py
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05176_b200 as gm  # noqa: E402
from paper_2302_05176_b200 import _device, _lib, workloads  # noqa: E402


def main():
    L = _lib.load()
    sp = _device.stream_ptr()
    for nv in (148, 296, 592, 1000, 2000, 4000, 8000):
        ids, w, off, k, seed = workloads.config2(n_vectors=nv)
        sc = gm.SeedScheme(seed)
        d_ids = torch.from_numpy(ids.view(np.int32)).cuda()
        d_w = torch.from_numpy(w).cuda()
        d_off = torch.from_numpy(off).cuda()
        y = torch.empty((nv, k), dtype=torch.float64, device="cuda")
        s = torch.empty((nv, k), dtype=torch.int64, device="cuda")

        def run():
            rc = L.gm_sketch_csr(d_ids.data_ptr(), 32, d_w.data_ptr(), 32, d_off.data_ptr(), nv, k,
                                 sc.global_seed, sc.stream_salt, _lib.GM_FLAG_ASYNC, y.data_ptr(),
                                 s.data_ptr(), 0, sp)
            assert rc == 0

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        a.record()
        for _ in range(reps):
            run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        print(f"n_vec {nv:5d}: {ms:.3f} ms  {ms / nv * 1e3:.3f} us/vector  {int(off[-1]) / ms / 1e6:.3f} Gelem/s")


if __name__ == "__main__":
    main()
