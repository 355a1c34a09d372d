"""Decompose the end-to-end host call of the config-2 bench (GPU box):
H2D of the inputs, the sketch with device outputs, the sketch storing
straight into pinned host outputs, D2H of the outputs, and the full
gm_sketch_csr_host call.  Prints one line per part (ms, median of 20).

  python tools/e2e_parts.py
"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05176_b200 as gm  # noqa: E402
from paper_2302_05176_b200 import _device, _lib, workloads  # noqa: E402


def timed(fn, n=20, host=False):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(n):
        if host:
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            out.append(1e3 * (time.perf_counter() - t0))
        else:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            out.append(a.elapsed_time(b))
    return float(np.median(out))


def main():
    ids, w, off, k, seed = workloads.config2()
    sc = gm.SeedScheme(seed)
    L = _lib.load()
    sp = _device.stream_ptr()
    n_vec = len(off) - 1
    h_ids = torch.from_numpy(ids.view(np.int32)).pin_memory()
    h_w = torch.from_numpy(w).pin_memory()
    h_off = torch.from_numpy(off).pin_memory()
    d_ids, d_w, d_off = h_ids.cuda(), h_w.cuda(), h_off.cuda()
    y = torch.empty((n_vec, k), dtype=torch.float64, device="cuda")
    s = torch.empty((n_vec, k), dtype=torch.int64, device="cuda")
    h_y = torch.empty((n_vec, k), dtype=torch.float64).pin_memory()
    h_s = torch.empty((n_vec, k), dtype=torch.int64).pin_memory()

    def sk(yp, spp, flags=_lib.GM_FLAG_ASYNC):
        rc = L.gm_sketch_csr(d_ids.data_ptr(), 32, d_w.data_ptr(), 32, d_off.data_ptr(), n_vec, k,
                             sc.global_seed, sc.stream_salt, flags, yp, spp, 0, sp)
        assert rc == 0, _lib.last_error()

    def h2d():
        d_ids.copy_(h_ids, non_blocking=True)
        d_w.copy_(h_w, non_blocking=True)
        d_off.copy_(h_off, non_blocking=True)

    def d2h():
        h_y.copy_(y, non_blocking=True)
        h_s.copy_(s, non_blocking=True)

    def host_call():
        rc = L.gm_sketch_csr_host(h_ids.data_ptr(), 32, h_w.data_ptr(), 32, h_off.data_ptr(), n_vec, k,
                                  sc.global_seed, sc.stream_salt, 0, h_y.data_ptr(), h_s.data_ptr(), 0, sp)
        assert rc == 0, _lib.last_error()

    print(f"h2d inputs ({(ids.nbytes + w.nbytes + off.nbytes) / 1e6:.1f} MB)   {timed(h2d):.3f} ms")
    print(f"sketch, device outputs           {timed(lambda: sk(y.data_ptr(), s.data_ptr())):.3f} ms")
    print(f"sketch, pinned host outputs      {timed(lambda: sk(h_y.data_ptr(), h_s.data_ptr())):.3f} ms")
    print(f"d2h outputs ({2 * y.numel() * 8 / 1e6:.1f} MB)   {timed(d2h):.3f} ms")
    print(f"h2d + sketch(dev) + d2h (events) {timed(lambda: (h2d(), sk(y.data_ptr(), s.data_ptr()), d2h())):.3f} ms")
    print(f"gm_sketch_csr_host (wall)        {timed(host_call, host=True):.3f} ms")
    print(f"sync sketch(dev) (wall)          {timed(lambda: sk(y.data_ptr(), s.data_ptr(), 0), host=True):.3f} ms")


if __name__ == "__main__":
    main()
