"""Config-2 batches back to back: serial (one stream, L2 flushed) vs two
streams alternating (consecutive batches overlap; inputs rotated over R
resident copies so no batch finds its input in L2), device-resident and
through gm_sketch_csr_host with pinned host buffers (GPU box).

  python tools/pipeline.py [steps] [streams]
"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05176_b200 as gm  # noqa: E402
from paper_2302_05176_b200 import _device, _lib, workloads  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    ns = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    L = _lib.load()
    ids, w, off, k, seed = workloads.config2()
    sc = gm.SeedScheme(seed)
    n_vec, n_el = off.size - 1, int(off[-1])
    R = 20  # 20 x 8 MB inputs > 126 MB L2
    d_ids = [torch.from_numpy(ids.view(np.int32)).cuda() for _ in range(R)]
    d_w = [torch.from_numpy(w).cuda() for _ in range(R)]
    d_off = torch.from_numpy(off).cuda()
    streams = [torch.cuda.Stream() for _ in range(ns)]
    ys = [torch.empty((n_vec, k), dtype=torch.float64, device="cuda") for _ in range(ns)]
    ss = [torch.empty((n_vec, k), dtype=torch.int64, device="cuda") for _ in range(ns)]
    flush = torch.empty(512 << 18, dtype=torch.int32, device="cuda")

    def launch(i, st):
        rc = L.gm_sketch_csr(d_ids[i % R].data_ptr(), 32, d_w[i % R].data_ptr(), 32, d_off.data_ptr(), n_vec, k,
                             sc.global_seed, sc.stream_salt, _lib.GM_FLAG_ASYNC, ys[i % ns].data_ptr(),
                             ss[i % ns].data_ptr(), 0, streams[i % ns].cuda_stream if st is None else st)
        assert rc == 0, _lib.last_error()

    # serial, L2 flushed between steps
    cur = torch.cuda.current_stream()
    for i in range(3):
        launch(i, cur.cuda_stream)
    torch.cuda.synchronize()
    tot = 0.0
    for i in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        launch(i, cur.cuda_stream)
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    print(f"serial        {tot / steps:.3f} ms/batch  {n_el * steps / tot / 1e6:.3f} Gelem/s")

    # pipelined over ns streams
    for i in range(2 * ns):
        launch(i, None)
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(streams[0])
    for st in streams[1:]:
        st.wait_event(start)
    for i in range(steps):
        launch(i, None)
    for st in streams[1:]:
        e = torch.cuda.Event()
        e.record(st)
        streams[0].wait_event(e)
    end.record(streams[0])
    torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    print(f"pipelined x{ns}  {ms / steps:.3f} ms/batch  {n_el * steps / ms / 1e6:.3f} Gelem/s")
    assert _device.call("gm_stream_status", streams[0].cuda_stream) == 0

    # end to end through the host API, pinned buffers, same pipeline
    h_ids = torch.from_numpy(ids.view(np.int32)).pin_memory()
    h_w = torch.from_numpy(w).pin_memory()
    h_off = torch.from_numpy(off).pin_memory()
    h_y = [torch.empty((n_vec, k), dtype=torch.float64).pin_memory() for _ in range(ns)]
    h_s = [torch.empty((n_vec, k), dtype=torch.int64).pin_memory() for _ in range(ns)]

    def hcall(i, flags):
        rc = L.gm_sketch_csr_host(h_ids.data_ptr(), 32, h_w.data_ptr(), 32, h_off.data_ptr(), n_vec, k,
                                  sc.global_seed, sc.stream_salt, flags, h_y[i % ns].data_ptr(),
                                  h_s[i % ns].data_ptr(), 0, streams[i % ns].cuda_stream)
        assert rc == 0, _lib.last_error()

    for i in range(2 * ns):
        hcall(i, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        hcall(i, 0)
    t1 = time.perf_counter()
    print(f"e2e serial    {1e3 * (t1 - t0) / steps:.3f} ms/batch")
    for i in range(2 * ns):  # warm the asynchronous path (its device staging)
        hcall(i, _lib.GM_FLAG_ASYNC)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        hcall(i, _lib.GM_FLAG_ASYNC)
    for st in streams:
        st.synchronize()
    t1 = time.perf_counter()
    print(f"e2e pipelined {1e3 * (t1 - t0) / steps:.3f} ms/batch  {n_el * steps / (t1 - t0) / 1e9:.3f} Gelem/s")
    for st in streams:
        assert _device.call("gm_stream_status", st.cuda_stream) == 0
    assert torch.equal(h_s[0], ss[0].cpu()) and torch.equal(h_y[0], ys[0].cpu())
    print("outputs identical")


if __name__ == "__main__":
    main()
