"""Timeline of one config-2 batch through the CSR kernel (-DGM_EVENTS build):
slot events (vector loaded / written / re-opened), slots holding a vector
over time, per-vector latency.  GPU box:

  python tools/timeline.py --build   (here, once: libgmsketch_b200_events.so)
  python tools/timeline.py [n_vec]
"""

import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2302_05176_b200", "libgmsketch_b200_events.so")
if "--build" in sys.argv:  # events-only build: slot events, no per-iteration counters
    import subprocess
    sys.path.insert(0, ROOT)
    from paper_2302_05176_b200 import build as b
    subprocess.run(["nvcc", *b.NVCC_FLAGS, "-DGM_EVENTS", "-o", SO, *b.SOURCES, "-lcudart"], check=True,
                   capture_output=True)
    sys.exit(0)
os.environ["GM_LIB_PATH"] = SO
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_05176_b200 as gm  # noqa: E402
from paper_2302_05176_b200 import _lib, workloads  # noqa: E402


def main():
    nv = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    bucket_us = 10.0
    L = _lib.load()
    ids, w, off, k, seed = workloads.config2(n_vectors=nv)
    d_ids = torch.from_numpy(ids.view(np.int32)).cuda()
    d_w = torch.from_numpy(w).cuda()
    d_off = torch.from_numpy(off).cuda()
    ev = (ctypes.c_ulonglong * 65536)()
    n = ctypes.c_uint()
    for _ in range(2):
        gm.sketch_csr(d_ids, d_w, d_off, k, gm.SeedScheme(seed))
        torch.cuda.synchronize()
        L.gm_trace_read(ev, ctypes.byref(n))
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    gm.sketch_csr(d_ids, d_w, d_off, k, gm.SeedScheme(seed))
    b.record()
    torch.cuda.synchronize()
    print(f"batch of {nv}: {a.elapsed_time(b):.3f} ms (events build)")
    assert L.gm_trace_read(ev, ctypes.byref(n)) == 0
    e = np.array(ev, dtype=np.uint64).reshape(-1, 2)[: n.value]
    t0 = int(e[:, 0].min())
    ts = (e[:, 0].astype(np.int64) - t0) / 1e3  # us
    w1 = e[:, 1]
    vec = (w1 & 0xFFFFFFFF).astype(np.int64)
    att = ((w1 >> 32) & 0xFF).astype(np.int64)
    kind = ((w1 >> 40) & 0xF).astype(np.int64)
    cta = ((w1 >> 48) & 0x3FF).astype(np.int64)
    opens = np.sort(ts[kind == 0])
    closes = np.sort(ts[(kind == 1) | (kind == 3)])
    reopen = np.sort(ts[kind == 2])
    print("time(us)  slots-holding-a-vector  writes-so-far  reopens-so-far")
    tmax = ts.max()
    tb = 0.0
    while tb <= tmax + bucket_us:
        active = np.searchsorted(opens, tb) - np.searchsorted(closes, tb)
        print(f"{tb:8.1f}  {active:6d}  {np.searchsorted(closes, tb):6d}  {np.searchsorted(reopen, tb):5d}")
        tb += bucket_us
    # per-vector latency (first load -> write)
    first = {}
    for ti, v, kd in zip(ts, vec, kind):
        if kd == 0 and v not in first:
            first[v] = ti
    lat = [(ti - first[v], v) for ti, v, kd in zip(ts, vec, kind) if kd == 1 and v in first]
    lat_v = np.array([x for x, _ in lat])
    print(f"vectors written: {len(lat)}; latency us: p10 {np.percentile(lat_v, 10):.1f} p50 {np.percentile(lat_v, 50):.1f} "
          f"p90 {np.percentile(lat_v, 90):.1f} max {lat_v.max():.1f}")
    print(f"re-opened passes: {int((kind == 2).sum())}; chunk events: {int((kind == 3).sum())}")
    writes = np.sort(ts[kind == 1])
    print("write-out times (us) at 50/90/99/100%:", [round(float(np.percentile(writes, q)), 1) for q in (50, 90, 99, 100)])
    loads = np.sort(ts[kind == 0])
    print("load times (us) at 50/90/99/100%:", [round(float(np.percentile(loads, q)), 1) for q in (50, 90, 99, 100)])
    # the last 10 vectors written: when loaded, passes
    order = np.argsort(ts)
    last = [(ts[i], vec[i], att[i], cta[i]) for i in order if kind[i] == 1][-10:]
    for tw, v, a_, c in last:
        print(f"  v={v} written {tw:.1f} us (pass {a_}, cta {c}), first load {first.get(v, float('nan')):.1f} us")


if __name__ == "__main__":
    main()
