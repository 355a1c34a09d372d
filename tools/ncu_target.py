"""A short, deterministic program for ncu evidence captures (never timed).

  python tools/ncu_target.py --config N [--out gpurun_out/target_configN.json]

Runs the roofline probe (chains 1, 2 and 4 -- the kernel arrival_probe_kernel)
and sketches of config N through the C ABI (configs 1-3: csr4_kernel, two
counted launches and a last one without counting, as bench.py runs it;
4-5: the element-set kernels), and writes the per-launch work the evidence
needs: algorithmic and executed arrivals per K1 launch, probe
arrivals per launch.  tools/make_evidence.py joins it with the ncu CSV."""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2302_05176_b200 as gm  # noqa: E402
from paper_2302_05176_b200 import _device, _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out = a.out or os.path.join(ROOT, "gpurun_out", f"target_config{a.config}.json")
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    L = _lib.load()
    info = {"config": a.config}
    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    ids, w, off, k, seed, desc = bench.load_workload(a.config)
    probe = {}
    names = {1: "<1, 1>", 2: "<2, 1>", 4: "<4, 1>", 5: "<1, 8>", 6: "<2, 6>", 7: "<1, 6>"}
    for variant, chains in bench.PROBE_VARIANTS.items():
        n_threads, iters = sms * 2048 // chains, 512
        _device.call("gm_probe_arrival_rate", n_threads, iters | (variant << 24), k, sink.data_ptr(), st.cuda_stream)
        probe[f"arrival_probe_kernel{names[variant]}"] = n_threads * chains * iters
    info["probe_arrivals_per_launch"] = probe
    sc = gm.SeedScheme(seed)
    if a.config in (2, 3):
        d_ids = torch.from_numpy(ids.view(np.int32)).to(dev)
        d_w = torch.from_numpy(w).to(dev)
        d_off = torch.from_numpy(off).to(dev)
        n_vec = off.size - 1
        y = torch.empty((n_vec, k), dtype=torch.float64, device=dev)
        s = torch.empty((n_vec, k), dtype=torch.int64, device=dev)
        em = torch.empty(n_vec, dtype=torch.int64, device=dev)
        for _ in range(2):
            _device.call("gm_sketch_csr", d_ids.data_ptr(), 32, d_w.data_ptr(), 32, d_off.data_ptr(), n_vec, k,
                         sc.global_seed, sc.stream_salt, 0, y.data_ptr(), s.data_ptr(), em.data_ptr(), st.cuda_stream)
        info["executed_arrivals_per_launch"] = int(em.sum().item())
        # the last launch (the one the evidence reads) runs as bench.py times
        # it: no arrival counting
        _device.call("gm_sketch_csr", d_ids.data_ptr(), 32, d_w.data_ptr(), 32, d_off.data_ptr(), n_vec, k,
                     sc.global_seed, sc.stream_salt, 0, y.data_ptr(), s.data_ptr(), None, st.cuda_stream)
        info["algorithmic_arrivals_per_launch"] = bench.algorithmic_arrivals(dev, st, d_ids, 32, d_w, 32, d_off,
                                                                             n_vec, k, sc.global_seed, y)
        info["input_bytes"] = int(ids.nbytes + w.nbytes + off.nbytes)
        info["output_bytes"] = int(n_vec * k * 16)
    elif a.config == 1:
        R = bench.CONFIG1_SEEDS
        b = gm.sketch_vector_seeds(ids, w, k, [gm.SeedScheme(1 + r) for r in range(R)], counted=True)
        b = gm.sketch_vector_seeds(ids, w, k, [gm.SeedScheme(1 + r) for r in range(R)], counted=True)
        info["executed_arrivals_per_launch"] = int(b.emitted.sum().item())
        b = gm.sketch_vector_seeds(ids, w, k, [gm.SeedScheme(1 + r) for r in range(R)])  # uncounted, last
    else:
        id_bits = ids.dtype.itemsize * 8
        d_ids = torch.from_numpy(ids.view(np.int64 if id_bits == 64 else np.int32)).to(dev)
        d_w = torch.from_numpy(w).to(dev)
        y = torch.empty(k, dtype=torch.float64, device=dev)
        s = torch.empty(k, dtype=torch.int64, device=dev)
        for _ in range(2):
            _device.call("gm_sketch_elements", d_ids.data_ptr(), id_bits, d_w.data_ptr(), 32, ids.size, k,
                         sc.global_seed, sc.stream_salt, 0, y.data_ptr(), s.data_ptr(), None, st.cuda_stream)
        info["input_bytes"] = int(ids.nbytes + w.nbytes)
    torch.cuda.synchronize()
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(info, f, indent=1)
    print(json.dumps(info))


if __name__ == "__main__":
    main()
