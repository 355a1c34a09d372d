"""bench.py -- FastGM sketch throughput on B200 (BASELINE.json metric).

Metric: positive elements sketched per second at k=1024 (BASELINE.json
configs[1], "config 2": 1,000 sparse vectors x 1,000 ids over 10**6,
fp32 Exponential(1) weights, vectors paired for J_P), seeded synthetic
input (paper_2302_05176_b200/workloads.py).  One step = one batched sketch
of all 1,000 vectors (10**6 elements) by the C-ABI entry gm_sketch_csr.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2|3|4|5]

N > 1 (torchrun): vectors are sharded across ranks by element count, no
collective on the data path (scaling "weak": every rank sketches its own
full config-2 batch); timing is max over ranks of device time.

--impl reference times the reference algorithm's CPU implementation (the
bit-exact C port of sketch_fast in oracle/, all host threads) on the same
workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=2, choices=[2, 3])
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def load_workload(cfg: int):
    from paper_2302_05176_b200 import workloads

    if cfg == 2:
        ids, w, off, k, seed = workloads.config2()
        desc = "config2: 1000 vectors x 1000 ids over 1e6, fp32 Exp(1), k=1024, pairs (2i,2i+1)"
    else:
        ids, w, off, k, seed = workloads.config3(n_vectors=100_000)
        desc = "config3: 1e5 CSR vectors, n~LogNormal(6,1), fp32 Pareto(1.5), k=512"
    return ids, w, off, k, seed, desc


class ClockSampler:
    """SM clock and clock-event (throttle) reasons polled through NVML every
    ~1 ms on a thread while the timed region runs (nvidia-smi's 100 ms loop is
    too coarse for a region of tens of milliseconds)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.sm_max = None
        self._stop = threading.Event()
        self._thread = None

    def _run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.sm_max = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, rs))
                time.sleep(0.001)
            pynvml.nvmlShutdown()
        except Exception:  # no NVML: report unavailable
            self.samples = []

    def __enter__(self):
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()
        time.sleep(0.05)  # first samples before the region starts
        return self

    def __exit__(self, *exc):
        time.sleep(0.01)
        self._stop.set()
        self._thread.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [x[0] for x in self.samples]
        reasons = sorted({name for _, r in self.samples for bit, name in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.sm_max, "reasons": reasons,
                "samples": len(self.samples), "source": "NVML polled ~1 ms during the timed region"}


def peaks():
    try:
        with open(MEASURED_PEAKS) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def cpu_oracle_time(ids, w, off, k, seed, n_vec_sample, threads):
    """Time the C port of the reference's sketch_fast (oracle/) over the
    first n_vec_sample vectors on `threads` host threads; returns (seconds, elements)."""
    from oracle import oracle as O

    ids64 = ids.astype(np.uint64)
    w64 = w.astype(np.float64)
    off_s = off[: n_vec_sample + 1]
    n = int(off_s[-1])
    t0 = time.perf_counter()
    rc, _, _, _ = O.sketch_csr(ids64[:n], w64[:n], off_s, k, seed, mode=0, threads=threads)
    dt = time.perf_counter() - t0
    assert rc == 0
    return dt, n


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm on the host CPU, rank 0 only."""
    if rank != 0:
        return
    ids, w, off, k, seed, desc = load_workload(args.config)
    threads = os.cpu_count() or 1
    n_vec = off.size - 1
    # bounded sample per step: a prefix of the batch sized for ~10 s of CPU work in total
    probe_dt, probe_n = cpu_oracle_time(ids, w, off, k, seed, min(n_vec, 64), threads)
    per_vec = probe_dt / 64
    budget = max(1.0, 8.0 / max(1, args.steps + args.warmup))
    n_sample = int(min(n_vec, max(threads, budget / max(per_vec, 1e-9))))
    for _ in range(args.warmup):
        cpu_oracle_time(ids, w, off, k, seed, n_sample, threads)
    times, elems = [], 0
    for _ in range(args.steps):
        dt, n = cpu_oracle_time(ids, w, off, k, seed, n_sample, threads)
        times.append(dt)
        elems = n
    total = sum(times)
    value = elems * args.steps / total
    line = {
        "impl": "reference", "metric": "positive elements sketched/sec at k=%d" % k, "value": value,
        "unit": "elements/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, workloads.py)",
        "config": {"workload": desc, "sample_vectors_per_step": n_sample,
                   "parallelism": f"host threads x{threads}"},
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": threads, "kind": "port",
                         "sample": f"first {n_sample} of {n_vec} vectors per step ({elems} elements), "
                                   "oracle/gm_oracle.c sketch_fast (bit-exact C port of sketch.py:218-311)"},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_2302_05176_b200 as gm
    from paper_2302_05176_b200 import _device, _lib, shard

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L = _lib.load()
    ids, w, off, k, seed, desc = load_workload(args.config)
    scheme = gm.SeedScheme(seed)
    # weak scaling: every rank sketches a full batch of its own; at N=1 this is the config
    n_vec = off.size - 1
    n_el = int(off[-1])
    d_ids = torch.from_numpy(ids.view(np.int32)).to(dev)
    d_w = torch.from_numpy(w).to(dev)
    d_off = torch.from_numpy(off).to(dev)
    y = torch.empty((n_vec, k), dtype=torch.float64, device=dev)
    s = torch.empty((n_vec, k), dtype=torch.int64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def step():
        rc = L.gm_sketch_csr(d_ids.data_ptr(), 32, d_w.data_ptr(), 32, d_off.data_ptr(), n_vec, k,
                             scheme.global_seed, scheme.stream_salt, _lib.GM_FLAG_ASYNC, y.data_ptr(),
                             s.data_ptr(), 0, sp)
        if rc:
            raise RuntimeError(_lib.last_error())

    for _ in range(max(3, args.warmup)):
        step()
    _device.call("gm_stream_status", sp)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clocks:
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    _device.call("gm_stream_status", sp)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    value = n_el * world * args.steps / (total_ms / 1e3)

    # ---- end to end through the public C-ABI with pinned host buffers
    h_ids = torch.from_numpy(ids.view(np.int32)).pin_memory()
    h_w = torch.from_numpy(w).pin_memory()
    h_off = torch.from_numpy(off).pin_memory()
    h_y = torch.empty((n_vec, k), dtype=torch.float64).pin_memory()
    h_s = torch.empty((n_vec, k), dtype=torch.int64).pin_memory()

    def e2e_step():
        rc = L.gm_sketch_csr_host(h_ids.data_ptr(), 32, h_w.data_ptr(), 32, h_off.data_ptr(), n_vec, k,
                                  scheme.global_seed, scheme.stream_salt, 0, h_y.data_ptr(), h_s.data_ptr(),
                                  0, sp)
        if rc:
            raise RuntimeError(_lib.last_error())

    for _ in range(max(3, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()  # synchronous: H2D, kernel, D2H, stream sync
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    e2e_total = sum(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = n_el * world * args.steps / (e2e_total / 1e3)
    h2d = ids.nbytes + w.nbytes + off.nbytes
    d2h = n_vec * k * 16

    # parity spot check of the timed output against the host result
    assert torch.equal(s.cpu(), h_s) and torch.equal(y.cpu(), h_y)

    if rank != 0:
        return

    # ---- roofline: arrival-generation speed of light, measured in this run
    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    n_threads, iters = 148 * 2048, 256
    for _ in range(2):
        _device.call("gm_probe_arrival_rate", n_threads, iters, k, sink.data_ptr(), sp)
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for _ in range(5):
        _device.call("gm_probe_arrival_rate", n_threads, iters, k, sink.data_ptr(), sp)
    a1.record(stream)
    torch.cuda.synchronize()
    peak_arrivals = 5 * n_threads * iters / (a0.elapsed_time(a1) / 1e3)

    # algorithmic arrivals per launch: n+ (one terminating arrival per element) +
    # arrivals <= the final max register of each vector (the survivors any exact
    # threshold walk must emit)
    tau = y.max(dim=1).values.contiguous()
    counts = torch.zeros(n_vec, dtype=torch.int64, device=dev)
    _device.call("gm_count_arrivals_csr", d_ids.data_ptr(), 32, d_w.data_ptr(), 32, d_off.data_ptr(), n_vec, k,
                 scheme.global_seed, tau.data_ptr(), counts.data_ptr(), sp)
    survivors = int(counts.sum().item())
    alg_arrivals = n_el + survivors
    emitted = torch.empty(n_vec, dtype=torch.int64, device=dev)
    L.gm_sketch_csr(d_ids.data_ptr(), 32, d_w.data_ptr(), 32, d_off.data_ptr(), n_vec, k, scheme.global_seed,
                    scheme.stream_salt, 0, y.data_ptr(), s.data_ptr(), emitted.data_ptr(), sp)
    executed = int(emitted.sum().item())
    kernel_ms = total_ms / args.steps
    achieved = alg_arrivals / (kernel_ms / 1e3)
    hbm_peak, hbm_kind = peaks()
    in_bytes = ids.nbytes + w.nbytes + off.nbytes
    out_bytes = n_vec * k * 16
    hbm_achieved = (in_bytes + out_bytes) / (kernel_ms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic_config2.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = os.cpu_count() or 1
        dt_probe, _ = cpu_oracle_time(ids, w, off, k, seed, 64, threads)
        n_sample = int(min(n_vec, max(threads, 15.0 / max(dt_probe / 64, 1e-9))))
        dt, n = cpu_oracle_time(ids, w, off, k, seed, n_sample, threads)
        cpu = {"value": n / dt, "unit": "elements/s", "cores": threads, "kind": "port",
               "sample": f"first {n_sample} of {n_vec} config-2 vectors ({n} elements), "
                         "oracle/gm_oracle.c sketch_fast, all host threads"}

    line = {
        "metric": "positive elements sketched/sec at k=%d" % k,
        "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, workloads.py)",
        "config": {"workload": desc, "elements_per_step_per_gpu": n_el, "k": k,
                   "parallelism": f"vector shards x{world}" if world > 1 else "single GPU",
                   "l2": "flushed (512 MiB write) between timed steps"},
        "e2e": {"value": e2e_value, "unit": "elements/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_total / args.steps, "api": "gm_sketch_csr_host (pinned host buffers)"},
        "gpu_launches": 2 * args.steps,  # per step: csr_prep_kernel + csr3_kernel
        "roofline": {"bound": "compute (exact fp64 arrival generation)", "unit": "arrivals/s",
                     "achieved": achieved, "peak": peak_arrivals, "frac": achieved / peak_arrivals,
                     "traffic": traffic,
                     "peak_source": "gm_probe_arrival_rate measured in this run (no pruning/registers)",
                     "algorithmic_arrivals_per_launch": alg_arrivals, "executed_arrivals_per_launch": executed,
                     "hbm": {"achieved_gbs": hbm_achieved, "peak_gbs": hbm_peak, "peak_kind": hbm_kind,
                             "frac": hbm_achieved / hbm_peak}},
        "clocks": clocks.summary(),
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
