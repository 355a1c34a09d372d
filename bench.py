"""bench.py -- FastGM sketch throughput on B200 (BASELINE.json metric).

Metric: positive elements sketched per second (BASELINE.json: "at k=1024 on
1-8 B200; % of roofline").  The default workload is BASELINE.json configs[1]
("config 2": 1,000 sparse vectors x 1,000 ids over 10**6, fp32
Exponential(1) weights, k=1024, vectors paired for J_P), seeded synthetic
input (paper_2302_05176_b200/workloads.py).  One step = one batched sketch of
all 1,000 vectors (10**6 elements) by the C-ABI entry gm_sketch_csr.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 1|2|3|4|5]

--config 1: one 10**4-element vector (k=256) sketched under R seeds per step
  (gm_sketch_csr_seeded, the vector stored once), plus the latency of one
  sketch through the host entry (grid-wide kernels).
--config 3: 10**5 CSR vectors (k=512).
--config 4 / 5: one sketch of the Zipf stream (1e8 pairs, k=4096) / the huge
  vector (1e9 elements, k=8192) per step.

N > 1: `--gpus N` without WORLD_SIZE in the environment re-launches itself
under torch.distributed.run with N ranks (one per GPU, NCCL).  Configs 1-2
scale weakly (every rank sketches its own full batch; replicas), config 3
strongly over element-balanced vector ranges (no collective), configs 4-5
strongly over contiguous element shards that every rank generates alone and
whose k registers are combined over NCCL inside the C ABI
(gm_allgather_merge_registers / gm_allreduce_min_registers).  Timing is the
max over ranks of CUDA-event device time.

Every full-size run checks the timed sketches against the committed oracle
digest (tests/golden/full_digests.json) and reports "parity".

--impl reference times the reference algorithm's CPU implementation (the
bit-exact C port in oracle/, all host threads) on the same workload; rank 0
only (other ranks exit 0).
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
DIGESTS = os.path.join(ROOT, "tests", "golden", "full_digests.json")
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2
N_COPIES = 20  # resident input copies the timed batches rotate over (20 x 8 MB > L2)
CONFIG1_SEEDS = 1000  # sketches of the config-1 vector per step (seeds 1..R)
# gm_probe_arrival_rate variants: chains per thread (and the resident-CTA bound)
PROBE_VARIANTS = {1: 1, 2: 2, 4: 4, 5: 1, 6: 2, 7: 1}
PROBE_OCC = {1: "registers unbounded", 2: "registers unbounded", 4: "registers unbounded", 5: "8 CTAs/SM",
             6: "6 CTAs/SM", 7: "6 CTAs/SM"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    p.add_argument("--n", type=float, default=0, help="configs 4/5: override the element count (default: BASELINE size)")
    p.add_argument("--elem-streams", type=int, default=3, help="configs 4/5 at N=1: CUDA streams the sketches rotate over")
    p.add_argument("--merge", default="allgather", choices=["allgather", "allreduce"],
                   help="configs 4/5, N > 1: NCCL all-gather + rank-order device merge, or two NCCL MIN all-reduces")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--streams", type=int, default=6, help="CUDA streams the batches rotate over")
    return p.parse_args()


# ---------------------------------------------------------------- launch
def maybe_spawn(args) -> bool:
    """--gpus N > 1 without a torch.distributed environment: run this script
    under torch.distributed.run with N ranks; rank 0's JSON line is printed."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    res = subprocess.run(cmd, env=env)
    sys.exit(res.returncode)


# ---------------------------------------------------------------- workloads
def load_workload(cfg: int, n: int = 0, lo: int = 0, hi: int | None = None):
    """(ids, w, offsets or None, k, seed, description); configs 4/5 generate
    only elements [lo, hi) (keyed chunks: a rank makes its shard alone)."""
    from paper_2302_05176_b200 import workloads

    if cfg == 1:
        ids, w, k, seed = workloads.config1()
        return ids, w, np.array([0, ids.size], np.int64), k, seed, (
            "config1: one vector, ids 0..9999 (u32), fp64 weights 1 - U[0,1), k=256, sketched under seeds "
            f"1..{CONFIG1_SEEDS} per step")
    if cfg == 4:
        ids, w, k, seed = workloads.config4(n_pairs=n or 10**8, lo=lo, hi=hi)
        return ids, w, None, k, seed, (f"config4: {n or 1e8:.3g} (u64 id, f32 weight) Zipf(1.1) stream pairs over 1e7 "
                                       "keys, key weights U(0.1,10), k=4096")
    if cfg == 5:
        ids, w, k, seed = workloads.config5(n=n or 10**9, lo=lo, hi=hi)
        return ids, w, None, k, seed, (f"config5: one vector of {n or 1e9:.3g} elements (u32 ids 0..n-1), "
                                       "f32 LogNormal(0,2), k=8192")
    if cfg == 2:
        ids, w, off, k, seed = workloads.config2()
        return ids, w, off, k, seed, "config2: 1000 vectors x 1000 ids over 1e6, fp32 Exp(1), k=1024, pairs (2i,2i+1)"
    ids, w, off, k, seed = workloads.config3()
    return ids, w, off, k, seed, "config3: 1e5 CSR vectors, n~LogNormal(6,1), fp32 Pareto(1.5), k=512"


def config_total(cfg: int, n: int = 0) -> int:
    return {4: n or 10**8, 5: n or 10**9}[cfg]


def digest_parity(cfg: int, y, s, full: bool) -> str:
    """The timed sketch(es) against the committed oracle digest of the full workload."""
    if not full:
        return "n/a (not the full workload)"
    try:
        with open(DIGESTS) as f:
            want = json.load(f)[f"config{cfg}"]["digest"]
    except (OSError, KeyError, ValueError):
        return "n/a (no committed digest)"
    from oracle import oracle as O

    got = O.digest(np.asarray(y), np.asarray(s).view(np.uint64))
    return "oracle digest ok" if got == want else f"MISMATCH (got {got[:16]}, want {want[:16]})"


# ---------------------------------------------------------------- measurement helpers
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


def hbm_peak():
    try:
        with open(MEASURED_PEAKS) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def evidence(cfg: int) -> dict:
    """ncu-derived per-launch figures committed under profiles/ for this
    config (DRAM traffic, instructions per arrival of the kernel and the
    probe); {} when absent."""
    path = os.path.join(ROOT, "profiles", f"evidence_config{cfg}.json")
    try:
        with open(path) as f:
            d = json.load(f)
        d["file"] = os.path.relpath(path, ROOT)
        return d
    except (OSError, ValueError):
        return {}


def probe_peak(dev, k: int, stream):
    """Arrivals/s of gm_probe_arrival_rate (the lane step's arithmetic at full
    occupancy, no pruning, tables or registers), best of 1/2/4 independent
    chains per thread, measured in this run."""
    import torch

    from paper_2302_05176_b200 import _device

    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    best, best_c = 0.0, 0
    for variant, chains in PROBE_VARIANTS.items():
        n_threads, iters = sms * 2048 // chains, 512
        arg = iters | (variant << 24)
        for _ in range(2):
            _device.call("gm_probe_arrival_rate", n_threads, arg, k, sink.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(5):
            _device.call("gm_probe_arrival_rate", n_threads, arg, k, sink.data_ptr(), stream.cuda_stream)
        a1.record(stream)
        torch.cuda.synchronize()
        rate = 5 * n_threads * chains * iters / (a0.elapsed_time(a1) / 1e3)
        if rate > best:
            best, best_c = rate, f"{chains} chain(s)/thread, {PROBE_OCC[variant]}"
    return best, best_c


def max_over_ranks(x: float, world: int, dev) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def base_line(args, world, value, step_ms, scaling, cfg_dict, k):
    return {"metric": "positive elements sketched/sec at k=%d" % k, "value": value, "unit": "elements/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, workloads.py)", "config": cfg_dict}


# ---------------------------------------------------------------- reference arm
def cpu_oracle_time(ids, w, off, k, seed, n_vec_sample, threads):
    """Time the C port of the reference's sketch_fast (oracle/) over the
    first n_vec_sample vectors on `threads` host threads; returns (seconds, elements)."""
    from oracle import oracle as O

    off_s = off[: n_vec_sample + 1]
    n = int(off_s[-1])
    ids64 = ids[:n].astype(np.uint64)
    w64 = w[:n].astype(np.float64)
    t0 = time.perf_counter()
    rc, _, _, _ = O.sketch_csr(ids64, w64, off_s, k, seed, mode=0, threads=threads)
    dt = time.perf_counter() - t0
    assert rc == 0
    return dt, n


def cpu_seeds_time(ids, w, k, seeds, threads):
    """The reference's sketch_fast of one vector under each of `seeds` (C port,
    a thread pool over seeds); returns seconds."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O

    order = np.argsort(ids, kind="stable")
    i64, w64 = ids[order].astype(np.uint64), w[order].astype(np.float64)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        rcs = list(ex.map(lambda sd: O.sketch_fast(i64, w64, k, sd)[0], seeds))
    assert all(rc == 0 for rc in rcs)
    return time.perf_counter() - t0


def cpu_stream_time(ids, w, k, seed, n_sample, threads):
    """Time the C port of the reference's sketch_stream (oracle/) over the
    first n_sample items, split into `threads` contiguous chunks sketched in
    parallel (ctypes releases the GIL) and merged (the partition law,
    estimate.py:103-125); returns seconds."""
    from oracle import oracle as O

    t0 = time.perf_counter()
    rc, _, _ = O.sketch_stream_chunked(ids[:n_sample], w[:n_sample], k, seed, threads=threads,
                                       chunk=max(1, -(-n_sample // threads)))
    assert rc == 0
    return time.perf_counter() - t0


def cpu_baseline_for(cfg, ids, w, off, k, seed, budget_s=12.0):
    """Bounded CPU sample of the same workload on all host threads:
    (elements/s, description)."""
    threads = os.cpu_count() or 1
    if cfg == 1:
        probe = cpu_seeds_time(ids, w, k, list(range(1, threads + 1)), threads) / threads
        n_seeds = int(max(threads, min(CONFIG1_SEEDS, budget_s / max(probe, 1e-9))))
        dt = cpu_seeds_time(ids, w, k, list(range(1, n_seeds + 1)), threads)
        return n_seeds * ids.size / dt, threads, (f"seeds 1..{n_seeds} of {CONFIG1_SEEDS} ({n_seeds * ids.size} elements), "
                                                  "oracle/gm_oracle.c sketch_fast, a thread per seed")
    if off is not None:
        n_vec = off.size - 1
        dt_probe, _ = cpu_oracle_time(ids, w, off, k, seed, min(n_vec, 64), threads)
        n_sample = int(min(n_vec, max(threads, budget_s / max(dt_probe / 64, 1e-9))))
        dt, n = cpu_oracle_time(ids, w, off, k, seed, n_sample, threads)
        return n / dt, threads, (f"first {n_sample} of {n_vec} config-{cfg} vectors ({n} elements), "
                                 "oracle/gm_oracle.c sketch_fast, all host threads")
    n_all = ids.size
    probe = min(n_all, 200_000)
    per_item = cpu_stream_time(ids, w, k, seed, probe, threads) / probe
    n_sample = int(min(n_all, max(probe, budget_s / max(per_item, 1e-12))))
    dt = cpu_stream_time(ids, w, k, seed, n_sample, threads)
    return n_sample / dt, threads, (f"first {n_sample} of {n_all} items, oracle/gm_oracle.c sketch_stream in "
                                    f"{threads} chunks + merge")


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm on the host CPU, rank 0 only."""
    if rank != 0:
        return
    cfg = args.config
    ids, w, off, k, seed, desc = load_workload(cfg, int(args.n))
    threads = os.cpu_count() or 1
    per_step_budget = max(1.0, 8.0 / max(1, args.steps + args.warmup))
    if cfg == 1:
        probe = cpu_seeds_time(ids, w, k, list(range(1, threads + 1)), threads) / threads
        n_seeds = int(max(threads, min(CONFIG1_SEEDS, per_step_budget / max(probe, 1e-9))))
        seeds = list(range(1, n_seeds + 1))
        for _ in range(args.warmup):
            cpu_seeds_time(ids, w, k, seeds, threads)
        total = sum(cpu_seeds_time(ids, w, k, seeds, threads) for _ in range(args.steps))
        elems = n_seeds * ids.size
        sample = f"seeds 1..{n_seeds} of {CONFIG1_SEEDS} per step ({elems} elements), sketch_fast C port, a thread per seed"
        scaling = "weak"
    elif off is not None:
        n_vec = off.size - 1
        probe_dt, _ = cpu_oracle_time(ids, w, off, k, seed, min(n_vec, 64), threads)
        n_sample = int(min(n_vec, max(threads, per_step_budget / max(probe_dt / 64, 1e-9))))
        for _ in range(args.warmup):
            cpu_oracle_time(ids, w, off, k, seed, n_sample, threads)
        times = []
        for _ in range(args.steps):
            dt, elems = cpu_oracle_time(ids, w, off, k, seed, n_sample, threads)
            times.append(dt)
        total = sum(times)
        sample = (f"first {n_sample} of {n_vec} vectors per step ({elems} elements), oracle/gm_oracle.c sketch_fast "
                  "(bit-exact C port of sketch.py:218-311)")
        scaling = "weak" if cfg == 2 else "strong"
    else:
        n = ids.size
        probe = min(n, 200_000)
        per_item = cpu_stream_time(ids, w, k, seed, probe, threads) / probe
        elems = int(min(n, max(probe, per_step_budget / max(per_item, 1e-12))))
        for _ in range(args.warmup):
            cpu_stream_time(ids, w, k, seed, elems, threads)
        total = sum(cpu_stream_time(ids, w, k, seed, elems, threads) for _ in range(args.steps))
        sample = (f"first {elems} of {n} items per step, oracle/gm_oracle.c sketch_stream (bit-exact C port of "
                  f"stream.py:58-153) in {threads} chunks + merge")
        scaling = "strong"
    value = elems * args.steps / total
    line = base_line(args, world, value, 1e3 * total / args.steps, scaling,
                     {"workload": desc, "parallelism": f"host threads x{threads}"}, k)
    line.update({"impl": "reference",
                 "cpu_baseline": {"value": value, "unit": "elements/s", "cores": threads, "kind": "port",
                                  "sample": sample},
                 "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- configs 1-3: K1 (csr4_kernel)
def csr_roofline(dev, stream, k, achieved_arrivals_per_s, alg_arrivals, executed, kernel_ms, in_bytes, out_bytes,
                 cfg):
    peak, chains = probe_peak(dev, k, stream)
    hbm, hbm_kind = hbm_peak()
    ev = evidence(cfg)
    hbm_achieved = (in_bytes + out_bytes) / (kernel_ms / 1e3) / 1e9
    roof = {"bound": "compute (exact fp64 arrival generation)", "unit": "arrivals/s",
            "achieved": achieved_arrivals_per_s, "peak": peak, "frac": achieved_arrivals_per_s / peak,
            "traffic": ev.get("dram_bytes_per_launch"),
            "peak_source": (f"gm_probe_arrival_rate in this run: the lane step's own arithmetic (hash, glibc-clone "
                            f"log, rounded product, branch-free divide, Barrett draw) at full occupancy, "
                            f"{chains}, no pruning/tables/registers"),
            "algorithmic_arrivals_per_launch": alg_arrivals, "executed_arrivals_per_launch": executed,
            "hbm": {"achieved_gbs": hbm_achieved, "peak_gbs": hbm, "peak_kind": hbm_kind, "frac": hbm_achieved / hbm}}
    for key in ("kernel_warp_inst_per_arrival", "probe_warp_inst_per_arrival", "probe_pipes", "kernel_pipes",
                "source"):
        if key in ev:
            roof[key] = ev[key]
    if ev:
        roof["evidence"] = ev["file"]
    return roof


def algorithmic_arrivals(dev, stream, ids_t, id_bits, w_t, w_bits, off_t, n_vec, k, seed, y):
    """n+ + #arrivals <= each vector's final max register: the minimum any
    exact threshold walk must emit (gm_count_arrivals_csr)."""
    import torch

    from paper_2302_05176_b200 import _device

    tau = y.max(dim=1).values.contiguous()
    counts = torch.zeros(n_vec, dtype=torch.int64, device=dev)
    _device.call("gm_count_arrivals_csr", ids_t.data_ptr(), id_bits, w_t.data_ptr(), w_bits, off_t.data_ptr(), n_vec,
                 k, seed, tau.data_ptr(), counts.data_ptr(), stream.cuda_stream)
    off = off_t.cpu().numpy()
    return int(off[-1] - off[0]) + int(counts.sum().item())


def run_config1(args, rank, world, local_rank):
    """One vector (config 1) under R seeds per step: R independent sketches in
    one launch (gm_sketch_csr_seeded, GM_FLAG_ONE_VECTOR); N > 1 runs replicas
    (every rank its own R seeds).  L2 is flushed between steps (the vector is
    120 KB: an L2-resident input is its natural state inside one launch)."""
    import torch
    import torch.distributed as dist

    import paper_2302_05176_b200 as gm
    from paper_2302_05176_b200 import _device, _lib

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L = _lib.load()
    ids, w, off, k, seed, desc = load_workload(1)
    R = CONFIG1_SEEDS
    seeds_np = np.arange(1, R + 1, dtype=np.uint64) + np.uint64(rank * R)
    d_ids = torch.from_numpy(ids.view(np.int32)).to(dev)
    d_w = torch.from_numpy(w).to(dev)
    d_off = torch.from_numpy(off).to(dev)
    d_seeds = torch.from_numpy(seeds_np.view(np.int64)).to(dev)
    y = torch.empty((R, k), dtype=torch.float64, device=dev)
    s = torch.empty((R, k), dtype=torch.int64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    salt = gm.SeedScheme(1).stream_salt

    def step():
        rc = L.gm_sketch_csr_seeded(d_ids.data_ptr(), 32, d_w.data_ptr(), 64, d_off.data_ptr(), R, k,
                                    d_seeds.data_ptr(), salt, _lib.GM_FLAG_ASYNC | _lib.GM_FLAG_ONE_VECTOR,
                                    y.data_ptr(), s.data_ptr(), None, sp)
        if rc:
            raise RuntimeError(_lib.last_error())

    for _ in range(max(3, args.warmup)):
        step()
    _device.call("gm_stream_status", sp)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clocks:
        for a0, a1 in ev:
            flush.zero_()
            a0.record(stream)
            step()
            a1.record(stream)
        torch.cuda.synchronize()
    _device.call("gm_stream_status", sp)
    step_ms = max_over_ranks(sum(a0.elapsed_time(a1) for a0, a1 in ev) / args.steps, world, dev)
    value = world * R * ids.size / (step_ms / 1e3)

    # parity: every sketch of the batch against the oracle's for rank 0's first seeds
    from oracle import oracle as O

    yc, sc_ = y.cpu().numpy(), s.cpu().numpy().view(np.uint64)
    order = np.argsort(ids, kind="stable")
    bad = 0
    for r in range(0, R, max(1, R // 16)):
        rc, yo, so, _ = O.sketch_fast(ids[order].astype(np.uint64), w[order], k, int(seeds_np[r]))
        bad += int(rc != 0 or yo.tobytes() != yc[r].tobytes() or not np.array_equal(so, sc_[r]))
    parity = "oracle ok (16 of the batch's sketches, bit-exact)" if bad == 0 else f"MISMATCH in {bad} sketches"

    # end to end: host buffers every step -- the vector and the seeds copied in
    # (pinned), the R sketches' registers copied out, wall clock
    h_ids = torch.from_numpy(ids.view(np.int32)).pin_memory()
    h_w = torch.from_numpy(w).pin_memory()
    h_seeds = torch.from_numpy(seeds_np.view(np.int64)).pin_memory()
    h_y = torch.empty((R, k), dtype=torch.float64).pin_memory()
    h_s = torch.empty((R, k), dtype=torch.int64).pin_memory()

    def e2e_step():
        d_ids.copy_(h_ids, non_blocking=True)
        d_w.copy_(h_w, non_blocking=True)
        d_seeds.copy_(h_seeds, non_blocking=True)
        step()
        h_y.copy_(y, non_blocking=True)
        h_s.copy_(s, non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(1e3 * (time.perf_counter() - t0) / args.steps, world, dev)
    _device.call("gm_stream_status", sp)

    # single-sketch latency through the host entry (one vector >= 4096
    # elements runs on the grid-wide kernels)
    hy = np.empty((1, k), np.float64)
    hs = np.empty((1, k), np.uint64)
    lat = []
    for i in range(12):
        t0 = time.perf_counter()
        _device.call("gm_sketch_csr_host", ids.ctypes.data, 32, w.ctypes.data, 64, off.ctypes.data, 1, k, seed,
                     salt, 0, hy.ctypes.data, hs.ctypes.data, None, sp)
        lat.append(1e3 * (time.perf_counter() - t0))
    one_ms = statistics.median(lat[2:])
    rc, yo, so, _ = O.sketch_fast(ids[order].astype(np.uint64), w[order], k, seed)
    one_ok = rc == 0 and yo.tobytes() == hy[0].tobytes() and np.array_equal(so, hs[0])
    if rank != 0:
        return

    # roofline: algorithmic arrivals of 16 of the seeds, scaled to R
    cnt = []
    for r in range(0, R, max(1, R // 16)):
        tau = torch.from_numpy(yc[r:r + 1].max(axis=1)).to(dev)
        c = torch.zeros(1, dtype=torch.int64, device=dev)
        _device.call("gm_count_arrivals_csr", d_ids.data_ptr(), 32, d_w.data_ptr(), 64, d_off.data_ptr(), 1, k,
                     int(seeds_np[r]), tau.data_ptr(), c.data_ptr(), sp)
        cnt.append(ids.size + int(c.item()))
    alg = float(np.mean(cnt)) * R
    em = torch.empty(R, dtype=torch.int64, device=dev)
    L.gm_sketch_csr_seeded(d_ids.data_ptr(), 32, d_w.data_ptr(), 64, d_off.data_ptr(), R, k, d_seeds.data_ptr(), salt,
                           _lib.GM_FLAG_ONE_VECTOR, y.data_ptr(), s.data_ptr(), em.data_ptr(), sp)
    executed = int(em.sum().item())
    roof = csr_roofline(dev, stream, k, alg / (step_ms / 1e3), alg, executed, step_ms, ids.nbytes + w.nbytes,
                        R * k * 16, 1)
    roof["algorithmic_arrivals_note"] = "mean over 16 of the R seeds x R"
    cfg = {"workload": desc, "sketches_per_step_per_gpu": R, "elements_per_step_per_gpu": R * ids.size, "k": k,
           "parallelism": f"replicas x{world} (every rank its own {R} seeds)" if world > 1 else "single GPU",
           "l2": "L2 flushed between steps (512 MB write, outside the per-step CUDA events)",
           "single_sketch_latency_ms": one_ms,
           "single_sketch_note": ("one sketch of the vector through gm_sketch_csr_host (host buffers in and out, "
                                  "grid-wide kernels), wall clock, median of 10"),
           "single_sketch_parity": "oracle ok (bit-exact)" if one_ok else "MISMATCH"}
    line = base_line(args, world, value, step_ms, "weak", cfg, k)
    line.update({
        "parity": parity,
        "e2e": {"value": world * R * ids.size / (e2e_ms / 1e3), "unit": "elements/s",
                "h2d_bytes_per_step": ids.nbytes + w.nbytes + seeds_np.nbytes, "d2h_bytes_per_step": R * k * 16,
                "ms_per_step": e2e_ms,
                "api": "pinned host vector + seeds copied in, gm_sketch_csr_seeded, registers (f64 y + u64 s) out"},
        "gpu_launches": args.steps, "roofline": roof, "clocks": clocks.summary()})
    if not args.no_cpu_baseline:
        v, cores, sample = cpu_baseline_for(1, ids, w, off, k, seed)
        line["cpu_baseline"] = {"value": v, "unit": "elements/s", "cores": cores, "kind": "port", "sample": sample}
    print(json.dumps(line), flush=True)


def run_csr(args, rank, world, local_rank):
    """Configs 2-3: batched CSR sketches (csr4_kernel)."""
    import torch
    import torch.distributed as dist

    import paper_2302_05176_b200 as gm
    from paper_2302_05176_b200 import _device, _lib, shard

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L = _lib.load()
    cfg_n = args.config
    ids, w, off, k, seed, desc = load_workload(cfg_n)
    scheme = gm.SeedScheme(seed)
    # config 2: weak scaling, every rank sketches a full batch of its own (at N=1
    # this is the config); config 3: strong scaling, the 1e5 vectors are split
    # into contiguous ranges balanced by element count (shard.vector_ranges),
    # no collective on the data path
    n_all = int(off[-1])
    strong = cfg_n == 3 and world > 1
    if strong:
        v0, v1 = shard.vector_ranges(off, world)[rank]
        lo_e, hi_e = int(off[v0]), int(off[v1])
        ids, w, off = ids[lo_e:hi_e], w[lo_e:hi_e], off[v0:v1 + 1] - lo_e
    n_vec = off.size - 1
    n_el = int(off[-1])
    n_job = n_all if strong else n_el * world  # elements the whole job sketches per step
    # Batches stream through `--streams` CUDA streams in turn, so one batch's
    # first CTAs and input copy overlap the previous batch's tail (a batch ends
    # with a ramp-down in which most SMs are idle).  Inputs
    # rotate over resident copies (> L2), so no batch finds its input in L2.
    n_copies = N_COPIES if cfg_n == 2 else 1  # config 3's input alone (532 MB) exceeds L2
    ns = args.streams
    d_ids_c = [torch.from_numpy(ids.view(np.int32)).to(dev) for _ in range(n_copies)]
    d_w_c = [torch.from_numpy(w).to(dev) for _ in range(n_copies)]
    d_ids, d_w = d_ids_c[0], d_w_c[0]
    d_off = torch.from_numpy(off).to(dev)
    pool = _device.stream_pool(dev, ns)
    ys = [torch.empty((n_vec, k), dtype=torch.float64, device=dev) for _ in range(ns)]
    ss = [torch.empty((n_vec, k), dtype=torch.int64, device=dev) for _ in range(ns)]
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def step(i, st=None):
        rc = L.gm_sketch_csr(d_ids_c[i % n_copies].data_ptr(), 32, d_w_c[i % n_copies].data_ptr(), 32,
                             d_off.data_ptr(), n_vec, k, scheme.global_seed, scheme.stream_salt, _lib.GM_FLAG_ASYNC,
                             ys[i % ns].data_ptr(), ss[i % ns].data_ptr(), None,
                             pool[i % ns].cuda_stream if st is None else st)
        if rc:
            raise RuntimeError(_lib.last_error())

    def status_all():
        for st_ in pool + [stream]:
            _device.call("gm_stream_status", st_.cuda_stream)

    def pipelined(fn):
        """device time of args.steps calls of fn(i) over the streams, barrier and sync on both sides"""
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(pool[0])
        for st_ in pool[1:]:
            st_.wait_event(start)
        for i in range(args.steps):
            fn(i)
        for st_ in pool[1:]:
            e = torch.cuda.Event()
            e.record(st_)
            pool[0].wait_event(e)
        end.record(pool[0])
        torch.cuda.synchronize()
        return start.elapsed_time(end)

    for i in range(max(3, args.warmup) * ns):
        step(i)
    status_all()
    with ClockSampler(local_rank) as clocks:
        total_ms = pipelined(step)
    status_all()
    total_ms = max_over_ranks(total_ms, world, dev)
    if world > 1:
        dist.barrier()
    step_ms = total_ms / args.steps
    value = n_job * args.steps / (total_ms / 1e3)
    y, s = ys[(args.steps - 1) % ns], ss[(args.steps - 1) % ns]
    parity = digest_parity(cfg_n, y.cpu().numpy(), s.cpu().numpy(), full=not strong)

    # one batch alone on an idle GPU (L2 flushed first): the latency figure
    lat = []
    for i in range(max(5, min(args.steps, 20))):
        flush.zero_()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        step(i, sp)
        a1.record(stream)
        torch.cuda.synchronize()
        lat.append(a0.elapsed_time(a1))
    status_all()
    batch_ms = statistics.median(lat)

    # ---- end to end through the public C-ABI with pinned host buffers: every
    # step copies its inputs in and its registers out, same stream rotation,
    # wall clock
    h_ids = torch.from_numpy(ids.view(np.int32)).pin_memory()
    h_w = torch.from_numpy(w).pin_memory()
    h_off = torch.from_numpy(off).pin_memory()
    h_y = [torch.empty((n_vec, k), dtype=torch.float64).pin_memory() for _ in range(ns)]
    h_s = [torch.empty((n_vec, k), dtype=torch.int32).pin_memory() for _ in range(ns)]  # GM_FLAG_S32: u32 ids

    def e2e_step(i):
        rc = L.gm_sketch_csr_host(h_ids.data_ptr(), 32, h_w.data_ptr(), 32, h_off.data_ptr(), n_vec, k,
                                  scheme.global_seed, scheme.stream_salt, _lib.GM_FLAG_ASYNC | _lib.GM_FLAG_S32,
                                  h_y[i % ns].data_ptr(), h_s[i % ns].data_ptr(), None, pool[i % ns].cuda_stream)
        if rc:
            raise RuntimeError(_lib.last_error())

    for i in range(max(3, args.warmup) * ns):
        e2e_step(i)
    torch.cuda.synchronize()
    status_all()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        e2e_step(i)
    for st_ in pool:
        st_.synchronize()
    e2e_total = max_over_ranks(1e3 * (time.perf_counter() - t0), world, dev)
    status_all()
    e2e_value = n_job * args.steps / (e2e_total / 1e3)
    h2d = ids.nbytes + w.nbytes + off.nbytes
    d2h = n_vec * k * 12  # y f64 + s u32
    j = (args.steps - 1) % ns
    e2e_parity = digest_parity(cfg_n, h_y[j].numpy(), h_s[j].numpy().view(np.uint32).astype(np.uint64),
                               full=not strong)
    if rank != 0:
        return

    alg = algorithmic_arrivals(dev, stream, d_ids, 32, d_w, 32, d_off, n_vec, k, scheme.global_seed, y)
    emitted = torch.empty(n_vec, dtype=torch.int64, device=dev)
    L.gm_sketch_csr(d_ids.data_ptr(), 32, d_w.data_ptr(), 32, d_off.data_ptr(), n_vec, k, scheme.global_seed,
                    scheme.stream_salt, 0, y.data_ptr(), s.data_ptr(), emitted.data_ptr(), sp)
    executed = int(emitted.sum().item())
    roof = csr_roofline(dev, stream, k, alg / (step_ms / 1e3), alg, executed, step_ms,
                        ids.nbytes + w.nbytes + off.nbytes, n_vec * k * 16, cfg_n)
    cfg = {"workload": desc, "elements_per_step_per_gpu": n_el, "k": k,
           "parallelism": (f"vector shards x{world} balanced by elements" if strong else
                           f"a full batch per rank x{world} (replicas)") if world > 1 else "single GPU",
           "batches": f"a stream of batches over {ns} CUDA streams (consecutive batches overlap)",
           "l2": (f"inputs rotated over {n_copies} resident copies ({n_copies * (ids.nbytes + w.nbytes) >> 20} MiB "
                  "> 126 MB L2)"),
           "batch_latency_ms": batch_ms,
           "batch_latency_note": "one batch alone on an idle GPU, L2 flushed first (median)"}
    line = base_line(args, world, value, step_ms, "strong" if strong else "weak", cfg, k)
    line.update({
        "parity": parity,
        "e2e": {"value": e2e_value, "unit": "elements/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_total / args.steps, "parity": e2e_parity,
                "api": f"gm_sketch_csr_host (pinned host buffers, GM_FLAG_ASYNC | GM_FLAG_S32 over {ns} streams), "
                       "wall clock"},
        "gpu_launches": args.steps,  # per step: one csr4_kernel (the slots compute the weight sums themselves)
        "roofline": roof, "clocks": clocks.summary()})
    if not args.no_cpu_baseline and world == 1:
        v, cores, sample = cpu_baseline_for(cfg_n, ids, w, off, k, seed)
        line["cpu_baseline"] = {"value": v, "unit": "elements/s", "cores": cores, "kind": "port", "sample": sample}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- configs 4-5: K2 (element sets)
def run_elements(args, rank, world, local_rank):
    """Configs 4-5: one sketch of a huge element set per step.  N > 1:
    contiguous element shards (every rank generates only its own), a sketch
    per rank, then one exchange of the k registers over NCCL inside the C ABI
    -- strong scaling, the whole job's elements per step are fixed."""
    import torch
    import torch.distributed as dist

    import paper_2302_05176_b200 as gm
    from paper_2302_05176_b200 import _device, _lib, shard

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L = _lib.load()
    n_all = config_total(args.config, int(args.n))
    lo, hi = shard.element_range(n_all, world, rank)
    ids, w, _, k, seed, desc = load_workload(args.config, int(args.n), lo, hi)
    scheme = gm.SeedScheme(seed)
    id_bits = ids.dtype.itemsize * 8
    n = hi - lo
    d_ids = torch.from_numpy(ids.view(np.int64 if id_bits == 64 else np.int32)).to(dev)
    d_w = torch.from_numpy(w).to(dev)
    y = torch.empty(k, dtype=torch.float64, device=dev)
    s = torch.empty(k, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    xchg = shard.RegisterExchange() if world > 1 else None

    def exchange(yy, ss_):
        if xchg is None:
            return yy, ss_
        return xchg.allreduce_min(yy, ss_) if args.merge == "allreduce" else xchg.allgather_merge(yy, ss_)

    # A stream of sketches: every step enqueues one pass at the list bound
    # (gm_sketch_elements_async, no host synchronisation between sketches) and
    # writes its unset-register count to the device; after the K steps the
    # counts are read and any incomplete sketch is finished synchronously
    # (GM_FLAG_ACCUMULATE) inside the timed region.  At N = 1 the sketches
    # rotate over --elem-streams CUDA streams (each with its own workspace), so
    # one sketch's latency-bound list walk overlaps the next one's filter; at
    # N > 1 one stream carries the sketches and the register exchanges.
    ns_e = max(1, args.elem_streams) if world == 1 else 1
    estreams = [stream] + _device.stream_pool(dev, ns_e - 1) if ns_e > 1 else [stream]
    outs = [(y, s)] + [(torch.empty_like(y), torch.empty_like(s)) for _ in range(ns_e - 1)]
    n_warm = max(3, args.warmup, 2 * ns_e)  # every stream's workspace is created and grown before timing
    unset = torch.zeros(max(args.steps, n_warm), dtype=torch.int32, device=dev)
    redone = [0]

    def step(i):
        st_, (yy, ss_) = estreams[i % ns_e], outs[i % ns_e]
        rc = L.gm_sketch_elements_async(d_ids.data_ptr(), id_bits, d_w.data_ptr(), 32, n, k, scheme.global_seed,
                                        scheme.stream_salt, 0, yy.data_ptr(), ss_.data_ptr(),
                                        unset[i].data_ptr(), st_.cuda_stream)
        if rc:
            raise RuntimeError(_lib.last_error())
        return yy, ss_

    def finish(steps):
        """join the streams, read the unset counts; complete a sketch that needs it"""
        for st_ in estreams[1:]:
            e = torch.cuda.Event()
            e.record(st_)
            stream.wait_event(e)
        cnt = unset[:steps].cpu().numpy()  # a copy, no kernel
        for j in np.nonzero(cnt > 0)[0]:
            redone[0] += 1
            yy, ss_ = outs[int(j) % ns_e]
            rc = L.gm_sketch_elements(d_ids.data_ptr(), id_bits, d_w.data_ptr(), 32, n, k, scheme.global_seed,
                                      scheme.stream_salt, _lib.GM_FLAG_ACCUMULATE, yy.data_ptr(), ss_.data_ptr(), None,
                                      sp)
            if rc:
                raise RuntimeError(_lib.last_error())
        for st_ in estreams:
            _device.call("gm_stream_status", st_.cuda_stream)

    for i in range(n_warm):
        exchange(*step(i))
    finish(n_warm)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    redone[0] = 0
    with ClockSampler(local_rank) as clocks:
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for st_ in estreams[1:]:
            st_.wait_event(a0)
        # the sketches (one pass each, no host sync); at N > 1 each followed by its exchange
        last = None
        for i in range(args.steps):
            last = exchange(*step(i)) if world > 1 else step(i)
        finish(args.steps)
        if world > 1:
            # every rank knows whether any rank re-ran a pass (an all-reduce of
            # the count): then the completed registers are exchanged once more
            rr = torch.tensor([redone[0]], dtype=torch.int32, device=dev)
            dist.all_reduce(rr)
            if int(rr.item()):
                last = exchange(*outs[0])
        a1.record(stream)
        torch.cuda.synchronize()
    step_ms = max_over_ranks(a0.elapsed_time(a1), world, dev) / args.steps
    value = n_all / (step_ms / 1e3)
    yo, so = last
    parity = digest_parity(args.config, yo.cpu().numpy(), so.cpu().numpy(), full=not args.n)

    # one sketch alone through the synchronous call (its latency, reported beside the stream figure)
    lat = []
    for _ in range(5):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        rc = L.gm_sketch_elements(d_ids.data_ptr(), id_bits, d_w.data_ptr(), 32, n, k, scheme.global_seed,
                                  scheme.stream_salt, 0, y.data_ptr(), s.data_ptr(), None, sp)
        if rc:
            raise RuntimeError(_lib.last_error())
        exchange(y, s)
        a1.record(stream)
        torch.cuda.synchronize()
        lat.append(a0.elapsed_time(a1))
    sketch_ms = max_over_ranks(statistics.median(lat), world, dev)

    # end to end: host buffers through gm_sketch_elements_host (every step copies
    # the shard in and the k registers out), exchanged across ranks
    h_ids = torch.from_numpy(ids.view(np.int64 if id_bits == 64 else np.int32)).pin_memory()
    h_w = torch.from_numpy(w).pin_memory()
    h_y = torch.empty(k, dtype=torch.float64).pin_memory()
    h_s = torch.empty(k, dtype=torch.int64).pin_memory()

    def e2e_step():
        rc = L.gm_sketch_elements_host(h_ids.data_ptr(), id_bits, h_w.data_ptr(), 32, n, k, scheme.global_seed,
                                       scheme.stream_salt, 0, h_y.data_ptr(), h_s.data_ptr(), None, sp)
        if rc:
            raise RuntimeError(_lib.last_error())
        if world > 1:
            y.copy_(h_y, non_blocking=True)
            s.copy_(h_s, non_blocking=True)
            exchange(y, s)
            h_y.copy_(y, non_blocking=True)
            h_s.copy_(s, non_blocking=True)
            torch.cuda.synchronize()

    e2e_steps = max(1, min(args.steps, 5))
    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(1e3 * (time.perf_counter() - t0) / e2e_steps, world, dev)
    e2e_parity = digest_parity(args.config, h_y.numpy(), h_s.numpy(), full=not args.n)
    if xchg is not None:
        xchg.close()
    if rank != 0:
        return
    hbm, hbm_kind = hbm_peak()
    in_bytes = n * (ids.itemsize + w.itemsize)  # this rank's shard
    achieved = in_bytes / (step_ms / 1e3) / 1e9
    ev = evidence(args.config)
    line = base_line(args, world, value, step_ms, "strong", {
        "workload": desc, "elements_per_step": n_all, "k": k,
        "parallelism": (f"element shards x{world} (each rank generates its own) + NCCL " +
                        ("MIN all-reduces (gm_allreduce_min_registers)" if args.merge == "allreduce"
                         else "all-gather + device merge (gm_allgather_merge_registers)")) if world > 1
        else "single GPU",
        "l2": f"inputs ({(ids.nbytes + w.nbytes) >> 20} MiB per rank) larger than the 126 MB L2",
        "schedule": (f"a stream of one-pass sketches over {ns_e} CUDA stream(s) (gm_sketch_elements_async, no host "
                     f"sync between them); incomplete ones finished synchronously in the timed region "
                     f"({redone[0]} needed it)"),
        "sketch_latency_ms": sketch_ms,
        "sketch_latency_note": "one sketch alone through the synchronous gm_sketch_elements (+ exchange), median of 5"},
        k)
    line.update({
        "parity": parity,
        "e2e": {"value": n_all / (e2e_ms / 1e3), "unit": "elements/s", "h2d_bytes_per_step": in_bytes,
                "d2h_bytes_per_step": 16 * k, "ms_per_step": e2e_ms, "parity": e2e_parity,
                "api": "gm_sketch_elements_host (pinned host buffers), wall clock"},
        "gpu_launches": 4 * args.steps + (args.steps if world > 1 else 0),
        "gpu_launches_note": ("per sketch: weight sample (+ register init, tau), filter, survivor walk, heavy walk "
                              "(+ register store) -- and the merge / mask kernel of the exchange for N > 1 -- when "
                              "the first walk completes every register"),
        "roofline": {"bound": "hbm", "unit": "GB/s", "achieved": achieved, "peak": hbm, "frac": achieved / hbm,
                     "traffic": ev.get("dram_bytes_per_launch"), "peak_kind": hbm_kind,
                     "achieved_note": "input bytes (ids + weights) per sketch / whole sketch step (all its kernels)",
                     **({"evidence": ev["file"]} if ev else {})},
        "clocks": clocks.summary()})
    if not args.no_cpu_baseline and world == 1:
        v, cores, sample = cpu_baseline_for(args.config, ids, w, None, k, seed)
        line["cpu_baseline"] = {"value": v, "unit": "elements/s", "cores": cores, "kind": "port", "sample": sample}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    maybe_spawn(args)
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
    if args.config == 1:
        run_config1(args, rank, world, local_rank)
    elif args.config in (4, 5):
        run_elements(args, rank, world, local_rank)
    else:
        run_csr(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
