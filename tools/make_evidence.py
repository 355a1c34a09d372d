"""Join an ncu metrics capture of tools/ncu_target.py with its work counts
into profiles/evidence_configN.json (read by bench.py for the roofline block).

  python tools/make_evidence.py --config N --csv gpurun_out/evidence_cN.csv \
      --target gpurun_out/target_configN.json [--tag r02]

Per kernel (last launch of each name): duration, warp instructions, pipe
utilisation (fp64, fma, alu, xu: % of peak sustained while active), issue
slots busy, SIMT efficiency, DRAM bytes; for configs 1-3 warp instructions
per arrival of the K1 kernel (algorithmic and executed) and of the probe."""

import argparse
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PIPES = {"fp64": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
         "fma": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
         "alu": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
         "xu": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
         "lsu": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
         "issue_active": "smsp__issue_active.avg.pct_of_peak_sustained_active",
         "warps_active": "sm__warps_active.avg.pct_of_peak_sustained_active"}


def load(path):
    hdr, rows = None, {}
    for r in csv.reader(open(path)):
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = rows.setdefault(d["ID"], {"name": d["Kernel Name"]})
            try:
                e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
            except ValueError:
                pass
    return list(rows.values())


def short(name):
    return name.split("(")[0].replace("void ", "").replace("gmk::", "")


def summary(e):
    out = {"duration_us": e.get("gpu__time_duration.sum", 0.0) / 1e3,
           "warp_inst": e.get("smsp__inst_executed.sum"),
           "simt_threads_per_inst": e.get("smsp__thread_inst_executed_per_inst_executed.ratio"),
           "dram_bytes": (e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0)),
           "pipes_pct": {k: e.get(v) for k, v in PIPES.items()}}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--csv", required=True)
    ap.add_argument("--target", required=True)
    ap.add_argument("--tag", default="r02")
    a = ap.parse_args()
    tgt = json.load(open(a.target))
    launches = load(a.csv)
    last = {}
    for e in launches:
        last[short(e["name"])] = e
    ev = {"source": f"ncu --metrics (tools/ncu_target.py --config {a.config}; {os.path.basename(a.csv)}), "
                    f"{a.tag}: per launch, the last launch of each kernel", "kernels": {}}
    for name, e in last.items():
        ev["kernels"][name] = summary(e)
    # the probe: best rate chain count, warp instructions per arrival
    best = None
    for name, e in last.items():
        if name.startswith("arrival_probe_kernel"):
            arr = tgt["probe_arrivals_per_launch"].get(name)
            if arr:
                rate = arr / (e["gpu__time_duration.sum"] / 1e9)
                ev["kernels"][name]["arrivals"] = arr
                ev["kernels"][name]["arrivals_per_s"] = rate
                ev["kernels"][name]["warp_inst_per_arrival"] = e["smsp__inst_executed.sum"] / arr
                if best is None or rate > best[0]:
                    best = (rate, name)
    if best:
        p = ev["kernels"][best[1]]
        ev["probe_kernel"] = best[1]
        ev["probe_warp_inst_per_arrival"] = p["warp_inst_per_arrival"]
        ev["probe_pipes"] = p["pipes_pct"]
    csr = [n for n in last if n.startswith("csr3_kernel") or n.startswith("csr4_kernel")]
    # the uncounted instantiation (kCount = 0: what bench.py times) before the counted one
    csr.sort(key=lambda n: not n.rstrip().endswith(", 0>"))
    if csr:
        e = ev["kernels"][csr[0]]
        ev["kernel"] = csr[0]
        ev["kernel_pipes"] = e["pipes_pct"]
        ev["dram_bytes_per_launch"] = e["dram_bytes"]
        if "algorithmic_arrivals_per_launch" in tgt:
            ev["kernel_warp_inst_per_arrival"] = {
                "algorithmic": e["warp_inst"] / tgt["algorithmic_arrivals_per_launch"],
                "executed": e["warp_inst"] / tgt["executed_arrivals_per_launch"]}
            ev["algorithmic_arrivals_per_launch"] = tgt["algorithmic_arrivals_per_launch"]
            ev["executed_arrivals_per_launch"] = tgt["executed_arrivals_per_launch"]
    filt = [n for n in last if n.startswith("elem_filter_kernel")]
    if filt:
        e = ev["kernels"][filt[0]]
        ev["kernel"] = filt[0]
        ev["dram_bytes_per_launch"] = e["dram_bytes"]
        ev["kernel_pipes"] = e["pipes_pct"]
        if "input_bytes" in tgt:
            ev["input_bytes"] = tgt["input_bytes"]
    out = os.path.join(ROOT, "profiles", f"evidence_config{a.config}.json")
    with open(out, "w") as f:
        json.dump(ev, f, indent=1, sort_keys=True)
    print(out)


if __name__ == "__main__":
    main()
