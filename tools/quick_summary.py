"""Summarise a gpu_scratch/quick.sh run: bench line + evidence counters."""
import json
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "q"
d = json.loads(open(f"gpurun_out/{tag}_c2.json").read().strip().splitlines()[-1])
r = d["roofline"]
print(f"c2 {d['ms_per_step']:.4f} ms/step  value {d['value']:.3g}  e2e {d['e2e']['value']:.3g}  lat {d['config']['batch_latency_ms']:.3f}"
      f"  frac {r['frac']:.3f} peak {r['peak']:.3g} exec {r['executed_arrivals_per_launch']} parity {d.get('parity')}")
subprocess.run([sys.executable, "tools/make_evidence.py", "--config", "2", "--csv", f"gpurun_out/{tag}_ev_c2.csv",
                "--target", f"gpurun_out/{tag}_target_c2.json", "--tag", tag], check=True, capture_output=True)
e = json.load(open("profiles/evidence_config2.json"))
for n, k in e["kernels"].items():
    p = k["pipes_pct"]
    print(f"  {n[:44]:44s} {k['duration_us']:8.1f} us inst {k['warp_inst']:.3g} simt {k['simt_threads_per_inst']:.1f} "
          f"issue {p['issue_active']:.1f} warps {p['warps_active']:.1f} fp64 {p['fp64']:.1f} "
          f"arr/s {k.get('arrivals_per_s', 0):.3g} inst/arr {k.get('warp_inst_per_arrival', 0):.2f}")
print("  K1 inst/arrival", e.get("kernel_warp_inst_per_arrival"))
