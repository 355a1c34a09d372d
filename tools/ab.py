"""A/B tuning builds of the library.

Local (build container):  python tools/ab.py build NAME -DX=1 ...   -> gpu_scratch/lib_NAME.so
GPU box:                  python tools/ab.py run --configs 2,3 --reps 2 NAME...
   (bench.py per variant and config with GM_LIB_PATH; 'base' = the in-tree build;
    variants interleaved rep by rep; one summary line each to stdout)"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCR = os.path.join(ROOT, "gpu_scratch")


def lib(name):
    return os.path.join(ROOT, "paper_2302_05176_b200", "libgmsketch_b200.so") if name == "base" else \
        os.path.join(SCR, f"lib_{name}.so")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["build", "run"])
    ap.add_argument("names", nargs="+")
    ap.add_argument("--configs", default="2")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--steps", type=int, default=20)
    a, extra = ap.parse_known_args()
    if a.mode == "build":
        sys.path.insert(0, ROOT)
        from paper_2302_05176_b200 import build
        os.makedirs(SCR, exist_ok=True)
        defs = [d[2:] for d in extra if d.startswith("-D")]
        print(build.build(out=lib(a.names[0]), defines=defs))
        return
    for rep in range(a.reps):
        for cfg in a.configs.split(","):
            for name in a.names:
                env = dict(os.environ, GM_LIB_PATH=lib(name))
                r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps",
                                    str(a.steps), "--warmup", "3", "--no-cpu-baseline"], env=env,
                                   capture_output=True, text=True)
                line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
                if not line:
                    print(f"rep {rep} config {cfg} {name}: FAILED rc={r.returncode} {r.stderr[-400:]}", flush=True)
                    continue
                d = json.loads(line[-1])
                print(f"rep {rep} config {cfg} {name:10s} {d['ms_per_step']:.4f} ms  frac "
                      f"{d.get('roofline', {}).get('frac', 0):.3f}  parity {d.get('parity')}", flush=True)


if __name__ == "__main__":
    main()
