"""Build libgmsketch_b200.so in-tree for sm_100a (nvcc -shared)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libgmsketch_b200.so")
SOURCES = [os.path.join(CSRC, "gm_capi.cu"), os.path.join(CSRC, "gm_exact.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("gm_core.cuh", "gm_walk.cuh", "gm_kernels.cuh", "gm_csr.cuh", "gm_csr4.cuh",
                                                  "gm_pairs.cuh", "gm_comm.cuh", "gm_glibc_log.cuh", "gm_glibc_logtab.h")] + [
    os.path.join(os.path.dirname(HERE), "include", "gmsketch_b200.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-shared", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.exists(cand) or cand == "nvcc"):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build the library (to `out` with extra -D `defines` for tuning and
    instrumented builds; the product build takes neither)."""
    if out is None and not defines and not force and up_to_date():
        return OUT
    out = out or OUT
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", out, *SOURCES, "-lcudart", "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libgmsketch_b200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
