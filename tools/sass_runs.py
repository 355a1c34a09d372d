"""Top SASS runs (equal execution count, contiguous) of a kernel from an ncu
SASS source page: share of warp instructions, executions x length, average
active threads, source lines.
  python tools/sass_runs.py <sass.csv> <mangled-kernel-prefix> [N]"""
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sass_profile import lineinfo  # noqa: E402


def main():
    path, kname = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    li = lineinfo(kname)
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ie, te = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
    data = [r for r in rows[2:] if len(r) > te and r[0].startswith("0x")]
    base = int(data[0][0], 16)
    runs, cur = [], None
    for r in data:
        a = int(r[0], 16) - base
        w, t = int(float(r[ie] or 0)), float(r[te] or 0)
        src = li.get(a, ((None, 0), ""))[0] or (None, 0)
        if cur and cur["w"] == w and a == cur["end"] + 16:
            cur["end"], cur["n"], cur["t"] = a, cur["n"] + 1, cur["t"] + t
            cur["lines"].add(src)
        else:
            if cur:
                runs.append(cur)
            cur = {"start": a, "end": a, "w": w, "n": 1, "t": t, "lines": {src}}
    runs.append(cur)
    tot = sum(x["w"] * x["n"] for x in runs)
    print(f"total warp instructions {tot:.4g}")
    for x in sorted(runs, key=lambda x: -x["w"] * x["n"])[:top]:
        act = x["t"] / max(1, x["w"] * x["n"])
        ls = sorted(f"{f[:8]}:{l}" for f, l in x["lines"] if f)[:6]
        print(f"{x['w'] * x['n'] / tot * 100:5.1f}% {x['w']:8d}x{x['n']:4d} active {act:5.1f} @{x['start']:#07x} {' '.join(ls)}")


if __name__ == "__main__":
    main()
