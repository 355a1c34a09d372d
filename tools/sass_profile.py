"""Join an ncu SASS source page (--print-source sass --csv) with nvdisasm -g
line info of the built library: dynamic instruction counts per source line
range of one kernel.

  python tools/sass_profile.py <sass.csv> <kernel-substring> [file:lo-hi ...]
"""
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def lineinfo(kname):
    so = os.path.join(ROOT, "paper_2302_05176_b200", "libgmsketch_b200.so")
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=d, capture_output=True)
        txt = ""
        for cub in sorted(f for f in os.listdir(d) if f.endswith(".cubin")):  # the cubin holding the kernel
            t = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
            if any(ln.startswith(".text.") and kname in ln for ln in t.splitlines()):
                txt = t
                break
    lines = txt.splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith(".text.") and kname in ln)
    cur = None
    out = {}
    for ln in lines[start + 1:]:
        if ln.startswith(".text."):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            out[int(m.group(1), 16)] = (cur, m.group(2))
    return out


def main():
    path, kname = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ie = hdr.index("Instructions Executed")
    te = hdr.index("Thread Instructions Executed")
    data = []
    for r in rows[2:]:
        if len(r) <= ie or not r[0].startswith("0x"):
            continue
        data.append((int(r[0], 16), r[1].strip(), float(r[ie] or 0), float(r[te] or 0)))
    base = data[0][0]
    li = lineinfo(kname)
    tot = sum(d[2] for d in data)
    print(f"total warp instructions {tot:.4g}")
    ranges = [a for a in sys.argv[3:]]
    for rg in ranges:
        fname, span = rg.split(":")
        lo, hi = map(int, span.split("-"))
        s = t = 0.0
        for a, src, n, th in data:
            c = li.get(a - base, (None, ""))[0]
            if c and c[0] == fname and lo <= c[1] <= hi:
                s += n
                t += th
        print(f"  {rg:28s} {100 * s / tot:5.1f}%  thr/inst {t / max(s, 1):5.1f}")
    # hottest SASS lines
    print("top instructions:")
    for a, src, n, th in sorted(data, key=lambda x: -x[2])[:40]:
        c = li.get(a - base, (None, ""))[0]
        print(f"  {n:12.0f} thr {th / max(n, 1):4.1f} {c[0] if c else ''}:{c[1] if c else ''} {src[:70]}")


if __name__ == "__main__":
    main()
