"""Group the SASS of one kernel (ncu --page source --print-source sass --csv)
into runs of equal execution count and show the source lines of each run,
heaviest first.   python tools/sass_blocks.py <sass.csv> <kernel-substring> [N]"""
import collections
import csv
import sys

sys.path.insert(0, __import__("os").path.dirname(__file__))
from sass_profile import lineinfo  # noqa: E402


def main():
    path, kname = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ie = hdr.index("Instructions Executed")
    data = [(int(r[0], 16), r[1].strip(), int(float(r[ie] or 0))) for r in rows[2:] if len(r) > ie and r[0].startswith("0x")]
    base = data[0][0]
    li = lineinfo(kname)
    tot = sum(d[2] for d in data)
    runs = []
    cur = None
    for a, src, n in data:
        if cur and cur["n"] == n and a == cur["end"] + 16:
            cur["end"] = a
            cur["len"] += 1
            cur["lines"].append(li.get(a - base, (None, ""))[0])
        else:
            cur = {"start": a, "end": a, "n": n, "len": 1, "lines": [li.get(a - base, (None, ""))[0]]}
            runs.append(cur)
    runs.sort(key=lambda r: -r["n"] * r["len"])
    for r in runs[:top]:
        c = collections.Counter(f"{x[0][:8]}:{x[1]}" for x in r["lines"] if x)
        print(f"{100 * r['n'] * r['len'] / tot:5.1f}%  {r['n']:>9,d} x {r['len']:4d}  @{r['start'] - base:#07x}  "
              + " ".join(f"{k}({v})" for k, v in c.most_common(5)))


if __name__ == "__main__":
    main()
