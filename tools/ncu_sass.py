"""List the SASS of an ncu source page (cuda,sass csv) in address order with
warp instructions executed, active threads per instruction, stall samples
and the CUDA source line each belongs to.

  python tools/ncu_sass.py src.csv [min_count] > sass.txt
"""
import csv
import sys


def main(path, min_count=0):
    rows = list(csv.reader(open(path)))
    cur_file, cur_line, hdr = None, None, None
    out = []
    for r in rows:
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        if r[0]:
            cur_line = r[0]
            continue
        d = dict(zip(hdr[2:], r[2:]))
        try:
            addr = int(r[2], 16)
        except ValueError:
            continue

        def f(k):
            try:
                return float(d.get(k, "0") or 0)
            except ValueError:
                return 0.0
        ie = f("Instructions Executed")
        te = f("Thread Instructions Executed")
        out.append((addr, ie, te / ie if ie else 0.0, f"{cur_file}:{cur_line}", r[3].strip(),
                    f("Warp Stall Sampling (All Samples)")))
    out.sort()
    base = out[0][0] if out else 0
    for a, ie, thr, src, sass, st in out:
        if ie >= float(min_count):
            print(f"{a - base:06x} {ie:10.0f} {thr:5.1f} {st:7.0f} {src:26s} {sass}")


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3]))
