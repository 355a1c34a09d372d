"""Summarise an ncu source page by CUDA source line: stall samples and warp
instructions executed, top-N.

  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
  python tools/ncu_lines.py src.csv [N]
"""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur_file = None
    hdr = None
    agg = []
    for r in rows:
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        try:
            line = int(r[0])
        except ValueError:
            continue
        d = dict(zip(hdr[4:], r[4:]))

        def num(key):
            try:
                return float(d.get(key, "0") or 0)
            except ValueError:
                return 0.0
        ie = num("Instructions Executed")
        agg.append((num("Warp Stall Sampling (All Samples)"), ie,
                    num("Thread Instructions Executed") / ie if ie else 0.0, cur_file, line, r[1][:90]))
    tot_s = sum(a[0] for a in agg) or 1
    tot_i = sum(a[1] for a in agg) or 1
    print(f"total stall samples {tot_s:.0f}, warp instructions {tot_i:.3e}")
    for a in sorted(agg, reverse=True)[:top]:
        print(f"{100*a[0]/tot_s:5.1f}% stall {100*a[1]/tot_i:5.1f}% inst thr={a[2]:4.1f} {a[3]}:{a[4]}  {a[5]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
