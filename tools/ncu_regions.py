"""Aggregate an ncu source page (cuda,sass csv) by file and by line ranges."""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    cur = None
    hdr = None
    out = []
    for r in rows:
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            cur = r[1].split("/")[-1]
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

        def f(k):
            try:
                return float(d.get(k, "0") or 0)
            except ValueError:
                return 0.0
        out.append((cur, line, f("Instructions Executed"), f("Warp Stall Sampling (All Samples)"),
                    f("Thread Instructions Executed"), r[1]))
    return out


def main(path, *ranges):
    rows = load(path)
    ti = sum(r[2] for r in rows) or 1
    ts = sum(r[3] for r in rows) or 1
    byf = {}
    for r in rows:
        a = byf.setdefault(r[0], [0, 0, 0])
        a[0] += r[2]
        a[1] += r[3]
        a[2] += r[4]
    print(f"total warp inst {ti:.4g}")
    for f_, a in sorted(byf.items(), key=lambda x: -x[1][0]):
        print(f"  {f_:34s} inst {100*a[0]/ti:5.1f}%  stall {100*a[1]/ts:5.1f}%  thr/inst {a[2]/max(a[0],1):5.1f}")
    for rg in ranges:
        fname, span = rg.split(":")
        lo, hi = map(int, span.split("-"))
        a = [0, 0, 0]
        for r in rows:
            if r[0] == fname and lo <= r[1] <= hi:
                a[0] += r[2]
                a[1] += r[3]
                a[2] += r[4]
        print(f"  {rg:34s} inst {100*a[0]/ti:5.1f}%  stall {100*a[1]/ts:5.1f}%  thr/inst {a[2]/max(a[0],1):5.1f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
