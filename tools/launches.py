"""Summarise an ncu --csv launch list (gpu__time_duration.sum and optional
dram bytes): one row per launch, or totals per kernel with --sum.

  python tools/launches.py file.csv [--sum] [--last N]"""
import collections
import csv
import sys


def load(path):
    hdr, by = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = by.setdefault(d["ID"], {"name": d["Kernel Name"]})
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return list(by.values())


def short(name):
    name = name.split("(")[0]
    return name.replace("void ", "").replace("gmk::", "")[:60]


if __name__ == "__main__":
    items = load(sys.argv[1])
    if "--last" in sys.argv:
        items = items[-int(sys.argv[sys.argv.index("--last") + 1]):]
    if "--sum" in sys.argv:
        agg = collections.OrderedDict()
        for it in items:
            a = agg.setdefault(short(it["name"]), [0, 0.0])
            a[0] += 1
            a[1] += it.get("gpu__time_duration.sum", 0.0)
        for k, (n, t) in agg.items():
            print(f"{k:60s} {n:5d} {t / 1e3:10.1f} us  {t / n / 1e3:9.1f} us/launch")
    else:
        for it in items:
            rd = it.get("dram__bytes_read.sum")
            wr = it.get("dram__bytes_write.sum")
            extra = f" {rd / 1e6:9.1f} MB rd {wr / 1e6:8.1f} MB wr" if rd is not None else ""
            print(f"{short(it['name']):60s} {it.get('gpu__time_duration.sum', 0) / 1e3:9.1f} us{extra}")
