"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel name, count and mean/last duration (cold-cache, serialised)."""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "second": 1e6, "s": 1e6}
    for d in data:
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        agg.setdefault(d["Kernel Name"][:70], []).append(v)
    for k, v in agg.items():
        print(f"{k:70s} n={len(v):4d} mean={sum(v)/len(v):10.1f}us last={v[-1]:10.1f}us")


if __name__ == "__main__":
    main()
