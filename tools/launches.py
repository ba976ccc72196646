"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys


def summary(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0][:60]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                 "ms": 1e3}.get(d["Metric Unit"], 1.0)
        agg.setdefault(k, []).append(float(d["Metric Value"].replace(",", "")) * scale)
    return agg


if __name__ == "__main__":
    for k, v in summary(sys.argv[1]).items():
        print(f"{len(v):4d} {sum(v) / len(v):10.1f} us  {k}")
