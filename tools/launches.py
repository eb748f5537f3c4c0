"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def short(name):
    name = name.replace("void ", "").replace("nesa::", "").replace("<unnamed>::", "")
    return name.split("(")[0][:60]


if __name__ == "__main__":
    data = load(sys.argv[1])
    last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    sel = data[-last:] if last else data
    agg = OrderedDict()
    tot = 0.0
    for d in sel:
        us = float(d["Metric Value"]) / 1e3
        k = short(d["Kernel Name"])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += us
        tot += us
    for k, (n, us) in agg.items():
        print(f"{us:9.1f} us  {n:4d}x  {100 * us / tot:5.1f}%  {k}")
    print(f"{tot:9.1f} us total ({len(sel)} launches)")
