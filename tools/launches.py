"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, mean, total."""
import csv
import re
import sys
from collections import OrderedDict


def summarise(path):
    rows = list(csv.reader([l for l in open(path) if not l.startswith("==")]))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    d = OrderedDict()
    for r in rows[1:]:
        name = re.sub(r"usk::(<unnamed>|\(anonymous namespace\))::", "", r[ki])
        name = re.split(r"[<(]", name)[0]
        d.setdefault(name, []).append(float(r[vi].replace(",", "")) / (1000.0 if r[ui] == "ns" else 1.0))
    return d


if __name__ == "__main__":
    d = summarise(sys.argv[1])
    tot = sum(sum(v) for v in d.values())
    print(f"{'kernel':36s} {'n':>4s} {'mean_us':>10s} {'total_us':>10s} {'share':>6s}")
    for k, v in d.items():
        print(f"{k:36s} {len(v):4d} {sum(v)/len(v):10.2f} {sum(v):10.2f} {sum(v)/tot:6.1%}")
