"""Summarise ncu launch lists (--metrics gpu__time_duration.sum --csv): per kernel, count and mean us.

usage: python tools/kt_summary.py FILE.csv..."""
import collections
import csv
import sys

for fn in sys.argv[1:]:
    lines = open(fn).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    d = collections.defaultdict(list)
    for r in csv.DictReader(lines[start:]):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v if unit == "us" else v / 1e3
        d[r["Kernel Name"].split("(")[0][-70:]].append(us)
    print("==", fn)
    for k, v in d.items():
        print(f"  {k:70s} n={len(v):3d} mean={sum(v)/len(v):10.1f} us  last={v[-1]:10.1f} us")
