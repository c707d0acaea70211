#!/usr/bin/env python3
"""Summarise an `ncu --csv --log-file X` launch list: per kernel name, launch
count and mean of each metric.   python tools/ncu_table.py X.csv"""
import collections
import csv
import sys


def main(path):
    with open(path) as f:
        rows = [r for r in csv.reader(line for line in f if not line.startswith("=="))]
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    acc = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) != len(h) or not r[vi]:
            continue
        name = r[ki].split("(")[0][:70]
        d = acc.setdefault(name, collections.defaultdict(list))
        d[(r[mi], r[ui])].append(float(r[vi].replace(",", "")))
    for name, d in acc.items():
        n = max(len(v) for v in d.values())
        cols = "  ".join(f"{m}={sum(v) / len(v):.4g} {u}" for (m, u), v in d.items())
        print(f"{name:70s} x{n:<4d} {cols}")


if __name__ == "__main__":
    main(sys.argv[1])
