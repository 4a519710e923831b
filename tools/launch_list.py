#!/usr/bin/env python
"""Median gpu__time_duration per kernel from an ncu --csv launch list: launch_list.py FILE.csv"""
import csv
import sys
from collections import defaultdict

t = defaultdict(list)
h = None
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            t[d["Kernel Name"][:90]].append(float(d["Metric Value"]) / 1e3)
for k, v in t.items():
    v.sort()
    print(f"{len(v):4d} {v[len(v) // 2]:10.2f} us  {k}")
