#!/usr/bin/env python
"""Key metrics of an `ncu --page raw --csv` export (one line per kernel)."""
import csv
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from tools.ncu_summary import METRICS, SCALE  # noqa: E402

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    out = {"kernel": d.get("Kernel Name")}
    for m in METRICS:
        v = d.get(m)
        if v in (None, ""):
            continue
        try:
            out[m] = round(float(v.replace(",", "")) * SCALE.get(u.get(m, ""), 1), 6)
        except ValueError:
            out[m] = v
    print(json.dumps(out))
