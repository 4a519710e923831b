#!/usr/bin/env python
"""Table of an A/B jsonl (tools/ab_*.sh): min over rounds of the median ms per (case, lib)."""
import collections
import json
import sys

res = collections.defaultdict(list)
libs = []
for line in open(sys.argv[1]):
    d = json.loads(line)
    lib = d.get("lib", d.get("order"))
    if lib not in libs:
        libs.append(lib)
    res[(d["case"], lib)].append((d["ms"], d["frac"]))
cases = sorted({k[0] for k in res})
print("case".ljust(44), *[lb[:12].rjust(14) for lb in libs])
for c in cases:
    cells = []
    for lb in libs:
        v = res.get((c, lb))
        cells.append(("%.3f (%.2f)" % min(v)).rjust(14) if v else "-".rjust(14))
    print(c[:44].ljust(44), *cells)
