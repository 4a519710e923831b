#!/usr/bin/env python
"""Construction cost of the C5 matrix (400^3 7-pt, SELL-32-256) in SpMV units, repeated:
build / update_values wall times of consecutive calls in one process."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1507_08101_b200 import sellkit  # noqa: E402

sk = sellkit.load()
crs = sk.crs_stencil(7, 400)
torch.cuda.synchronize()
res = []
for rep in range(4):
    t0 = time.perf_counter()
    A = crs.build(32, 256)
    tb = time.perf_counter() - t0
    t0 = time.perf_counter()
    sk.call("sellkit_mat_update_values", A.h, crs.h)
    tu = time.perf_counter() - t0
    res.append({"rep": rep, "build_ms": tb * 1e3, "update_ms": tu * 1e3})
    if rep < 3:
        del A
print(json.dumps(res))
