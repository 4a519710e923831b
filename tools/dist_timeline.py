#!/usr/bin/env python
"""Timeline of the row-distributed SpMMV (single process, k ranks; on one GPU the ranks
share the device): per rank the halo exchange interval (communication stream: pack
kernels storing straight into the receivers' halo blocks) against the local and
remote sweeps (main stream), from the library's own timing events
(sellkit_ext_ctx_set_trace).  nsys is not available on this pool; this is its stand-in.

    python tools/dist_timeline.py [--n 400] [--w 8] [--k 2] [--reps 5]

Prints one JSON line per rank and repetition plus a summary: the exchange ends before
the local sweep does when the halo is hidden behind it."""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1507_08101_b200 import dist, sellkit  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=400)
p.add_argument("--w", type=int, default=8)
p.add_argument("--k", type=int, default=2)
p.add_argument("--reps", type=int, default=5)
a = p.parse_args()

sk = sellkit.load()
crs = sk.crs_stencil(7, a.n)
ctx = dist.DistContext(sk, crs, a.k, 32, 256, record=False)
del crs
N = a.n ** 3
x, y = ctx.vec(a.w), ctx.vec(a.w)
# x: hash-filled per part through a global vector would need 2 x N x w on the host; the
# timeline does not depend on the values, so the parts keep their zero initialisation
sk.call("sellkit_ext_ctx_set_trace", ctx.h, 1)
names = ["exchange_start", "exchange_end", "local_start", "local_end", "remote_end"]
rows = []
for rep in range(a.reps + 1):
    ctx.spmv(y, x)
    n = C.c_int(0)
    sk.call("sellkit_ext_ctx_timeline", ctx.h, None, C.byref(n))
    buf = (C.c_double * n.value)()
    sk.call("sellkit_ext_ctx_timeline", ctx.h, buf, C.byref(n))
    t = np.array(buf[:]).reshape(a.k, 5)
    if rep == 0:
        continue  # warm-up
    for r in range(a.k):
        rec = {"rep": rep, "rank": r, **{nm: round(float(v), 4) for nm, v in zip(names, t[r])}}
        rows.append(rec)
        print(json.dumps(rec))
hidden = [r["exchange_end"] <= r["local_end"] for r in rows]
print(json.dumps({"summary": f"k={a.k} n={a.n} w={a.w}", "exchange_hidden_in_local_sweep": all(hidden),
                  "exchange_ms_median": float(np.median([r["exchange_end"] - r["exchange_start"] for r in rows])),
                  "local_sweep_ms_median": float(np.median([r["local_end"] - r["local_start"] for r in rows])),
                  "remote_ms_median": float(np.median([r["remote_end"] - r["local_end"] for r in rows])),
                  "step_ms_median": float(np.median([max(r["remote_end"] for r in rows if r["rep"] == q)
                                                     for q in range(1, a.reps + 1)]))}))
