#!/usr/bin/env python
"""One SpMMV case on the 3-D 7-point stencil (or the 2-D 5-point one):

    python tools/stencil_step.py --n 400 --w 8 [--flags plain|axpby|dots|kpm] [--points 7]
        [--C 32 --sigma 256] [--reps 20] [--warm 3] [--flush]

Median CUDA-event time on the library stream, algorithmic GB/s and the fraction of the
measured HBM peak (one JSON line).  --flush writes 256 MB between reps (L2 flush)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1507_08101_b200 import sellkit  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=400)
p.add_argument("--w", type=int, default=8)
p.add_argument("--points", type=int, default=7)
p.add_argument("--C", type=int, default=32)
p.add_argument("--sigma", type=int, default=256)
p.add_argument("--flags", default="plain", choices=["plain", "axpby", "dots", "kpm"])
p.add_argument("--reps", type=int, default=20)
p.add_argument("--warm", type=int, default=3)
p.add_argument("--flush", action="store_true")
a = p.parse_args()

sk = sellkit.load()
stream = torch.cuda.ExternalStream(sk.stream())
PEAK = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
n, w = a.n, a.w
N = n ** 3 if a.points == 7 else n * n
A = sk.crs_stencil(a.points, n).build(a.C, a.sigma)
_, _, nnz = A.dims()
x, y = sk.densemat(N, w), sk.densemat(N, w)
x.fill_hash(42)
y.fill_hash(43)
dots = torch.zeros(3 * w, dtype=torch.float64, device="cuda")
DOTS = sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX
flags = {"plain": 0, "axpby": sellkit.AXPBY, "dots": DOTS, "kpm": sellkit.AXPBY | sellkit.SHIFT | DOTS}[a.flags]
o = sellkit.spmv_opts()
sk.lib.sellkit_spmv_opts_init(sellkit.C.byref(o))
keep = []


def sc(v):
    arr = np.array([v], np.float64)
    keep.append(arr)
    return arr.ctypes.data_as(sellkit.vp)


o.flags = flags
if flags & sellkit.AXPBY:
    o.alpha, o.beta, o.gamma = sc(0.5), sc(-1.0), sc(0.25)
o.dot = sellkit.vp(dots.data_ptr())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if a.flush else None


def fn():
    sk.call("sellkit_spmv", y.h, A.h, x.h, sellkit.C.byref(o))


sk.set_sync(False)
for _ in range(a.warm):
    fn()
sk.synchronize()
ts = []
for _ in range(a.reps):
    if flush is not None:
        with torch.cuda.stream(stream):
            flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn()
    e1.record(stream)
    sk.synchronize()
    ts.append(e0.elapsed_time(e1))
sk.set_sync(True)
ms = float(np.median(ts))
alg = 12.0 * nnz + 8.0 * w * N * (2 + (1 if flags & sellkit.AXPBY else 0))
print(json.dumps({"case": f"{a.points}pt n={n} SELL-{a.C}-{a.sigma} w={w} {a.flags}", "ms": ms, "min_ms": min(ts),
                  "gflops": 2.0 * nnz * w / ms / 1e6, "gbs": alg / ms / 1e6, "frac": alg / ms / 1e6 / PEAK,
                  "flushed": a.flush}), flush=True)
