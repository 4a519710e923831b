#!/usr/bin/env python
"""C3: the augmented KPM step on the synthetic TI Hamiltonian (2^24 rows, w = 16),
y = 2a(H - bI)x - y with <y,y>, <x,y>, <x,x> (a = 0.25, b = 0.25).

    python tools/c3_step.py [--dt c64|r64] [--order rows|pencil16|auto] [--reps 20] [--warm 3]

Prints one JSON line (median CUDA-event time over reps, algorithmic GB/s and the
fraction of the measured HBM peak).  Short and fixed, so it is also the command to
wrap in ncu (-k regex:spmv_tma_rows -s <warm> -c 1)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1507_08101_b200 import sellkit  # noqa: E402
from paper_1507_08101_b200.orders import pencil_order  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--dt", default="c64", choices=["c64", "r64"])
p.add_argument("--order", default="rows")
p.add_argument("--reps", type=int, default=20)
p.add_argument("--warm", type=int, default=3)
p.add_argument("--flags", default="kpm", choices=["kpm", "plain", "axpby"])
p.add_argument("--w", type=int, default=16)
a = p.parse_args()

sk = sellkit.load()
stream = torch.cuda.ExternalStream(sk.stream())
PEAK = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
lx, ly, lz, w = 256, 128, 128, a.w
N = 4 * lx * ly * lz
dt = sellkit.C64 if a.dt == "c64" else sellkit.R64
vb = 16 if dt == sellkit.C64 else 8
A = sk.crs_ti(lx, ly, lz, 1.0, dt=dt).build(32, 256)
_, _, nnz = A.dims()
if a.order.startswith("pencil"):
    A.set_sweep_order(256, pencil_order(lx, ly, lz, per_site=4, block_rows=256, yb=int(a.order[6:] or 16)))
x, y = sk.densemat(N, w, dt), sk.densemat(N, w, dt)
x.fill_hash(42)
y.fill_hash(43)
dots = torch.zeros(3 * w * (2 if dt == sellkit.C64 else 1), dtype=torch.float64, device="cuda")
flags = {"kpm": sellkit.AXPBY | sellkit.SHIFT | sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX,
         "plain": 0, "axpby": sellkit.AXPBY}[a.flags]
o = sellkit.spmv_opts()
sk.lib.sellkit_spmv_opts_init(sellkit.C.byref(o))
keep = []


def sc(v):
    arr = np.array([v], sellkit.NP_DTYPE[dt])
    keep.append(arr)
    return arr.ctypes.data_as(sellkit.vp)


o.flags = flags
if flags:
    o.alpha, o.beta, o.gamma = sc(0.5), sc(-1.0), sc(0.25)
o.dot = sellkit.vp(dots.data_ptr())


def fn():
    sk.call("sellkit_spmv", y.h, A.h, x.h, sellkit.C.byref(o))


sk.set_sync(False)
for _ in range(a.warm):
    fn()
sk.synchronize()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn()
    e1.record(stream)
    sk.synchronize()
    ts.append(e0.elapsed_time(e1))
sk.set_sync(True)
ms = float(np.median(ts))
nvec = 2 + (1 if flags & sellkit.AXPBY else 0)
alg = (vb + 4.0) * nnz + vb * w * N * nvec
fl = (8.0 if dt == sellkit.C64 else 2.0) * nnz * w
print(json.dumps({"case": f"c3 TI 2^24 rows w={w} {a.dt} {a.flags}", "order": a.order, "ms": ms, "min_ms": min(ts),
                  "gflops": fl / ms / 1e6, "gbs": alg / ms / 1e6, "frac": alg / ms / 1e6 / PEAK, "nnz": nnz}),
      flush=True)
