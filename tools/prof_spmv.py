#!/usr/bin/env python
"""Small driver for ncu / microbenchmarks of the SpMMV kernel.

    python tools/prof_spmv.py --n 400 --w 8 --reps 3 [--flags 0] [--C 32 --sigma 256]
Prints per-launch CUDA-event times (ms) and GB/s of algorithmic traffic.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1507_08101_b200 import sellkit  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=400)
p.add_argument("--w", type=int, nargs="+", default=[8])
p.add_argument("--C", type=int, default=32)
p.add_argument("--sigma", type=int, default=256)
p.add_argument("--reps", type=int, default=3)
p.add_argument("--flags", type=int, default=0)
a = p.parse_args()

sk = sellkit.load()
N = a.n ** 3
nnz = 7 * a.n ** 3 - 6 * a.n ** 2
A = sk.crs_stencil(7, a.n).build(a.C, a.sigma)
stream = torch.cuda.ExternalStream(sk.stream())
for w in a.w:
    x = sk.densemat(N, w)
    x.fill_hash(42)
    y = sk.densemat(N, w)
    dots = np.zeros(3 * w)
    sk.set_sync(False)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.reps + 1)]
    sk.spmv(y, A, x, flags=a.flags, dot=dots if a.flags & 0x38 else None)
    ev[0].record(stream)
    for i in range(a.reps):
        sk.spmv(y, A, x, flags=a.flags, dot=dots if a.flags & 0x38 else None)
        ev[i + 1].record(stream)
    sk.synchronize()
    sk.set_sync(True)
    ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(a.reps)]
    alg = 12.0 * nnz + 16.0 * w * N
    t = float(np.median(ts))
    print(f"n={a.n} w={w} C={a.C} sigma={a.sigma}: {t:.3f} ms  {alg / t / 1e6:.0f} GB/s  "
          f"{2 * nnz * w / t / 1e6:.0f} GF/s  (min {min(ts):.3f})", flush=True)
    del x, y
