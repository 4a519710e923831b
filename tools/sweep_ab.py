#!/usr/bin/env python
"""A/B of sweep orders on the headline 7-point stencil (SpMMV, y = A x).

    python tools/sweep_ab.py --n 400 --w 8 --reps 200 --lines 8 16
Alternates the natural row order with slab ("pencil") orders whose blocks are
`lines` x-lines; prints CUDA-event medians and checks y is bit-identical."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1507_08101_b200 import sellkit  # noqa: E402
from paper_1507_08101_b200.orders import pencil_order  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=400)
p.add_argument("--w", type=int, default=8)
p.add_argument("--reps", type=int, default=200)
p.add_argument("--rounds", type=int, default=3)
p.add_argument("--lines", type=int, nargs="+", default=[8, 16])
a = p.parse_args()

sk = sellkit.load()
n = a.n
N = n ** 3
nnz = 7 * n ** 3 - 6 * n ** 2
A = sk.crs_stencil(7, n).build(32, 256)
stream = torch.cuda.ExternalStream(sk.stream())
x = sk.densemat(N, a.w)
x.fill_hash(42)
y = sk.densemat(N, a.w)
alg = 12.0 * nnz + 16.0 * a.w * N


def run(label):
    sk.set_sync(False)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.reps + 1)]
    sk.spmv(y, A, x)
    ev[0].record(stream)
    for i in range(a.reps):
        sk.spmv(y, A, x)
        ev[i + 1].record(stream)
    sk.synchronize()
    sk.set_sync(True)
    ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(a.reps)]
    t = float(np.median(ts))
    print(f"{label}: {t:.3f} ms  {alg / t / 1e6:.0f} GB/s  (min {min(ts):.3f})", flush=True)


orders = {"rows": None}
for ln in a.lines:
    br = ln * n
    orders[f"slab{ln}"] = (br, pencil_order(br, n // ln, n, block_rows=br, yb=1))
ref = None
for r in range(a.rounds):
    for name, o in orders.items():
        if o is None:
            A.set_sweep_order(0, None)
        else:
            A.set_sweep_order(*o)
        run(f"r{r} {name}")
        if r == 0:
            yv = y.copy_out()
            if yv is not None:
                if ref is None:
                    ref = yv.copy()
                else:
                    print(f"  y bit-identical to row order: {np.array_equal(ref.view(np.uint64), yv.view(np.uint64))}")
