"""Time the reference single-process distributed API (sellkit_dist_spmv) with k ranks
on the visible GPU(s): python tools/dist_prof.py [n] [k] [w]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1507_08101_b200 import sellkit  # noqa: E402
from paper_1507_08101_b200.dist import DistContext  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = int(sys.argv[3]) if len(sys.argv) > 3 else 8
sk = sellkit.load()
crs = sk.crs_stencil(7, n)
ctx = DistContext(sk, crs, k, 32, 256)
x, y = ctx.vec(w), ctx.vec(w)
xg = sk.densemat(n ** 3, w)
xg.fill_hash(42)
ctx.scatter(xg, x)
for _ in range(3):
    ctx.spmv(y, x)
torch.cuda.synchronize()
reps = 20
t0 = time.perf_counter()
for _ in range(reps):
    ctx.spmv(y, x)
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) / reps * 1e3
nnz = 7 * n ** 3 - 6 * n ** 2
print(f"dist_spmv n={n} k={k} w={w}: {ms:.3f} ms/call  {2 * nnz * w / ms / 1e6:.0f} GF/s")
