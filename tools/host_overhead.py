"""Host cost of one sellkit_spmv call (Python binding + C ABI + launch) on the C1 matrix
(5-pt 1000^2, w = 1), asynchronous mode: enqueue time per call and back-to-back time per
call (GPU-bound when larger).  Measured on B200: 8.6 us enqueue, 12.3 us per call with the
operands L2-resident."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1507_08101_b200 import sellkit
sk = sellkit.load()
A = sk.crs_stencil(5, 1000).build(32, 1)
x, y = sk.densemat(10**6, 1), sk.densemat(10**6, 1)
x.fill_hash(1)
sk.set_sync(False)
for _ in range(20): sk.spmv(y, A, x)
sk.synchronize()
for n in (1000,):
    t = time.perf_counter()
    for _ in range(n): sk.spmv(y, A, x)
    t1 = time.perf_counter()
    sk.synchronize()
    t2 = time.perf_counter()
    print(f"enqueue {1e6*(t1-t)/n:.1f} us/call, total {1e6*(t2-t)/n:.1f} us/call")
