"""TSMTTSM / TSMM timing over (m, k) shapes, N rows: python tools/tsm_shapes.py [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1507_08101_b200 import sellkit  # noqa: E402

sk = sellkit.load()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
stream = torch.cuda.ExternalStream(sk.stream())
one, zero = np.array([1.0]), np.array([0.0])
out = []
for m, k in [(1, 8), (8, 1), (2, 4), (4, 2), (2, 8), (8, 2), (4, 4), (4, 8), (8, 4)]:
    V, W, X = sk.densemat(N, m), sk.densemat(N, k), sk.densemat(m, k)
    V.fill_hash(1)
    W.fill_hash(2)
    sk.set_sync(False)
    ts = []
    for r in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sk.call("sellkit_tsmttsm", X, V, W, one.ctypes.data, zero.ctypes.data, 0)
        e1.record(stream)
        sk.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    sk.set_sync(True)
    out.append(f"{m}x{k}:{np.median(ts):.3f}")
    del V, W, X
print(" ".join(out))
