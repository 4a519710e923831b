#!/usr/bin/env python
"""C4 shapes: TSMM (beta = 0) and TSMTTSM at N = 1e8 for the given m = k; median CUDA-event
time of 5 reps, fraction of the measured HBM peak (8 N (m + k) bytes).
    python tools/tsm_case.py 1 2 8 32"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1507_08101_b200 import sellkit  # noqa: E402

sk = sellkit.load()
stream = torch.cuda.ExternalStream(sk.stream())
PEAK = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
N = 100_000_000
one, zero = np.array([1.0]), np.array([0.0])


def timed(fn, reps=5):
    sk.set_sync(False)
    fn()
    sk.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        sk.synchronize()
        ts.append(e0.elapsed_time(e1))
    sk.set_sync(True)
    return float(np.median(ts))


for m in [int(a) for a in sys.argv[1:]]:
    V, W, X = sk.densemat(N, m), sk.densemat(N, m), sk.densemat(m, m)
    V.fill_hash(1)
    W.fill_hash(2)
    X.fill_hash(3)
    alg = 8.0 * N * 2 * m
    for name, fn in [("tsmm", lambda: sk.call("sellkit_tsmm", W, V, X, one.ctypes.data, zero.ctypes.data)),
                     ("tsmttsm", lambda: sk.call("sellkit_tsmttsm", X, V, W, one.ctypes.data, zero.ctypes.data, 0))]:
        ms = timed(fn)
        print(json.dumps({"case": f"c4 {name} N=1e8 m=k={m}", "ms": ms, "gbs": alg / ms / 1e6,
                          "frac": alg / ms / 1e6 / PEAK}), flush=True)
    del V, W, X
