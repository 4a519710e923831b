#!/usr/bin/env python
"""Secondary measurements (BASELINE.json configs other than the bench.py headline):

  c1   SpMV SELL-32-1, 2-D 5-point 1000^2, w = 1 (L2 flushed between reps)
  c2   SpMMV SELL-32-256, 3-D 7-point 256^3, w in {1, 4, 8, 16, 32} (+ AXPBY)
  c4   TSMM / TSMTTSM, N = 1e8, m = k in {1, 2, 4, 8, 16, 32, 64}

Device-resident inputs, CUDA events on the library stream, median of reps.
One JSON line per case on stdout.  Usage: python tools/bench_suite.py [c1] [c2] [c4]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1507_08101_b200 import sellkit  # noqa: E402
from paper_1507_08101_b200.orders import pencil_order  # noqa: E402

sk = sellkit.load()
stream = torch.cuda.ExternalStream(sk.stream())
PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
flush_buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10, warm=2, flush=False):
    sk.set_sync(False)
    for _ in range(warm):
        fn()
    sk.synchronize()
    ts = []
    for _ in range(reps):
        if flush:
            with torch.cuda.stream(stream):
                flush_buf.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        sk.synchronize()
        ts.append(e0.elapsed_time(e1))
    sk.set_sync(True)
    return float(np.median(ts))


def emit(**kw):
    print(json.dumps(kw), flush=True)


def spmv_case(tag, A, N, nnz, w, flags=0, flush=False, reps=10):
    x = sk.densemat(N, w)
    x.fill_hash(42)
    y = sk.densemat(N, w)
    if flags & sellkit.AXPBY:
        y.fill_hash(43)
    beta = np.array([0.5])

    def fn():
        if flags:
            sk.spmv(y, A, x, flags=flags, beta=beta)
        else:
            sk.spmv(y, A, x)
    ms = timed(fn, reps=reps, flush=flush)
    alg = 12.0 * nnz + 8.0 * w * N * (2 + (1 if flags & sellkit.AXPBY else 0))
    emit(case=tag, w=w, flags=flags, ms=ms, gflops=2.0 * nnz * w / ms / 1e6, gbs=alg / ms / 1e6,
         frac=alg / ms / 1e6 / PEAK, l2_flushed=flush)


def c1():
    n = 1000
    A = sk.crs_stencil(5, n).build(32, 1)
    spmv_case("c1 5pt 1000^2 SELL-32-1", A, n * n, 5 * n * n - 4 * n, 1, flush=True, reps=30)
    # the same event bracket around a one-element kernel: the launch floor inside the C1 number
    one = torch.empty(1, device="cuda")

    def tiny():
        with torch.cuda.stream(stream):
            one.zero_()
    emit(case="c1 launch floor (1-element kernel after the flush)", ms=timed(tiny, reps=30, flush=True))


def c2():
    n = 256
    A = sk.crs_stencil(7, n).build(32, 256)
    nnz = 7 * n ** 3 - 6 * n ** 2
    for w in (1, 4, 8, 16, 32):
        spmv_case("c2 7pt 256^3 SELL-32-256", A, n ** 3, nnz, w)
    spmv_case("c2 7pt 256^3 SELL-32-256", A, n ** 3, nnz, 8, flags=sellkit.AXPBY)


def c3():
    """Augmented KPM step on the synthetic TI Hamiltonian, 2^24 rows, w = 16:
    y = 2a(H - bI)x - y with <y,y>, <x,y>, <x,x> (a = 0.25, b = 0.25); C64 and the
    real-valued surrogate with the same pattern."""
    lx, ly, lz = 256, 128, 128
    N = 4 * lx * ly * lz
    for dt, vb in ((sellkit.C64, 16), (sellkit.R64, 8)):
        A = sk.crs_ti(lx, ly, lz, 1.0, dt=dt).build(32, 256)
        nnz = 13 * N
        w = 16
        x, y = sk.densemat(N, w, dt), sk.densemat(N, w, dt)
        x.fill_hash(42)
        y.fill_hash(43)
        dots = np.zeros(3 * w, sellkit.NP_DTYPE[dt])
        flags = sellkit.AXPBY | sellkit.SHIFT | sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX

        def fn():
            sk.spmv(y, A, x, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, dot=dots)
        alg = (vb + 4.0) * nnz + vb * w * N * 3  # x read, y read + write
        fl = (8.0 if dt == sellkit.C64 else 2.0) * nnz * w
        # natural row order, then a pencil sweep order (orders.py: z-reuse window of yb x-lines)
        for order in ("rows", "pencil16"):
            if order != "rows":
                A.set_sweep_order(256, pencil_order(lx, ly, lz, per_site=4, block_rows=256, yb=16))
            ms = timed(fn, reps=5)
            emit(case=f"c3 TI KPM step 2^24 rows w=16 {'C64' if dt == sellkit.C64 else 'R64'}", order=order, ms=ms,
                 gflops=fl / ms / 1e6, gbs=alg / ms / 1e6, frac=alg / ms / 1e6 / PEAK)
        del A, x, y


def c4():
    N = 100_000_000
    for m in (1, 2, 4, 8, 16, 32, 64):
        k = m
        V, W, X = sk.densemat(N, m), sk.densemat(N, k), sk.densemat(m, k)
        V.fill_hash(1)
        W.fill_hash(2)
        X.fill_hash(3)
        one, zero = np.array([1.0]), np.array([0.0])
        ms = timed(lambda: sk.call("sellkit_tsmm", W, V, X, one.ctypes.data, zero.ctypes.data), reps=5)
        alg = 8.0 * N * (m + k)
        emit(case="c4 tsmm N=1e8 beta=0", m=m, k=k, ms=ms, gflops=2.0 * N * m * k / ms / 1e6, gbs=alg / ms / 1e6,
             frac=alg / ms / 1e6 / PEAK)
        ms = timed(lambda: sk.call("sellkit_tsmttsm", X, V, W, one.ctypes.data, zero.ctypes.data, 0), reps=5)
        emit(case="c4 tsmttsm N=1e8", m=m, k=k, ms=ms, gflops=2.0 * N * m * k / ms / 1e6, gbs=alg / ms / 1e6,
             frac=alg / ms / 1e6 / PEAK)
        del V, W, X


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c4"]
    for w in which:
        globals()[w]()
