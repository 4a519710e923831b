"""Row-distributed SpMMV on the GPU: the reference's single-process API with k
ranks (all on the one visible B200 here: halos move through device memory, no
rank waits on another inside a kernel) against golden fixtures produced by the
reference's own dist_spmv, and against the serial oracle; plus the
one-process-per-GPU rank context at world size 1."""
import numpy as np
import pytest

from oracle.oracle import hash_block, stencil_crs
from paper_1507_08101_b200 import dist, sellkit

pytestmark = pytest.mark.gpu


def logical_y(orc_layout_perm, y_storage):
    return y_storage[orc_layout_perm]


def test_dist_vs_reference_golden(sk, golden):
    g = golden("dist.npz")
    cases = sorted({tuple(k.split("|")[:5]) for k in g.files if "|crs|" not in k})
    assert cases
    for name, k, by_nnz, C, sigma in cases:
        key = f"{name}|{k}|{by_nnz}|{C}|{sigma}"
        rp, c, v = g[f"{name}|crs|rowptr"], g[f"{name}|crs|col"], g[f"{name}|crs|val"]
        n = len(rp) - 1
        crs = sk.crs(rp, c, v)
        ctx = dist.DistContext(sk, crs, int(k), int(C), int(sigma), by_nnz=bool(int(by_nnz)), record=True)
        off = g[key + "|row_offset"]
        for r in range(int(k)):
            f, cnt = ctx.rank_range(r)
            assert (f, cnt) == (off[r], off[r + 1] - off[r]), key
            assert ctx.halo_size(r) == len(g[f"{key}|r{r}.halo_cols"]), key
        xv = g[key + "|x"]
        w = xv.shape[1]
        xg, yg = sk.densemat_from(xv), sk.densemat(n, w)
        dx, dy = ctx.vec(w), ctx.vec(w)
        ctx.scatter(xg, dx)
        dots = np.zeros(3 * w)
        ctx.spmv(dy, dx, flags=sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX, dot=dots)
        ctx.gather(dy, yg)
        y = yg.copy_out()
        assert np.array_equal(y, g[key + "|y"]), key  # local + remote split summed like the reference
        sc = np.concatenate([np.sum(y ** 2, 0), np.sum(np.abs(xv * y), 0), np.sum(xv ** 2, 0)])
        assert np.all(np.abs(dots - g[key + "|dot"]) <= 1e-12 * (1 + sc)), key
        assert list(ctx.comm_stats()) == g[key + "|comm"].tolist(), key  # byte/message counts exact


def test_dist_fused_vs_reference_golden(sk, golden):
    """The fused golden cases (shift / vshift, AXPBY, chain, dots) of the reference's own
    dist_spmv: y and z bit for bit, dots within 1e-12 (single process, all ranks here)."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from fused_cases import FUSED
    g = golden("dist.npz")
    cases = sorted({tuple(k.split("|")[:5]) for k in g.files if "|crs|" not in k})
    w = 2
    for name, k, by_nnz, C, sigma in cases:
        key = f"{name}|{k}|{by_nnz}|{C}|{sigma}"
        rp, c, v = g[f"{name}|crs|rowptr"], g[f"{name}|crs|col"], g[f"{name}|crs|val"]
        n = len(rp) - 1
        ctx = dist.DistContext(sk, sk.crs(rp, c, v), int(k), int(C), int(sigma), by_nnz=bool(int(by_nnz)))
        dx, dy, dz = ctx.vec(w), ctx.vec(w), ctx.vec(w)
        for fname, flags, gam in FUSED:
            fk = f"{key}|{fname}"
            for arr, dv in [(g[fk + "|x"], dx), (g[fk + "|y0"], dy), (g[fk + "|z0"], dz)]:
                ctx.scatter(sk.densemat_from(arr), dv)
            dots = np.zeros(3 * w)
            ctx.spmv(dy, dx, flags=flags, alpha=0.5, beta=-1.0, gamma=gam if len(gam) > 1 else gam[0], delta=1.0,
                     eta=0.3, z=dz, dot=dots)
            yg, zg = sk.densemat(n, w), sk.densemat(n, w)
            ctx.gather(dy, yg)
            ctx.gather(dz, zg)
            y = yg.copy_out()
            assert np.array_equal(y, g[fk + "|y"]), fk
            assert np.array_equal(zg.copy_out(), g[fk + "|z"]), fk
            xv = g[fk + "|x"]
            sc = np.concatenate([np.sum(y ** 2, 0), np.sum(np.abs(xv * y), 0), np.sum(xv ** 2, 0)])
            for s in range(3):
                if flags & (sellkit.DOT_YY << s):
                    part = slice(s * w, (s + 1) * w)
                    assert np.all(np.abs(dots[part] - g[fk + "|dot"][part]) <= 1e-12 * (1 + sc[part])), fk


@pytest.mark.parametrize("k", [1, 2, 3, 4, 7, 8])
@pytest.mark.parametrize("mode", [sellkit.NO_OVERLAP, sellkit.NAIVE_OVERLAP, sellkit.TASK_OVERLAP])
def test_dist_fused_vs_serial(sk, orc, k, mode):
    """Every flag through the distributed path equals the serial fused SpMV (1e-12)."""
    n, w = 14, 8
    N = n ** 3
    rp, c, v = stencil_crs(7, n)
    crs = sk.crs(rp, c, v)
    ctx = dist.DistContext(sk, crs, k, 32, 64, record=False)
    xv, y0, z0 = hash_block(N, w, 1), hash_block(N, w, 2), hash_block(N, w, 3)
    dx, dy, dz = ctx.vec(w), ctx.vec(w), ctx.vec(w)
    for arr, dv in [(xv, dx), (y0, dy), (z0, dz)]:
        ctx.scatter(sk.densemat_from(arr), dv)
    flags = (sellkit.AXPBY | sellkit.SHIFT | sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX |
             sellkit.CHAIN_AXPBY)
    dots = np.zeros(3 * w)
    ctx.spmv(dy, dx, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, delta=1.0, eta=0.3, z=dz, dot=dots, mode=mode)
    yg, zg = sk.densemat(N, w), sk.densemat(N, w)
    ctx.gather(dy, yg)
    ctx.gather(dz, zg)
    # serial reference in logical order: SELL-1-1 oracle is plain CRS order
    A = orc.build(rp, c, v, 1, 1)
    yo, zo, do = orc.spmv(A, xv, y0, z0, flags, alpha=0.5, beta=-1.0, gamma=0.25, delta=1.0, eta=0.3)
    rel = lambda a, b: np.max(np.abs(a - b) / (1 + np.abs(b)))  # noqa: E731
    assert rel(yg.copy_out(), yo) < 1e-12
    assert rel(zg.copy_out(), zo) < 1e-12
    assert np.all(np.abs(dots - do) <= 1e-12 * (1 + np.abs(do)))


@pytest.mark.parametrize("k", [2, 3])
def test_dist_wide_rows(sk, orc, k):
    """512-B RHS rows (w = 64) through the distributed path: the remote-part sweep takes the
    row-mapped wide-row kernel; every flag against the serial fused SpMV (1e-12)."""
    n, w = 12, 64
    N = n ** 3
    rp, c, v = stencil_crs(7, n)
    ctx = dist.DistContext(sk, sk.crs(rp, c, v), k, 32, 64, record=False)
    xv, y0, z0 = hash_block(N, w, 4), hash_block(N, w, 5), hash_block(N, w, 6)
    dx, dy, dz = ctx.vec(w), ctx.vec(w), ctx.vec(w)
    for arr, dv in [(xv, dx), (y0, dy), (z0, dz)]:
        ctx.scatter(sk.densemat_from(arr), dv)
    flags = (sellkit.AXPBY | sellkit.SHIFT | sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX |
             sellkit.CHAIN_AXPBY)
    dots = np.zeros(3 * w)
    ctx.spmv(dy, dx, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, delta=1.0, eta=0.3, z=dz, dot=dots,
             mode=sellkit.TASK_OVERLAP)
    yg, zg = sk.densemat(N, w), sk.densemat(N, w)
    ctx.gather(dy, yg)
    ctx.gather(dz, zg)
    A = orc.build(rp, c, v, 1, 1)
    yo, zo, do = orc.spmv(A, xv, y0, z0, flags, alpha=0.5, beta=-1.0, gamma=0.25, delta=1.0, eta=0.3)
    rel = lambda a, b: np.max(np.abs(a - b) / (1 + np.abs(b)))  # noqa: E731
    assert rel(yg.copy_out(), yo) < 1e-12
    assert rel(zg.copy_out(), zo) < 1e-12
    assert np.all(np.abs(dots - do) <= 1e-12 * (1 + np.abs(do)))


def test_nocomm_is_local_only(sk, orc):
    """spmv_nocomm drops the remote columns (partition.hpp:554-600)."""
    n, w, k = 8, 2, 4
    N = n ** 3
    rp, c, v = stencil_crs(7, n)
    ctx = dist.DistContext(sk, sk.crs(rp, c, v), k, 8, 32)
    xv = hash_block(N, w, 5)
    dx, dy = ctx.vec(w), ctx.vec(w)
    ctx.scatter(sk.densemat_from(xv), dx)
    ctx.spmv(dy, dx, nocomm=True)
    yg = sk.densemat(N, w)
    ctx.gather(dy, yg)
    off = dist.partition(sk, N, k)
    want = np.zeros((N, w))
    for r in range(k):
        for i in range(off[r], off[r + 1]):
            for jj in range(rp[i], rp[i + 1]):
                if off[r] <= c[jj] < off[r + 1]:
                    want[i] += v[jj] * xv[c[jj]]
    assert np.max(np.abs(yg.copy_out() - want)) < 1e-12


def test_rank_context_world1(sk, orc):
    """The multi-process rank context at world size 1 (no NCCL) equals serial spmv bit for bit."""
    n, w = 12, 8
    N = n ** 3
    rp, c, v = stencil_crs(7, n)
    off = np.array([0, N], np.int64)
    rows = sk.crs_stencil(7, n, 0, N)
    rc = dist.RankContext(sk, rows, off, 0, 32, 256)
    rc.connect(bytes(128))
    perm = rc.row_perm()
    xv = hash_block(N, w, 9)
    xs = np.empty_like(xv)
    xs[perm] = xv
    x, y = sk.densemat_from(xs), sk.densemat(N, w)
    dots = np.zeros(3 * w)
    rc.spmv(y, x, flags=sellkit.DOT_YY, dot=dots)
    Ao = orc.build(rp, c, v, 32, 256)
    yo, _, do = orc.spmv(Ao, xs, flags=sellkit.DOT_YY)
    assert np.array_equal(y.copy_out(), yo)
    assert abs(dots[0] - do[0]) <= 1e-12 * (1 + abs(do[0]))


def test_dist_timeline_trace(sk):
    """sellkit_ext_ctx_set_trace / _timeline: per rank exchange and sweep intervals of
    one dist_spmv, ordered as the streams run them."""
    import ctypes as C
    n, k, w = 24, 3, 4
    ctx = dist.DistContext(sk, sk.crs_stencil(7, n), k, 32, 256, record=False)
    x, y = ctx.vec(w), ctx.vec(w)
    sk.call("sellkit_ext_ctx_set_trace", ctx.h, 1)
    ctx.spmv(y, x)
    cnt = C.c_int(0)
    sk.call("sellkit_ext_ctx_timeline", ctx.h, None, C.byref(cnt))
    assert cnt.value == 5 * k
    buf = (C.c_double * cnt.value)()
    sk.call("sellkit_ext_ctx_timeline", ctx.h, buf, C.byref(cnt))
    t = np.array(buf[:]).reshape(k, 5)
    for r in range(k):
        xs, xe, ls, le, re_ = t[r]
        assert 0 <= xs <= xe and 0 <= ls <= le <= re_, t[r]
        # the remote sweep waited for the halo of its owners (the neighbouring slabs)
        for o in (r - 1, r + 1):
            if 0 <= o < k:
                assert t[o][1] <= re_, (r, o, t)


@pytest.mark.parametrize("k", [2, 3])
def test_dist_col_major_vectors(sk, k):
    """Distributed vectors in column-major order (sellkit_dvec_create order argument): the
    pack kernel and the generic sweeps take the strides, so y, z and the dots equal the
    row-major run bit for bit (same per-row order)."""
    n, w = 10, 3
    N = n ** 3
    rp, c, v = stencil_crs(7, n)
    ctx = dist.DistContext(sk, sk.crs(rp, c, v), k, 4, 8, record=False)
    xv, y0, z0 = hash_block(N, w, 31), hash_block(N, w, 32), hash_block(N, w, 33)
    flags = (sellkit.AXPBY | sellkit.SHIFT | sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX |
             sellkit.CHAIN_AXPBY)
    out = {}
    for order in (sellkit.ROW_MAJOR, sellkit.COL_MAJOR):
        dx, dy, dz = ctx.vec(w, order), ctx.vec(w, order), ctx.vec(w, order)
        for arr, dv in [(xv, dx), (y0, dy), (z0, dz)]:
            ctx.scatter(sk.densemat_from(arr), dv)
        dots = np.zeros(3 * w)
        ctx.spmv(dy, dx, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, delta=1.0, eta=0.3, z=dz, dot=dots)
        yg, zg = sk.densemat(N, w), sk.densemat(N, w)
        ctx.gather(dy, yg)
        ctx.gather(dz, zg)
        out[order] = (yg.copy_out(), zg.copy_out(), dots)
    yr, zr, dr = out[sellkit.ROW_MAJOR]
    yc, zc, dc = out[sellkit.COL_MAJOR]
    assert np.array_equal(yr, yc) and np.array_equal(zr, zc)
    sc = np.concatenate([np.sum(yr ** 2, 0), np.sum(np.abs(xv * yr), 0), np.sum(xv ** 2, 0)])
    assert np.all(np.abs(dr - dc) <= 1e-12 * (1 + sc))
