"""Parity of the B200 SELL-C-sigma construction and fused SpMV/SpMMV with the
reference (golden fixtures) and the CPU oracle.  Bar: layouts and y/z
bit-identical; dots within 1e-12 relative to sum |x||y| (the reference's own dots
depend on its worker count)."""
import numpy as np
import pytest

from oracle.oracle import hash_block, random_crs, stencil_crs
from paper_1507_08101_b200 import sellkit

pytestmark = pytest.mark.gpu

LAYOUT_KEYS = ["row_perm_inv", "row_perm", "rowlen", "chunk_len", "chunk_offset", "val", "col"]
DOT_TOL = 1e-12


def golden_mats(g):
    names = sorted({k.split("|")[0] for k in g.files if "|crs|" in k})
    return {n: (g[f"{n}|crs|rowptr"], g[f"{n}|crs|col"], g[f"{n}|crs|val"], int(g[f"{n}|crs|ncols"][0]))
            for n in names}


def dots_close(got, want, scale):
    return np.all(np.abs(got - want) <= DOT_TOL * (1.0 + scale))


def test_layout_bit_exact_vs_reference(sk, golden):
    g = golden("sell_layouts.npz")
    mats = golden_mats(g)
    combos = sorted({tuple(k.split("|")[:3]) for k in g.files if "|crs|" not in k})
    for name, C, sigma in combos:
        rp, c, v, nc = mats[name]
        A = sk.crs(rp, c, v, nc).build(int(C), int(sigma))
        L = A.export()
        for key in LAYOUT_KEYS:
            assert np.array_equal(L[key], g[f"{name}|{C}|{sigma}|{key}"]), (name, C, sigma, key)
        beta, nbytes = A.stats()
        assert beta == g[f"{name}|{C}|{sigma}|beta"][0]


def test_worked_4x4_and_errors(sk):
    A = sk.crs([0, 1, 3, 4, 7], [0, 0, 1, 2, 1, 2, 3], np.arange(1, 8, dtype=float)).build(2, 4)
    L = A.export()
    assert L["val"][:6].tolist() == [5, 2, 6, 3, 7, 0]
    assert L["chunk_offset"].tolist() == [0, 6, 8]
    crs = sk.crs([0, 1, 3, 4, 7], [0, 0, 1, 2, 1, 2, 3], np.arange(1, 8, dtype=float))
    for C, s in [(0, 1), (4, 2)]:
        with pytest.raises(sellkit.SellkitError) as e:
            crs.build(C, s)
        assert e.value.code == sellkit.ERR_INVALID_ARG
    crs.build(3, 7)
    with pytest.raises(sellkit.SellkitError) as e:
        sk.crs([0, 1, 3, 4, 7], [9, 0, 1, 2, 1, 2, 3], np.arange(1, 8, dtype=float))
    assert e.value.code == sellkit.ERR_INVALID_ARG
    with pytest.raises(sellkit.SellkitError) as e:  # unit_capi.cpp:50-54: rowptr not monotone
        sk.crs([0, 2, 1], [0, 0, 1], np.ones(3))
    assert e.value.code == sellkit.ERR_INVALID_ARG


def test_fusion_all_flag_combinations(sk, golden):
    g = golden("spmv.npz")
    rp, c, v, nc = golden_mats(golden("sell_layouts.npz"))["rand0"]
    A = sk.crs(rp, c, v, nc).build(4, 8)
    x0, y0, z0 = g["fusion|x"], g["fusion|y0"], g["fusion|z0"]
    gammas = np.array([0.5, -1.5, 2.0])
    n = 0
    for flags in range(128):
        if (flags & sellkit.SHIFT) and (flags & sellkit.VSHIFT):
            continue
        x, y, z = sk.densemat_from(x0), sk.densemat_from(y0), sk.densemat_from(z0)
        dots = np.full(9, 99.0)
        gam = gammas if flags & sellkit.VSHIFT else gammas[:1]
        sk.spmv(y, A, x, flags=flags, alpha=1.3, beta=-0.7, gamma=gam, delta=0.4, eta=2.2, z=z, dot=dots)
        assert np.array_equal(y.copy_out(), g[f"fusion|{flags}|y"]), flags
        assert np.array_equal(z.copy_out(), g[f"fusion|{flags}|z"]), flags
        want = g[f"fusion|{flags}|dot"]
        yv = g[f"fusion|{flags}|y"]
        scales = [np.sum(np.abs(yv) ** 2, 0), np.sum(np.abs(x0 * yv), 0), np.sum(np.abs(x0) ** 2, 0)]
        for s, bit in enumerate((sellkit.DOT_YY, sellkit.DOT_XY, sellkit.DOT_XX)):
            seg = slice(3 * s, 3 * s + 3)
            if flags & bit:
                assert dots_close(dots[seg], want[seg], scales[s]), (flags, dots[seg], want[seg])
            else:
                assert np.all(dots[seg] == 99.0), flags  # only requested thirds are written
        n += 1
    assert n == 96


def test_sweeps_vs_reference(sk, golden):
    g = golden("spmv.npz")
    mats = golden_mats(golden("sell_layouts.npz"))
    keys = sorted({tuple(k.split("|")[1:5]) for k in g.files if k.startswith("sweep|")})
    for name, C, sigma, w in keys:
        rp, c, v, nc = mats[name]
        A = sk.crs(rp, c, v, nc).build(int(C), int(sigma))
        key = f"sweep|{name}|{C}|{sigma}|{w}"
        xv = g[key + "|x"]
        x, y = sk.densemat_from(xv), sk.densemat(len(rp) - 1, int(w))
        dots = np.zeros(3 * int(w))
        sk.spmv(y, A, x, flags=0x38, dot=dots)
        yv = y.copy_out()
        assert np.array_equal(yv, g[key + "|y"]), key
        sc = np.concatenate([np.sum(yv ** 2, 0), np.sum(np.abs(xv * yv), 0), np.sum(xv ** 2, 0)])
        assert dots_close(dots, g[key + "|dot"], sc), key


@pytest.mark.parametrize("w", [1, 2, 3, 4, 5, 8, 12, 16, 32, 64])
@pytest.mark.parametrize("C,sigma", [(32, 256), (32, 1), (8, 32), (4, 4), (1, 1), (16, 64)])
def test_stencil_widths_vs_oracle(sk, orc, w, C, sigma):
    n = 20
    rp, c, v = stencil_crs(7, n)
    A = sk.crs(rp, c, v).build(C, sigma)
    Ao = orc.build(rp, c, v, C, sigma)
    xv = hash_block(n ** 3, w, 42)
    x, y = sk.densemat_from(xv), sk.densemat(n ** 3, w)
    z0 = hash_block(n ** 3, w, 44)
    z = sk.densemat_from(z0)
    y0 = hash_block(n ** 3, w, 43)
    y.copy_in(y0)
    flags = sellkit.AXPBY | sellkit.SHIFT | sellkit.CHAIN_AXPBY
    sk.spmv(y, A, x, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, delta=1.0, eta=0.3, z=z)
    yo, zo, _ = orc.spmv(Ao, xv, y0, z0, flags, alpha=0.5, beta=-1.0, gamma=0.25, delta=1.0, eta=0.3)
    assert np.array_equal(y.copy_out(), yo)
    assert np.array_equal(z.copy_out(), zo)


def test_device_stencil_generator_matches_numpy(sk, orc):
    for points, n in [(5, 33), (7, 17)]:
        rp, c, v = stencil_crs(points, n)
        A_dev = sk.crs_stencil(points, n).build(32, 256)
        A_host = orc.build(rp, c, v, 32, 256).layout()
        L = A_dev.export()
        for key in LAYOUT_KEYS:
            assert np.array_equal(L[key], A_host[key]), (points, key)
    # a row block of the 3-D stencil keeps global columns
    crs = sk.crs_stencil(7, 10, 300, 700)
    assert crs.dims() == (400, 1000, int(stencil_crs(7, 10, 300, 700)[0][-1]))


def test_complex_vs_oracle(sk, orc):
    rng = np.random.default_rng(3)
    rp, c, v = random_crs(rng, 300, 300, 0.03, cplx=True)
    for C, sigma, w in [(32, 64, 4), (8, 8, 3), (32, 1, 16), (4, 300, 1)]:
        A = sk.crs(rp, c, v).build(C, sigma)
        Ao = orc.build(rp, c, v, C, sigma)
        xv = rng.uniform(-1, 1, (300, w)) + 1j * rng.uniform(-1, 1, (300, w))
        y0 = rng.uniform(-1, 1, (300, w)) + 1j * rng.uniform(-1, 1, (300, w))
        x, y = sk.densemat_from(xv), sk.densemat_from(y0)
        dots = np.zeros(3 * w, np.complex128)
        flags = sellkit.AXPBY | sellkit.SHIFT | sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX
        sk.spmv(y, A, x, flags=flags, alpha=0.5 + 0.25j, beta=-1.0, gamma=0.1 - 0.2j, dot=dots)
        yo, _, do = orc.spmv(Ao, xv, y0, None, flags, alpha=0.5 + 0.25j, beta=-1.0, gamma=0.1 - 0.2j)
        assert np.array_equal(y.copy_out(), yo), (C, sigma, w)
        assert np.allclose(dots, do, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("dt,w", [("r64", 64), ("c64", 32), ("c64", 64), ("r32", 64), ("c32", 64)])
@pytest.mark.parametrize("C,sigma", [(32, 256), (8, 32), (4, 1)])
def test_wide_rhs_rows(sk, orc, dt, w, C, sigma):
    """RHS rows of 512 B / 1 KB (the rows kernel with 64- / 128-byte lane vectors): y
    bit-identical to the oracle for the plain sweep and the KPM step, dots within 1e-12."""
    rng = np.random.default_rng(w + C)
    cplx = dt in ("c64", "c32")
    rp, c, v = random_crs(rng, 700, 700, 0.012, cplx=cplx)
    sdt = {"r64": sellkit.R64, "c64": sellkit.C64, "r32": sellkit.R32, "c32": sellkit.C32}[dt]
    npdt = sellkit.NP_DTYPE[sdt]
    v = v.astype(npdt)
    A = sk.crs(rp, c, v, dt=sdt).build(C, sigma)
    Ao = orc.build(rp, c, v.astype(np.complex128 if cplx else np.float64), C, sigma)
    xv = rng.uniform(-1, 1, (700, w)) + (1j * rng.uniform(-1, 1, (700, w)) if cplx else 0)
    y0 = rng.uniform(-1, 1, (700, w)) + (1j * rng.uniform(-1, 1, (700, w)) if cplx else 0)
    xv, y0 = xv.astype(npdt), y0.astype(npdt)
    x = sk.densemat_from(xv)
    y = sk.densemat(700, w, sdt)
    sk.spmv(y, A, x)
    if dt in ("r64", "c64"):
        yo, _, _ = orc.spmv(Ao, xv)
        assert np.array_equal(y.copy_out(), yo)
        y = sk.densemat_from(y0)
        dots = np.zeros(3 * w, npdt)
        flags = sellkit.AXPBY | sellkit.SHIFT | sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX
        al = 0.5 + 0.25j if cplx else 0.5
        ga = 0.1 - 0.2j if cplx else 0.25
        sk.spmv(y, A, x, flags=flags, alpha=al, beta=-1.0, gamma=ga, dot=dots)
        yo, _, do = orc.spmv(Ao, xv, y0, None, flags, alpha=al, beta=-1.0, gamma=ga)
        assert np.array_equal(y.copy_out(), yo)
        assert np.allclose(dots, do, rtol=1e-12, atol=1e-12)
    else:  # single precision: against the oracle's double-precision sweep of the same values
        yo, _, _ = orc.spmv(Ao, xv.astype(np.complex128 if cplx else np.float64))
        assert np.max(np.abs(y.copy_out() - yo)) <= 1e-4 * (1 + np.max(np.abs(yo)))


@pytest.mark.parametrize("off", [0, 8, 1])
def test_wide_column_views(sk, orc, off):
    """64-column row-major views into 80-column parents (sellkit_densemat_view with a
    contiguous column range): strided x and y rows, 64-B aligned (off 0, 8) and not (off 1,
    which must leave the vector kernels); y bit-identical to the oracle, other columns untouched."""
    import ctypes as C
    rng = np.random.default_rng(11 + off)
    rp, c, v = random_crs(rng, 600, 600, 0.015)
    A = sk.crs(rp, c, v).build(32, 64)
    Ao = orc.build(rp, c, v, 32, 64)
    X = rng.uniform(-1, 1, (600, 80))
    Y = rng.uniform(-1, 1, (600, 80))
    xp, yp = sk.densemat_from(X), sk.densemat_from(Y)
    cols = (C.c_int32 * 64)(*range(off, off + 64))
    xh, yh = C.c_void_p(), C.c_void_p()
    sk.call("sellkit_densemat_view", xp.h, 0, 600, cols, 64, C.byref(xh))
    sk.call("sellkit_densemat_view", yp.h, 0, 600, cols, 64, C.byref(yh))
    x, y = sellkit.DenseMat(sk, xh, sellkit.R64), sellkit.DenseMat(sk, yh, sellkit.R64)
    flags = sellkit.AXPBY | sellkit.SHIFT
    sk.spmv(y, A, x, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25)
    yo, _, _ = orc.spmv(Ao, np.ascontiguousarray(X[:, off:off + 64]), np.ascontiguousarray(Y[:, off:off + 64]), None,
                        flags, alpha=0.5, beta=-1.0, gamma=0.25)
    got = yp.copy_out()
    assert np.array_equal(got[:, off:off + 64], yo)
    rest = np.ones(80, bool)
    rest[off:off + 64] = False
    assert np.array_equal(got[:, rest], Y[:, rest])


def test_ti_generator_and_kpm_step(sk, orc):
    """C3: the device TI Hamiltonian equals the numpy restatement; the augmented KPM
    step y = 2a(H - bI)x - y with <y,y>, <x,y>, <x,x> (w = 16, complex) is bit-identical
    to the oracle in y and within 1e-12 in the dots."""
    from oracle.oracle import ti_crs
    lx, ly, lz, dis = 8, 6, 5, 0.7
    rp, c, v = ti_crs(lx, ly, lz, dis)
    n = len(rp) - 1
    for dt in (sellkit.C64, sellkit.R64):
        vv = v if dt == sellkit.C64 else v.real.copy()
        A = sk.crs_ti(lx, ly, lz, dis, dt=dt).build(32, 128)
        Ao = orc.build(rp, c, vv, 32, 128).layout()
        L = A.export()
        for key in LAYOUT_KEYS:
            assert np.array_equal(L[key], Ao[key]), (dt, key)
    A = sk.crs_ti(lx, ly, lz, dis).build(32, 128)
    Ao = orc.build(rp, c, v, 32, 128)
    rng = np.random.default_rng(4)
    w = 16
    xv = rng.uniform(-1, 1, (n, w)) + 1j * rng.uniform(-1, 1, (n, w))
    y0 = rng.uniform(-1, 1, (n, w)) + 1j * rng.uniform(-1, 1, (n, w))
    x, y = sk.densemat_from(xv), sk.densemat_from(y0)
    dots = np.zeros(3 * w, np.complex128)
    flags = sellkit.AXPBY | sellkit.SHIFT | sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX
    sk.spmv(y, A, x, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, dot=dots)
    yo, _, do = orc.spmv(Ao, xv, y0, None, flags, alpha=0.5, beta=-1.0, gamma=0.25)
    assert np.array_equal(y.copy_out(), yo)
    assert np.allclose(dots, do, rtol=1e-12, atol=1e-12)


def test_single_precision(sk, orc):
    rng = np.random.default_rng(9)
    rp, c, v = random_crs(rng, 200, 200, 0.05)
    for dt, tol in [(sellkit.R32, 1e-5), (sellkit.C32, 1e-5)]:
        cplx = dt == sellkit.C32
        vv = (v + 0.5j * v) if cplx else v
        A = sk.crs(rp, c, vv.astype(sellkit.NP_DTYPE[dt]), dt=dt).build(32, 32)
        Ao = orc.build(rp, c, vv.astype(np.complex128 if cplx else np.float64), 32, 32)
        xv = rng.uniform(-1, 1, (200, 8)).astype(sellkit.NP_DTYPE[dt])
        x, y = sk.densemat_from(xv), sk.densemat(200, 8, dt)
        sk.spmv(y, A, x)
        yo, _, _ = orc.spmv(Ao, xv.astype(np.complex128 if cplx else np.float64))
        assert np.max(np.abs(y.copy_out() - yo) / (1 + np.abs(yo))) < tol


def test_col_major_and_host_views(sk, orc):
    rp, c, v = stencil_crs(5, 30)
    n = 900
    A = sk.crs(rp, c, v).build(32, 128)
    Ao = orc.build(rp, c, v, 32, 128)
    xv = hash_block(n, 4, 7)
    yo, _, _ = orc.spmv(Ao, xv)
    # column-major block vectors -> generic kernel
    x = sk.densemat_from(xv, order=sellkit.COL_MAJOR)
    y = sk.densemat(n, 4, order=sellkit.COL_MAJOR)
    sk.spmv(y, A, x)
    assert np.array_equal(y.copy_out(), yo)
    # host memory through view_plain (staged by the library)
    xh = np.ascontiguousarray(xv)
    yh = np.zeros((n, 4))
    xvw = sk.view_plain(xh.ctypes.data, xh.size, n, 4, 4, keep=xh)
    yvw = sk.view_plain(yh.ctypes.data, yh.size, n, 4, 4, keep=yh)
    sk.spmv(yvw, A, xvw)
    assert np.array_equal(yh, yo)


@pytest.mark.parametrize("w", [1, 8])
def test_streamed_pinned_host_buffers(sk, orc, w):
    """sellkit_spmv on pinned host views streams x in / y out by row blocks (column
    watermarks); results are bit-identical to the resident path and the oracle."""
    import torch
    n = 40
    N = n ** 3
    rp, c, v = stencil_crs(7, n)
    A = sk.crs_stencil(7, n).build(32, 256)
    Ao = orc.build(rp, c, v, 32, 256)
    xv, y0, z0 = hash_block(N, w, 11), hash_block(N, w, 12), hash_block(N, w, 13)
    bufs = {}
    for name, arr in [("x", xv), ("y", y0), ("z", z0)]:
        t = torch.empty((N, w), dtype=torch.float64, pin_memory=True)
        t.copy_(torch.from_numpy(arr))
        bufs[name] = t
    views = {k: sk.view_plain(t.data_ptr(), N * w, N, w, w, keep=t) for k, t in bufs.items()}
    flags = sellkit.AXPBY | sellkit.SHIFT | sellkit.DOT_YY | sellkit.DOT_XY | sellkit.CHAIN_AXPBY
    dots = np.zeros(3 * w)
    sk.spmv(views["y"], A, views["x"], flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, delta=1.0, eta=0.3,
            z=views["z"], dot=dots)
    yo, zo, do = orc.spmv(Ao, xv, y0, z0, flags, alpha=0.5, beta=-1.0, gamma=0.25, delta=1.0, eta=0.3)
    assert np.array_equal(bufs["y"].numpy(), yo)
    assert np.array_equal(bufs["z"].numpy(), zo)
    assert np.all(np.abs(dots[:2 * w] - do[:2 * w]) <= 1e-12 * (1 + np.abs(do[:2 * w])))


@pytest.mark.parametrize("w", [1, 4])
def test_streamed_pinned_strictly_lower(sk, orc, w):
    """Streamed pinned-host spmv with x read at the block's own rows (SHIFT, <x,y>,
    <x,x>) on a matrix whose rows only reach columns BELOW them (strictly lower, many
    empty rows): a block's column watermark is then smaller than its own rows, so the
    x slab holding those rows must also have arrived (spmv.cu streamed path)."""
    import torch
    rng = np.random.default_rng(77 + w)
    n = 20000
    rows, rp = [], [0]
    for r in range(n):
        k = 0 if (r % 97) > 60 or r == 0 else int(rng.integers(1, 4))
        c = np.sort(rng.choice(max(1, min(r, 64)), size=min(k, max(1, min(r, 64))), replace=False)) if k else []
        rows.append(np.asarray(c, np.int64))
        rp.append(rp[-1] + len(c))
    rp = np.array(rp, np.int64)
    col = np.concatenate(rows).astype(np.int64)
    val = rng.uniform(-1, 1, len(col))
    A = sk.crs(rp, col, val).build(32, 1)
    Ao = orc.build(rp, col, val, 32, 1)
    xv, y0 = hash_block(n, w, 21), hash_block(n, w, 22)
    bufs = {}
    for name, arr in [("x", xv), ("y", y0)]:
        t = torch.empty((n, w), dtype=torch.float64, pin_memory=True)
        t.copy_(torch.from_numpy(arr))
        bufs[name] = t
    views = {k: sk.view_plain(t.data_ptr(), n * w, n, w, w, keep=t) for k, t in bufs.items()}
    flags = sellkit.AXPBY | sellkit.SHIFT | sellkit.DOT_XY | sellkit.DOT_XX
    dots = np.zeros(3 * w)
    sk.spmv(views["y"], A, views["x"], flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, dot=dots)
    yo, _, do = orc.spmv(Ao, xv, y0, None, flags, alpha=0.5, beta=-1.0, gamma=0.25)
    assert np.array_equal(bufs["y"].numpy(), yo)
    assert np.all(np.abs(dots[w:] - do[w:]) <= 1e-12 * (1 + np.abs(do[w:])))


def test_spmv_validation(sk):
    I = sk.crs(np.arange(4), np.arange(3), np.ones(3)).build(1, 1)
    x, y = sk.densemat(3, 1), sk.densemat(3, 1)
    with pytest.raises(sellkit.SellkitError) as e:
        sk.spmv(y, I, x, flags=sellkit.SHIFT | sellkit.VSHIFT, gamma=[1.0])
    assert e.value.code == sellkit.ERR_INVALID_ARG
    with pytest.raises(sellkit.SellkitError) as e:
        sk.spmv(y, I, x, flags=sellkit.DOT_YY)
    assert e.value.code == sellkit.ERR_INVALID_ARG
    wide = sk.densemat(3, 2)
    with pytest.raises(sellkit.SellkitError) as e:
        sk.spmv(wide, I, x)
    assert e.value.code == sellkit.ERR_SHAPE
    with pytest.raises(sellkit.SellkitError) as e:
        sk.spmv(x, I, x)
    assert e.value.code == sellkit.ERR_INVALID_ARG
    with pytest.raises(sellkit.SellkitError) as e:
        sk.spmv(y, I, x, flags=0x80)
    assert e.value.code == sellkit.ERR_INVALID_ARG
    xf = sk.densemat(3, 1, sellkit.R32)
    with pytest.raises(sellkit.SellkitError) as e:
        sk.spmv(y, I, xf)
    assert e.value.code == sellkit.ERR_INVALID_ARG
    # shift annihilates the identity (unit_sparse.cpp:322-331)
    x.copy_in(np.arange(1.0, 4.0))
    sk.spmv(y, I, x, flags=sellkit.SHIFT, gamma=1.0)
    assert np.all(y.copy_out() == 0.0)


def test_capi_identity_dot(sk):
    # unit_capi.cpp:63-114: diag(1..8) * ones => <y,y> = 204
    rp = np.arange(9)
    A = sk.crs(rp, np.arange(8), np.arange(1.0, 9.0)).build(4, 4)
    x, y = sk.densemat_from(np.ones(8)), sk.densemat(8, 1)
    dots = np.zeros(3)
    sk.spmv(y, A, x, flags=sellkit.DOT_YY, dot=dots)
    assert dots[0] == 204.0
    assert y.copy_out().sum() == 36.0


def test_large_stencil_bitwise(sk, orc):
    """A size where every kernel path runs many CTAs: 3-D 96^3, SELL-32-256, w = 8."""
    n, w = 96, 8
    rp, c, v = stencil_crs(7, n)
    A = sk.crs_stencil(7, n).build(32, 256)
    Ao = orc.build(rp, c, v, 32, 256)
    x = sk.densemat(n ** 3, w)
    x.fill_hash(42)
    xv = x.copy_out()
    assert np.array_equal(xv, hash_block(n ** 3, w, 42))
    y = sk.densemat(n ** 3, w)
    dots = np.zeros(3 * w)
    sk.spmv(y, A, x, flags=0x38, dot=dots)
    yo, _, do = orc.spmv(Ao, xv, flags=0x38)
    assert np.array_equal(y.copy_out(), yo)
    sc = np.concatenate([np.sum(yo ** 2, 0), np.sum(np.abs(xv * yo), 0), np.sum(xv ** 2, 0)])
    assert dots_close(dots, do, sc)


@pytest.mark.parametrize("w", [1, 4, 8, 16, 32, 64])
@pytest.mark.parametrize("C,sigma", [(32, 256), (8, 64), (4, 1)])
def test_irregular_rows_all_paths(sk, orc, w, C, sigma):
    """Rows of very different lengths (empty rows, a 3000-nonzero row, a dense block of
    long rows): exercises tiles whose chunks overflow a shared-memory stage, the
    row-length remainder paths and the fallback kernels; y must stay bit-identical."""
    rng = np.random.default_rng(1000 * w + C)
    n = 5000
    lens = rng.integers(0, 12, n)
    lens[17] = 0
    lens[100] = 3000
    lens[2000:2040] = 400
    rows, cols, vals = [], [], []
    rp = [0]
    for r in range(n):
        c = np.sort(rng.choice(n, size=int(lens[r]), replace=False))
        cols.append(c)
        vals.append(rng.uniform(-1, 1, len(c)))
        rp.append(rp[-1] + len(c))
    rp = np.array(rp, np.int64)
    col = np.concatenate(cols).astype(np.int64)
    val = np.concatenate(vals)
    A = sk.crs(rp, col, val).build(C, sigma)
    Ao = orc.build(rp, col, val, C, sigma)
    xv = hash_block(n, w, 7)
    y0 = hash_block(n, w, 8)
    x, y = sk.densemat_from(xv), sk.densemat_from(y0)
    flags = sellkit.AXPBY | sellkit.SHIFT
    sk.spmv(y, A, x, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25)
    yo, _, _ = orc.spmv(Ao, xv, y0, None, flags, alpha=0.5, beta=-1.0, gamma=0.25)
    assert np.array_equal(y.copy_out(), yo)
    y2 = sk.densemat(n, w)
    sk.spmv(y2, A, x)
    yo2, _, _ = orc.spmv(Ao, xv)
    assert np.array_equal(y2.copy_out(), yo2)
