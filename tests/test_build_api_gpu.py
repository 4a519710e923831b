"""Construction and refresh entry points: matrices from the
row callback (sellkit_crs_from_rowfunc / sellkit_mat_build_rowfunc), value refresh
(sellkit_mat_update_values) and the CRS export (sellkit_mat_to_crs), checked like the
reference's own tests (proj/tests/unit_sparse.cpp:155-246, unit_capi.cpp:64-110,225-245):
layouts bit-identical to the CRS build, exact round trips, typed errors."""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import random_crs
from paper_1507_08101_b200 import sellkit
from paper_1507_08101_b200.sellkit import ROW_FN, SellkitError, vp

pytestmark = pytest.mark.gpu

LAYOUT = ["row_perm_inv", "row_perm", "rowlen", "chunk_len", "chunk_offset", "val", "col"]


def _rowfn(rp, col, val, cap=None):
    """ctypes row callback serving CRS rows (optionally writing at most `cap` entries)."""
    def fn(row, lenp, cols, vals, _arg):
        b, e = int(rp[row]), int(rp[row + 1])
        lenp[0] = e - b
        k = e - b if cap is None else min(e - b, cap)
        vv = C.cast(vals, C.POINTER(C.c_double))
        for j in range(k):
            cols[j] = int(col[b + j])
            vv[j] = float(val[b + j])
        return 0
    return ROW_FN(fn)


def _gcrs(crs, path):
    crs.write_bin(str(path))
    return open(path, "rb").read()


def _irregular(seed=3, n=700):
    rng = np.random.default_rng(seed)
    rp, col, val = random_crs(rng, n, n, 0.01)
    return rp, col, val


def test_rowfunc_build_matches_crs_build(sk, tmp_path):
    rp, col, val = _irregular()
    n = len(rp) - 1
    maxlen = int(np.max(np.diff(rp)))
    for C_, sigma in [(32, 256), (4, 8), (1, 1), (8, 1)]:
        A = sk.crs(rp, col, val).build(C_, sigma)
        cb = _rowfn(rp, col, val)
        h = vp()
        sk.call("sellkit_mat_build_rowfunc", sellkit.R64, n, n, maxlen, cb, None, C_, sigma, C.byref(h))
        B = sellkit.Mat(sk, h, sellkit.R64)
        la, lb = A.export(), B.export()
        for key in LAYOUT:
            assert np.array_equal(la[key], lb[key]), (C_, sigma, key)
    # CRS from the callback == CRS from the arrays (byte-identical GCRS files)
    cb = _rowfn(rp, col, val)
    h = vp()
    sk.call("sellkit_crs_from_rowfunc", sellkit.R64, n, n, maxlen, cb, None, C.byref(h))
    assert _gcrs(sellkit.Crs(sk, h, sellkit.R64), tmp_path / "a.gcrs") == _gcrs(sk.crs(rp, col, val), tmp_path / "b.gcrs")
    # a row longer than max_rowlen is rejected (the callback never writes past the capacity)
    lying = _rowfn(rp, col, val, cap=maxlen - 1)
    with pytest.raises(SellkitError) as ei:
        sk.call("sellkit_mat_build_rowfunc", sellkit.R64, n, n, maxlen - 1, lying, None, 32, 256, C.byref(vp()))
    assert ei.value.code == sellkit.ERR_INVALID_ARG


def test_update_values_and_to_crs_round_trip(sk, tmp_path):
    rp, col, val = _irregular(seed=5)
    src = sk.crs(rp, col, val)
    A = src.build(32, 256)
    before = A.export()
    # to_crs recovers the input exactly (unit_sparse.cpp:221-231)
    h = vp()
    sk.call("sellkit_mat_to_crs", A, C.byref(h))
    back = sellkit.Crs(sk, h, sellkit.R64)
    assert _gcrs(back, tmp_path / "back.gcrs") == _gcrs(src, tmp_path / "src.gcrs")
    # update_values: layout untouched, values = those of a fresh build (unit_sparse.cpp:189-219)
    doubled = sk.crs(rp, col, 2.0 * val)
    sk.call("sellkit_mat_update_values", A, doubled)
    after = A.export()
    fresh = sk.crs(rp, col, 2.0 * val).build(32, 256).export()
    for key in LAYOUT:
        if key != "val":
            assert np.array_equal(after[key], before[key]), key
    assert np.array_equal(after["val"], fresh["val"])
    again = after["val"].copy()
    sk.call("sellkit_mat_update_values", A, doubled)
    assert np.array_equal(A.export()["val"], again)  # idempotent
    # one more nonzero: pattern mismatch
    rp2 = rp.copy()
    rp2[1:] += 1
    col2 = np.insert(col, 0, 0 if col[0] != 0 else 1)
    if rp[1] > 0:
        seg = np.sort(col2[: rp2[1]])
        col2[: rp2[1]] = seg
    val2 = np.insert(val, 0, 1.0)
    try:
        extra = sk.crs(rp2, col2, val2)
    except SellkitError:
        pytest.skip("could not form the extra-nonzero matrix")
    with pytest.raises(SellkitError) as ei:
        sk.call("sellkit_mat_update_values", A, extra)
    assert ei.value.code == sellkit.ERR_PATTERN


def test_capi_identity_callback_and_empty_rows(sk, tmp_path):
    """unit_capi.cpp:64-110 (diag(1..8) through the callback, <y,y> = 204) and the empty-row
    round trip of unit_sparse.cpp:235-246."""
    def diag(row, lenp, cols, vals, _arg):
        lenp[0] = 1
        cols[0] = row
        C.cast(vals, C.POINTER(C.c_double))[0] = float(row + 1)
        return 0
    cb = ROW_FN(diag)
    h = vp()
    sk.call("sellkit_crs_from_rowfunc", sellkit.R64, 8, 8, 1, cb, None, C.byref(h))
    A = sellkit.Crs(sk, h, sellkit.R64).build(4, 4)
    assert A.stats()[0] == 1.0
    x, y = sk.densemat_from(np.ones((8, 1))), sk.densemat(8, 1)
    d = np.zeros(3)
    sk.spmv(y, A, x, flags=sellkit.DOT_YY, dot=d)
    assert d[0] == 204.0 and y.copy_out().sum() == 36.0
    gaps = sk.crs(np.array([0, 1, 1, 2]), np.array([0, 2]), np.array([1.0, 2.0]))
    G = gaps.build(2, 1)
    h = vp()
    sk.call("sellkit_mat_to_crs", G, C.byref(h))
    assert _gcrs(sellkit.Crs(sk, h, sellkit.R64), tmp_path / "g.gcrs") == _gcrs(gaps, tmp_path / "g0.gcrs")


def test_apply_override_matrix_free(sk):
    """sellkit_ext_mat_set_apply_override: the matrix-free operator slot of the reference
    (SellMatrix::apply_override, sellcs.hpp:116-119), KAT of unit_sparse.cpp:520-531:
    an override computing y = 2 x on identity(3) gives y[1] = 4; validation still runs
    first; removing the override restores the built-in multiply."""
    import ctypes as C
    A = sk.crs([0, 1, 2, 3], [0, 1, 2], np.ones(3)).build(1, 1)
    calls = []
    CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)

    def fn(y, x, opts, stream, ctx):
        calls.append(stream)
        two, zero = np.array([2.0]), np.array([0.0])
        return sk.lib.sellkit_axpby(y, x, two.ctypes.data, zero.ctypes.data)  # y = 2 x
    cb = CB(fn)
    sk.call("sellkit_ext_mat_set_apply_override", A.h, cb, None)
    x = sk.densemat_from(np.array([[1.0], [2.0], [3.0]]))
    y = sk.densemat_from(np.zeros((3, 1)))
    sk.spmv(y, A, x)
    assert y.copy_out()[1, 0] == 4.0 and len(calls) == 1 and calls[0]
    with pytest.raises(sellkit.SellkitError) as e:          # validated before the override runs
        sk.spmv(sk.densemat(4, 1), A, x)
    assert e.value.code == sellkit.ERR_SHAPE and len(calls) == 1
    sk.call("sellkit_ext_mat_set_apply_override", A.h, None, None)
    sk.spmv(y, A, x)
    assert y.copy_out()[:, 0].tolist() == [1.0, 2.0, 3.0]


@pytest.mark.parametrize("sigma,maxlen", [(256, 13), (4096, 63), (4096, 64), (1024, 200), (96, 5)])
def test_sigma_permutation_stable_descending(sk, orc, sigma, maxlen):
    """The σ-sort (sellcs.hpp:80-91): within each scope, rows stably ordered by descending
    length -- both the counting path (all rows < 64 entries) and the comparison path, ties,
    several 256-row chunks per scope and a ragged last scope."""
    rng = np.random.default_rng(sigma + maxlen)
    n = 3 * sigma + sigma // 3 + 1
    lens = rng.integers(0, maxlen + 1, n)
    lens[rng.integers(0, n, n // 8)] = maxlen  # many ties at the top length
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    step = n // (maxlen + 1)
    col = np.concatenate([(r % step) + step * np.arange(l) for r, l in enumerate(lens)]).astype(np.int64)
    val = rng.standard_normal(int(rp[-1]))
    A = sk.crs(rp, col, val).build(4, sigma)
    pinv = A.export()["row_perm_inv"]
    want = np.concatenate([s0 + np.argsort(-lens[s0:s0 + sigma], kind="stable") for s0 in range(0, n, sigma)])
    assert np.array_equal(pinv[:n], want)
    # whole layouts against the oracle: C = 32 takes the fused perm + chunk-length kernel,
    # C = 4 as well (4 divides the warp), both with short and long chunks
    for C_ in (32, 4):
        L = sk.crs(rp, col, val).build(C_, sigma).export()
        R = orc.build(rp, col, val, C_, sigma).layout()
        for key in LAYOUT:
            assert np.array_equal(L[key], R[key]), (C_, key)


def test_buffer_cache_reuse_and_release(sk):
    """Freed SELL storage is reused by the next build of the same size (layout unchanged) and
    returned to the driver by sellkit_ext_release_cached; builds after the release still work."""
    rp, col, val = _irregular(seed=9, n=900)
    crs = sk.crs(rp, col, val)
    first = crs.build(32, 64).export()
    for _ in range(2):
        again = crs.build(32, 64).export()  # the previous Mat was freed into the cache
        for key in LAYOUT:
            assert np.array_equal(first[key], again[key]), key
    sk.call("sellkit_ext_release_cached")
    after = crs.build(32, 64).export()
    for key in LAYOUT:
        assert np.array_equal(first[key], after[key]), key
