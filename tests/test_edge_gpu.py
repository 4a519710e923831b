"""Edge shapes through the C ABI: empty matrices (0 rows, 0 nonzeros), a single row,
block widths past the specialised kernels, and TSM on 0 rows.  The reference admits
nrows >= 0 (capi.cpp:239) and zero-length rows everywhere (sellcs.hpp); results are
compared bit-exactly with row sums in the reference's order (separate rounding, j
ascending: spmv_epilogue.hpp / sellcs.hpp)."""
import numpy as np
import pytest

from oracle.oracle import random_crs
from paper_1507_08101_b200 import sellkit

pytestmark = pytest.mark.gpu


def test_zero_rows(sk):
    # a 0-row CRS matrix is valid (capi.cpp:239), SELL construction needs a row
    # (sellcs.hpp:149) and a dense block needs rows (densemat.hpp:30)
    crs = sk.crs(np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0), 4)
    assert crs.dims()[0] == 0
    for fn in (lambda: crs.build(32, 1), lambda: sk.densemat(0, 8)):
        with pytest.raises(sellkit.SellkitError) as e:
            fn()
        assert e.value.code == sellkit.ERR_INVALID_ARG


@pytest.mark.parametrize("w", [1, 4, 8, 16])
def test_all_rows_empty(sk, w):
    n = 100
    A = sk.crs(np.zeros(n + 1, np.int64), np.zeros(0, np.int32), np.zeros(0), n).build(32, 256)
    x, y = sk.densemat(n, w), sk.densemat(n, w)
    x.fill_hash(3)
    y.fill_hash(4)
    sk.spmv(y, A, x)
    assert np.array_equal(y.copy_out(), np.zeros((n, w)))


@pytest.mark.parametrize("w", [1, 3, 8, 64])
def test_single_row_and_single_nonempty_row(sk, w):
    rng = np.random.default_rng(w)
    A = sk.crs([0, 1], [0], np.array([2.5]), 1).build(32, 1)
    X = rng.uniform(-1, 1, (1, w))
    x, y = sk.densemat_from(X), sk.densemat(1, w)
    sk.spmv(y, A, x)
    assert np.array_equal(y.copy_out(), 2.5 * X)
    # 5 x 5, only row 3 stored (sigma = 1: no permutation)
    rp, col, val = [0, 0, 0, 0, 3, 3], [0, 2, 4], np.array([1.5, -2.0, 0.25])
    A = sk.crs(rp, col, val, 5).build(32, 1)
    X = rng.uniform(-1, 1, (5, w))
    x, y = sk.densemat_from(X), sk.densemat(5, w)
    sk.spmv(y, A, x)
    want = np.zeros((5, w))
    # row sum in j order with separate rounding, as the reference
    want[3] = ((0.0 + val[0] * X[0]) + val[1] * X[2]) + val[2] * X[4]
    assert np.array_equal(y.copy_out(), want)


@pytest.mark.parametrize("w", [65, 100, 128])
def test_widths_past_specialised_kernels(sk, w):
    n = 3000
    rp, col, val = random_crs(np.random.default_rng(w), n, n, 9 / n)
    A = sk.crs(rp, col, val, n).build(32, 1)  # sigma = 1: x and y in the original order
    rng = np.random.default_rng(w)
    X = rng.uniform(-1, 1, (n, w))
    x, y = sk.densemat_from(X), sk.densemat(n, w)
    sk.spmv(y, A, x)
    want = np.zeros((n, w))
    for r in range(n):
        acc = np.zeros(w)
        for j in range(rp[r], rp[r + 1]):
            acc = acc + val[j] * X[col[j]]
        want[r] = acc
    assert np.array_equal(y.copy_out(), want)
