"""Tall-skinny kernels on the B200 vs the reference (golden) and the CPU oracle
(proj/tests/unit_sparse.cpp:609-860).  TSMM with m*k <= 64 rounds exactly like
the reference (bit-identical); larger shapes use FMA and agree within 1e-12.
TSMTTSM reductions run in a different (fixed) order: 1e-12 relative to sum |v||w|."""
import ctypes as C

import numpy as np
import pytest

from paper_1507_08101_b200 import sellkit

pytestmark = pytest.mark.gpu


def run_tsmttsm(sk, V, W, X0, alpha, beta, kahan=False):
    x, v, w = sk.densemat_from(X0), sk.densemat_from(V), sk.densemat_from(W)
    a = np.atleast_1d(np.asarray(alpha, V.dtype))
    b = np.atleast_1d(np.asarray(beta, V.dtype))
    sk.call("sellkit_tsmttsm", x.h, v.h, w.h, a.ctypes.data, b.ctypes.data, 1 if kahan else 0)
    return x.copy_out()


def run_tsmm(sk, V, X, W0, alpha, beta):
    w, v, x = sk.densemat_from(W0), sk.densemat_from(V), sk.densemat_from(X)
    a = np.atleast_1d(np.asarray(alpha, V.dtype))
    b = np.atleast_1d(np.asarray(beta, V.dtype))
    sk.call("sellkit_tsmm", w.h, v.h, x.h, a.ctypes.data, b.ctypes.data)
    return w.copy_out()


def test_tsm_vs_reference_golden(sk, golden):
    g = golden("tsm.npz")
    shapes = sorted({tuple(k.split("|")[:3]) for k in g.files})
    for n, m, k in shapes:
        key = f"{n}|{m}|{k}"
        V, W, X = g[key + "|V"], g[key + "|W"], g[key + "|X"]
        scale = np.abs(V).T @ np.abs(W)
        for a, b in [(1.0, 0.0), (0.5, -1.25)]:
            got = run_tsmttsm(sk, V, W, X, a, b)
            want = g[key + f"|tsmttsm|{a}|{b}"]
            assert np.all(np.abs(got - want) <= 1e-12 * (1 + abs(a) * scale + abs(b) * np.abs(X))), key
            got = run_tsmm(sk, V, X, W, a, b)
            want = g[key + f"|tsmm|{a}|{b}"]
            if int(m) * int(k) <= 64:
                assert np.array_equal(got, want), key
            else:
                assert np.max(np.abs(got - want) / (1 + np.abs(want))) < 1e-12, key


@pytest.mark.parametrize("m,k", [(1, 1), (2, 2), (4, 4), (8, 8), (16, 16), (32, 32), (64, 64), (3, 7), (64, 8),
                                 (8, 64), (1, 64)])
def test_tsm_shapes_vs_oracle(sk, orc, m, k):
    rng = np.random.default_rng(m * 100 + k)
    n = 3000
    V, W, X = rng.uniform(-1, 1, (n, m)), rng.uniform(-1, 1, (n, k)), rng.uniform(-1, 1, (m, k))
    want = orc.tsmttsm(V, W, X, 0.75, 0.5)
    got = run_tsmttsm(sk, V, W, X, 0.75, 0.5)
    scale = np.abs(V).T @ np.abs(W)
    assert np.all(np.abs(got - want) <= 1e-12 * (1 + scale + np.abs(X)))
    W0 = rng.uniform(-1, 1, (n, k))
    want = orc.tsmm(V, X, W0, 1.5, -0.5)
    got = run_tsmm(sk, V, X, W0, 1.5, -0.5)
    if m * k <= 64:
        assert np.array_equal(got, want)
    else:
        assert np.max(np.abs(got - want) / (1 + np.abs(want))) < 1e-12


def test_tsm_complex(sk, orc):
    rng = np.random.default_rng(5)
    n, m, k = 500, 4, 3
    V = rng.uniform(-1, 1, (n, m)) + 1j * rng.uniform(-1, 1, (n, m))
    W = rng.uniform(-1, 1, (n, k)) + 1j * rng.uniform(-1, 1, (n, k))
    X = rng.uniform(-1, 1, (m, k)) + 1j * rng.uniform(-1, 1, (m, k))
    got = run_tsmttsm(sk, V, W, X, 1.0 + 0.5j, 0.25)
    want = orc.tsmttsm(V, W, X, 1.0 + 0.5j, 0.25)  # conjugates V (tsm.hpp:164)
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)
    assert np.allclose(want, (1.0 + 0.5j) * (V.conj().T @ W) + 0.25 * X, rtol=1e-12, atol=1e-12)
    got = run_tsmm(sk, V, X, W, 2.0, 0.5 - 1j)
    want = orc.tsmm(V, X, W, 2.0, 0.5 - 1j)
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


def test_kahan_cancellation(sk):
    # proj/tests/unit_sparse.cpp:625-636
    v = np.ones((3, 1))
    w = np.array([[1e16], [1.0], [-1e16]])
    assert run_tsmttsm(sk, v, w, np.zeros((1, 1)), 1.0, 0.0, kahan=True)[0, 0] == 1.0


@pytest.mark.parametrize("m,k", [(1, 1), (2, 4), (4, 4), (4, 8), (8, 8), (3, 7), (16, 16)])
def test_kahan_shapes(sk, orc, m, k):
    """Kahan TSMTTSM on every kernel it routes to (register kernel up to 32 cells, the
    shared-memory tile kernel for 8 x 8 and wider): the cancellation KAT in every cell, and
    random data against the oracle's compensated sums."""
    v = np.ones((3, m))
    w = np.tile(np.array([[1e16], [1.0], [-1e16]]), (1, k))
    assert np.array_equal(run_tsmttsm(sk, v, w, np.zeros((m, k)), 1.0, 0.0, kahan=True), np.ones((m, k)))
    rng = np.random.default_rng(m * 31 + k)
    n = 5000
    V, W, X = rng.uniform(-1, 1, (n, m)), rng.uniform(-1, 1, (n, k)), rng.uniform(-1, 1, (m, k))
    want = orc.tsmttsm(V, W, X, 0.75, 0.5, kahan=True)
    got = run_tsmttsm(sk, V, W, X, 0.75, 0.5, kahan=True)
    assert np.all(np.abs(got - want) <= 1e-12 * (1 + np.abs(V).T @ np.abs(W) + np.abs(X)))


def test_tsmm_inplace_and_gemm(sk, orc):
    rng = np.random.default_rng(8)
    n, m = 700, 6
    V, X = rng.uniform(-1, 1, (n, m)), rng.uniform(-1, 1, (m, m))
    v, x = sk.densemat_from(V), sk.densemat_from(X)
    a, b = np.array([0.5]), np.array([2.0])
    sk.call("sellkit_tsmm_inplace", v.h, x.h, a.ctypes.data, b.ctypes.data)
    want = orc.tsmm_inplace(V, X, 0.5, 2.0)
    assert np.max(np.abs(v.copy_out() - want) / (1 + np.abs(want))) < 1e-12
    # gemm routing (tsm.hpp:281-305): A^T B -> tsmttsm, A X -> tsmm, else naive
    A, B = rng.uniform(-1, 1, (200, 5)), rng.uniform(-1, 1, (200, 3))
    c = sk.densemat(5, 3)
    sk.call("sellkit_gemm", c, sk.densemat_from(A), sk.densemat_from(B), None, None, sellkit.TRANS_T,
            sellkit.TRANS_NONE)
    assert np.allclose(c.copy_out(), A.T @ B, rtol=1e-12, atol=1e-12)
    S = rng.uniform(-1, 1, (5, 5))
    c2 = sk.densemat(200, 5)
    sk.call("sellkit_gemm", c2, sk.densemat_from(A), sk.densemat_from(S), None, None, sellkit.TRANS_NONE,
            sellkit.TRANS_NONE)
    assert np.allclose(c2.copy_out(), A @ S, rtol=1e-12, atol=1e-12)
    P, Q = rng.uniform(-1, 1, (30, 40)), rng.uniform(-1, 1, (30, 20))
    c3 = sk.densemat(40, 20)
    sk.call("sellkit_gemm", c3, sk.densemat_from(P), sk.densemat_from(Q), None, None, sellkit.TRANS_T,
            sellkit.TRANS_NONE)
    assert np.allclose(c3.copy_out(), P.T @ Q, rtol=1e-12, atol=1e-12)


def test_tsm_shape_errors(sk):
    v, w, x = sk.densemat(10, 2), sk.densemat(11, 3), sk.densemat(2, 3)
    with pytest.raises(sellkit.SellkitError) as e:
        sk.call("sellkit_tsmttsm", x.h, v.h, w.h, None, None, 0)
    assert e.value.code == sellkit.ERR_SHAPE
    with pytest.raises(sellkit.SellkitError) as e:
        sk.call("sellkit_tsmm", v, v, sk.densemat(2, 2), None, None)
    assert e.value.code == sellkit.ERR_INVALID_ARG  # V and W must be distinct


def test_blas1(sk, orc):
    rng = np.random.default_rng(12)
    X, Y = rng.uniform(-1, 1, (1000, 3)), rng.uniform(-1, 1, (1000, 3))
    y, x = sk.densemat_from(Y), sk.densemat_from(X)
    a, b = np.array([1.5]), np.array([-0.25])
    sk.call("sellkit_axpby", y.h, x.h, a.ctypes.data, b.ctypes.data)
    assert np.array_equal(y.copy_out(), 1.5 * X + (-0.25) * Y)  # densemat.hpp:247, exact rounding
    al, be = np.array([1.0, 2.0, 3.0]), np.array([0.5, 0.25, 0.125])
    y2 = sk.densemat_from(Y)
    sk.call("sellkit_vaxpby", y2.h, x.h, al.ctypes.data, be.ctypes.data)
    assert np.array_equal(y2.copy_out(), al * X + be * Y)
    y3 = sk.densemat_from(Y)
    sk.call("sellkit_vscal", y3.h, al.ctypes.data)
    assert np.array_equal(y3.copy_out(), Y * al)
    out = np.zeros(3)
    sk.call("sellkit_dot", sk.densemat_from(X), sk.densemat_from(Y), out.ctypes.data)
    want = orc.dot(X, Y)
    assert np.all(np.abs(out - want) <= 1e-12 * (1 + np.abs(X * Y).sum(0)))
    # views / scattered / convert_order (unit_capi.cpp:116-151)
    m = sk.densemat_from(np.arange(16.0).reshape(4, 4))
    cols = (C.c_int32 * 2)(0, 2)
    vh = C.c_void_p()
    sk.call("sellkit_densemat_view", m.h, 0, 4, cols, 2, C.byref(vh))
    assert sk.lib.sellkit_densemat_is_scattered(vh) == 1
    ch = C.c_void_p()
    sk.call("sellkit_densemat_compact_clone", vh, C.byref(ch))
    cv = np.zeros(8)
    sk.call("sellkit_densemat_copy_out", ch, cv.ctypes.data, 8)
    assert cv.tolist() == [0, 2, 4, 6, 8, 10, 12, 14]
    conv = C.c_void_p()
    sk.call("sellkit_densemat_convert_order", ch, sellkit.COL_MAJOR, 0, C.byref(conv))
    cc = np.zeros(8)
    sk.call("sellkit_densemat_copy_out", conv, cc.ctypes.data, 8)
    assert cc.tolist() == cv.tolist()
    for h in (vh, ch, conv):
        sk.lib.sellkit_densemat_destroy(h)


def test_sharded_tsm_wrappers_single_rank(sk, orc):
    """dist.tsmttsm / dist.tsmm at world size 1 equal the local kernels."""
    from paper_1507_08101_b200 import dist
    rng = np.random.default_rng(9)
    n, m, k = 5000, 16, 8
    V, W, X = rng.uniform(-1, 1, (n, m)), rng.uniform(-1, 1, (n, k)), rng.uniform(-1, 1, (m, k))
    x, v, w = sk.densemat_from(X), sk.densemat_from(V), sk.densemat_from(W)
    dist.tsmttsm(sk, x, v, w, alpha=0.75, beta=0.5)
    want = orc.tsmttsm(V, W, X, 0.75, 0.5)
    scale = np.abs(V).T @ np.abs(W)
    assert np.all(np.abs(x.copy_out() - want) <= 1e-12 * (1 + scale + np.abs(X)))
    w2 = sk.densemat_from(W)
    xs = sk.densemat_from(X[:m, :k])
    dist.tsmm(sk, w2, v, xs, alpha=1.5, beta=-0.5)
    assert np.max(np.abs(w2.copy_out() - (1.5 * V @ X - 0.5 * W)) / (1 + np.abs(W))) < 1e-12


@pytest.mark.parametrize("m,k", [(32, 32), (64, 64), (32, 64), (64, 32), (16, 64)])
@pytest.mark.parametrize("n", [5, 1001, 70001])
def test_tsm_tensor_core_ragged_rows(sk, orc, m, k, n):
    # DMMA kernels with bulk-copied row tiles: short last tiles, one-tile ranges
    rng = np.random.default_rng(n + m * 7 + k)
    V, W, X = rng.uniform(-1, 1, (n, m)), rng.uniform(-1, 1, (n, k)), rng.uniform(-1, 1, (m, k))
    want = orc.tsmttsm(V, W, X, 1.25, -0.5) if n < 5000 else 1.25 * (V.T @ W) - 0.5 * X
    got = run_tsmttsm(sk, V, W, X, 1.25, -0.5)
    scale = np.abs(V).T @ np.abs(W)
    assert np.all(np.abs(got - want) <= 1e-12 * (1 + scale + np.abs(X)))
    W0 = rng.uniform(-1, 1, (n, k))
    want = orc.tsmm(V, X, W0, 1.5, 0.0) if n < 5000 else 1.5 * (V @ X)
    got = run_tsmm(sk, V, X, W0, 1.5, 0.0)
    assert np.max(np.abs(got - want) / (1 + np.abs(V) @ np.abs(X))) < 1e-12


@pytest.mark.parametrize("mk", [1, 2])
@pytest.mark.parametrize("n", [1, 3, 5, 1003, 4097, 300001])
def test_tsm_chunked_narrow_ragged(sk, orc, mk, n):
    """The 1 x 1 / 2 x 2 paths move R = 4 / 2 rows per 32-byte access; row counts that are
    not multiples of R (and of the CTA ranges) end in a per-row tail.  TSMM stays
    bit-identical to the reference order, TSMTTSM within 1e-12 * sum |v||w|."""
    rng = np.random.default_rng(7 * n + mk)
    V, W, X = rng.uniform(-1, 1, (n, mk)), rng.uniform(-1, 1, (n, mk)), rng.uniform(-1, 1, (mk, mk))
    want = orc.tsmttsm(V, W, X, 0.75, 0.5)
    got = run_tsmttsm(sk, V, W, X, 0.75, 0.5)
    scale = np.abs(V).T @ np.abs(W)
    assert np.all(np.abs(got - want) <= 1e-12 * (1 + scale + np.abs(X)))
    W0 = rng.uniform(-1, 1, (n, mk))
    for a, b in [(1.5, -0.5), (2.0, 0.0)]:
        assert np.array_equal(run_tsmm(sk, V, X, W0, a, b), orc.tsmm(V, X, W0, a, b))
