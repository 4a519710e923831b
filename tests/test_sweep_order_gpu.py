"""Sweep order (sellkit_ext_mat_set_sweep_order): results independent of the block
order (y, z bit-identical; dots within the dot tolerance), argument checks."""
import numpy as np
import pytest

from oracle.oracle import hash_block
from paper_1507_08101_b200 import sellkit
from paper_1507_08101_b200.orders import pencil_order

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dt,w", [(sellkit.C64, 16), (sellkit.R64, 16), (sellkit.R64, 8), (sellkit.R64, 1)])
def test_pencil_order_same_result(sk, dt, w):
    lx, ly, lz = 64, 16, 16
    N = 4 * lx * ly * lz
    A = sk.crs_ti(lx, ly, lz, 1.0, dt=dt).build(32, 256)
    npdt = sellkit.NP_DTYPE[dt]
    xv = hash_block(N, w, 42).astype(npdt)
    y0 = hash_block(N, w, 43).astype(npdt)
    flags = sellkit.AXPBY | sellkit.SHIFT | sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX

    def run():
        x, y = sk.densemat_from(xv), sk.densemat_from(y0)
        d = np.zeros(3 * w, npdt)
        sk.spmv(y, A, x, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, dot=d)
        y2 = sk.densemat(N, w, dt)
        sk.spmv(y2, A, x)
        return y.copy_out(), y2.copy_out(), d
    ya, pa, da = run()
    A.set_sweep_order(256, pencil_order(lx, ly, lz, per_site=4, block_rows=256, yb=4))
    yb_, pb, db = run()
    assert np.array_equal(ya, yb_) and np.array_equal(pa, pb)
    scale = np.concatenate([np.sum(np.abs(ya) ** 2, 0), np.sum(np.abs(xv) * np.abs(ya), 0),
                            np.sum(np.abs(xv) ** 2, 0)])
    assert np.all(np.abs(da - db) <= 1e-12 * (1 + scale))
    A.set_sweep_order(256, None)
    yc, pc, _ = run()
    assert np.array_equal(ya, yc) and np.array_equal(pa, pc)


def test_sweep_order_checks(sk):
    A = sk.crs_stencil(7, 16).build(32, 256)  # 4096 rows -> 16 blocks of 256
    with pytest.raises(sellkit.SellkitError):
        A.set_sweep_order(256, np.arange(15))             # wrong count
    with pytest.raises(sellkit.SellkitError):
        A.set_sweep_order(256, np.zeros(16))              # not a permutation
    with pytest.raises(sellkit.SellkitError):
        A.set_sweep_order(100, np.arange(41))             # not a multiple of 32
    A.set_sweep_order(256, np.arange(16)[::-1])
    x = sk.densemat(4096, 8)
    x.fill_hash(1)
    y1, y2 = sk.densemat(4096, 8), sk.densemat(4096, 8)
    sk.spmv(y1, A, x)
    A.set_sweep_order(256, None)
    sk.spmv(y2, A, x)
    assert np.array_equal(y1.copy_out(), y2.copy_out())


@pytest.mark.parametrize("dt,w", [(sellkit.C64, 16), (sellkit.R64, 16), (sellkit.R64, 32)])
def test_auto_locality_order(sk, dt, w, monkeypatch):
    """The automatic locality order (default policy) engages when the coupling distance
    times the streamed bytes per row exceeds half the L2 (here a 1 MB L2 is assumed via
    SELLKIT_AUTO_ORDER_L2): y bit-identical to the natural order, dots within tolerance."""
    lx, ly, lz = 64, 16, 16
    N = 4 * lx * ly * lz
    npdt = sellkit.NP_DTYPE[dt]
    xv = hash_block(N, w, 42).astype(npdt)
    y0 = hash_block(N, w, 43).astype(npdt)
    flags = sellkit.AXPBY | sellkit.SHIFT | sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX

    def run(A):
        x, y = sk.densemat_from(xv), sk.densemat_from(y0)
        d = np.zeros(3 * w, npdt)
        sk.spmv(y, A, x, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, dot=d)
        return y.copy_out(), d
    A = sk.crs_ti(lx, ly, lz, 1.0, dt=dt).build(32, 256)
    A.set_sweep_order(256, None)                      # natural row order
    yn, dn = run(A)
    monkeypatch.setenv("SELLKIT_AUTO_ORDER_L2", "1000000")
    B = sk.crs_ti(lx, ly, lz, 1.0, dt=dt).build(32, 256)   # default policy: automatic
    ya, da = run(B)
    assert np.array_equal(yn, ya)
    scale = np.concatenate([np.sum(np.abs(yn) ** 2, 0), np.sum(np.abs(xv) * np.abs(yn), 0),
                            np.sum(np.abs(xv) ** 2, 0)])
    assert np.all(np.abs(dn - da) <= 1e-12 * (1 + scale))
