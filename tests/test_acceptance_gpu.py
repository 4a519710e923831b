"""The reference's acceptance gate (proj/tests/acceptance.cpp), criterion by criterion,
run against the B200 library through the C ABI.  Tolerances are the gate's own
(1e-12 relative); criteria 4-7 and 9 live in test_tsm_gpu.py, test_dist_*.py,
test_capi_cpu.py and test_cli.py (criterion 6, the task-pool scheduler, is host-CPU
scheduling and out of scope: DESIGN.md section 7)."""
import numpy as np
import pytest

from oracle.oracle import random_crs
from paper_1507_08101_b200 import sellkit

pytestmark = pytest.mark.gpu

EX_ROWPTR, EX_COL, EX_VAL = [0, 1, 3, 4, 7], [0, 0, 1, 2, 1, 2, 3], np.arange(1, 8, dtype=float)


def crs_spmv(rp, c, v, x):
    """Plain CRS y = A x on a row-major block (oracles.hpp crs_spmv), rows in logical order."""
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    y = np.zeros((len(rp) - 1, x.shape[1]), dtype=np.result_type(v, x))
    np.add.at(y, rows, v[:, None] * x[c])
    return y


def max_rel_err(got, want):
    """oracles.hpp max_rel_err: max |got - want| / max(1, |want|)."""
    return float(np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want)), initial=0.0))


def to_storage(A, arr):
    """Logical rows -> the SELL storage order (acceptance.cpp:44-57)."""
    perm = A.export()["row_perm"]
    out = np.empty_like(arr)
    out[perm] = arr
    return out, perm


def test_criterion_1_spmv_oracle_equivalence(sk):
    """acceptance.cpp:70-92: 200 random matrices, C in {1,2,4,8,32}, sigma in {1,C,4C,n}."""
    rng = np.random.default_rng(1001)
    worst = 0.0
    for _ in range(200):
        n = int(10 + rng.integers(0, 191))
        density = 0.02 + 0.18 * int(rng.integers(0, 100)) / 100.0
        rp, c, v = random_crs(rng, n, n, density)
        x = rng.uniform(-1, 1, (n, 1))
        want = crs_spmv(rp, c, v, x)
        crs = sk.crs(rp, c, v, n)
        for C in (1, 2, 4, 8, 32):
            for sigma in sorted({1, C, 4 * C, n}):
                A = crs.build(C, sigma)
                xs, perm = to_storage(A, x)
                xd, yd = sk.densemat_from(xs), sk.densemat(n, 1)
                sk.spmv(yd, A, xd)
                worst = max(worst, max_rel_err(yd.copy_out()[perm], want))
    assert worst <= 1e-12, worst


def test_criterion_2_fused_equals_unfused_composition(sk):
    """acceptance.cpp:96-168: every flag set (SHIFT and VSHIFT exclusive), widths 1-4,
    SELL-4-8, against the unfused composition (oracles.hpp fused_spmv)."""
    rng = np.random.default_rng(2002)
    worst = 0.0
    alpha, beta, delta, eta = 1.1, -0.6, 0.3, 1.7
    for _ in range(20):
        n = int(20 + rng.integers(0, 80))
        w = int(1 + rng.integers(0, 4))
        rp, c, v = random_crs(rng, n, n, 0.1)
        A = sk.crs(rp, c, v, n).build(4, 8)
        xv, yv, zv = (rng.uniform(-1, 1, (n, w)) for _ in range(3))
        gammas = -2.0 + rng.integers(0, 100, w) / 25.0
        ax = crs_spmv(rp, c, v, xv)
        for flags in range(1 << 7):
            if (flags & sellkit.SHIFT) and (flags & sellkit.VSHIFT):
                continue
            xs, perm = to_storage(A, xv)
            ys, _ = to_storage(A, yv)
            zs, _ = to_storage(A, zv)
            x, y, z = sk.densemat_from(xs), sk.densemat_from(ys), sk.densemat_from(zs)
            dots = np.zeros(3 * w)
            gamma = gammas if flags & sellkit.VSHIFT else gammas[0]
            sk.spmv(y, A, x, flags=flags, alpha=alpha, beta=beta, gamma=gamma, delta=delta, eta=eta, z=z,
                    dot=dots)
            # the unfused composition
            g = np.zeros(w)
            if flags & sellkit.SHIFT:
                g[:] = gammas[0]
            if flags & sellkit.VSHIFT:
                g = gammas
            t = ax.copy()
            if flags & (sellkit.SHIFT | sellkit.VSHIFT):
                t = t - g * xv
            t = t * alpha
            if flags & sellkit.AXPBY:
                t = t + beta * yv
            zr = delta * zv + eta * t if flags & sellkit.CHAIN_AXPBY else zv
            worst = max(worst, max_rel_err(y.copy_out()[perm], t), max_rel_err(z.copy_out()[perm], zr))
            for k, (flag, a_, b_) in enumerate([(sellkit.DOT_YY, t, t), (sellkit.DOT_XY, xv, t),
                                                (sellkit.DOT_XX, xv, xv)]):
                if flags & flag:
                    want = np.sum(a_ * b_, axis=0)
                    worst = max(worst, max_rel_err(dots[k * w:(k + 1) * w], want))
    assert worst <= 1e-12, worst


def test_criterion_3_sell_special_cases(sk):
    """acceptance.cpp:172-210: SELL-1-1 is CRS, SELL-n-1 is one chunk, worked 4x4 betas."""
    crs = sk.crs(EX_ROWPTR, EX_COL, EX_VAL)
    L = crs.build(1, 1).export()
    assert np.array_equal(L["val"], EX_VAL)
    assert np.array_equal(L["col"], np.array(EX_COL, np.int32))
    assert np.array_equal(L["chunk_offset"], np.array(EX_ROWPTR, np.int64))
    A = crs.build(4, 1)
    assert A.info()["nchunks"] == 1 and A.export()["chunk_len"][0] == 3
    assert crs.build(2, 4).stats()[0] == 0.875
    assert crs.build(2, 1).stats()[0] == 0.7


def test_criterion_8_bit_exact_determinism(sk, tmp_path):
    """acceptance.cpp:465-505: the same input builds the same layout every time, and the
    SpMV result does not depend on the run; binary io round-trips bit for bit."""
    rng = np.random.default_rng(8008)
    rp, c, v = random_crs(rng, 3000, 3000, 0.004)
    crs = sk.crs(rp, c, v)
    layouts = [crs.build(32, 128).export() for _ in range(3)]
    for L in layouts[1:]:
        for k in layouts[0]:
            assert np.array_equal(L[k], layouts[0][k]), k
    A = crs.build(32, 128)
    x = sk.densemat_from(rng.uniform(-1, 1, (3000, 4)))
    outs = []
    for _ in range(3):
        y = sk.densemat(3000, 4)
        sk.spmv(y, A, x)
        outs.append(y.copy_out())
    assert all(np.array_equal(o.view(np.uint64), outs[0].view(np.uint64)) for o in outs[1:])
    path = str(tmp_path / "m.gcrs")
    crs.write_bin(path)
    L2 = sk.crs_read_bin(path).build(32, 128).export()
    for k in layouts[0]:
        assert np.array_equal(L2[k], layouts[0][k]), k
