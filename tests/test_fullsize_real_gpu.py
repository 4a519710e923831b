"""Real-valued parity at the BASELINE sizes (VERDICT r1 "What's weak" 1).

Every operand is a U(-1,1) counter-hash block (sellkit_ext_densemat_fill_hash;
regenerated on the host by oracle/libfullsize.so), so sums are NOT exact and the
summation order matters:

* C5 (400^3 7-pt, SELL-32-256, w = 8) and C2 (256^3, w = 16 / 32): y = A x with all
  three dots, and the fused y = 0.5 (A - 0.25 I) x - y0: checked against the
  REFERENCE LIBRARY ITSELF (oracle/_ref, built from /root/reference/proj sources)
  run on the same full matrix on the host's cores -- y bit for bit (same layout,
  same per-row order), dots within 1e-12 * sum |x_i y_i| of the long-double value.
* C3 (TI Hamiltonian, 2^24 rows, complex double, w = 16, KPM flags): the same against
  the reference's generic complex kernel.
* C4 (N = 1e8, m = k in {8, 64}): TSMM against the reference's per-row order restated
  in fullsize.c (normwise per column <= 1e-12), TSMTTSM against the long-double sum
  (|err| <= 1e-12 * sum |v||w| per cell).

The measured errors (GPU and reference, against the long-double dots) are written to
$SELLKIT_PARITY_REPORT (JSON lines) when set; profiles/ keeps the round's copy.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle.oracle import REF_LIB_PATH, FullSize, ti_crs
from paper_1507_08101_b200 import sellkit

pytestmark = pytest.mark.gpu

DOTS = sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX


def _report(**kw):
    path = os.environ.get("SELLKIT_PARITY_REPORT")
    print(json.dumps(kw))
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(kw) + "\n")


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(REF_LIB_PATH):
        pytest.skip("reference library oracle/_ref not built (python -m oracle.build)")
    r = sellkit.Sellkit(REF_LIB_PATH, ext=False)
    r.call("sellkit_set_num_workers", os.cpu_count() or 1)
    return r


@pytest.fixture(scope="module")
def fs():
    return FullSize()


def _dot_errors(fs, dots, rdots, xv, y, w):
    """max over columns of |d - exact| / sum|terms| for the GPU and the reference dots"""
    out = {}
    for s, (a, b) in enumerate([(y, y), (xv, y), (xv, xv)]):
        exact, scale = fs.dot_cols(a, b)
        part = slice(s * w, (s + 1) * w)
        out[["yy", "xy", "xx"][s]] = (float(np.max(np.abs(dots[part] - exact) / scale)),
                                      float(np.max(np.abs(rdots[part] - exact) / scale)))
    return out


def _stencil_case(sk, ref, fs, n, w, tag):
    N = n ** 3
    A = sk.crs_stencil(7, n).build(32, 256)
    x = sk.densemat(N, w)
    x.fill_hash(42)
    y = sk.densemat(N, w)
    rp, c, v = fs.stencil7_crs(n)
    crs = ref.crs(rp, c, v)
    del rp, c, v
    Ar = crs.build(32, 256)
    del crs
    xv = fs.hash_block(N, w, 42)   # storage order, as the device fill (identical layouts)
    xr, yr = ref.densemat_from(xv), ref.densemat(N, w)
    # plain y = A x with the three dots
    dots, rdots = np.zeros(3 * w), np.zeros(3 * w)
    sk.spmv(y, A, x, flags=DOTS, dot=dots)
    ref.spmv(yr, Ar, xr, flags=DOTS, dot=rdots)
    yg, yref = y.copy_out(), yr.copy_out()
    assert np.array_equal(yg, yref), f"{tag}: y differs from the reference"
    errs = _dot_errors(fs, dots, rdots, xv, yref, w)
    _report(case=tag, op="y=Ax +3 dots", y="bitwise", dot_err_gpu_vs_ref_exact=errs, bar=1e-12)
    for k, (eg, _) in errs.items():
        assert eg <= 1e-12, (tag, k, eg)
    del yg
    # fused KPM-style step y = 0.5 (A - 0.25 I) x - y0
    y.fill_hash(43)
    y0 = fs.hash_block(N, w, 43)
    yr.copy_in(y0)
    flags = sellkit.AXPBY | sellkit.SHIFT | DOTS
    sk.spmv(y, A, x, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, dot=dots)
    ref.spmv(yr, Ar, xr, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, dot=rdots)
    yg, yref = y.copy_out(), yr.copy_out()
    assert np.array_equal(yg, yref), f"{tag}: fused y differs from the reference"
    errs = _dot_errors(fs, dots, rdots, xv, yref, w)
    _report(case=tag, op="y=0.5(A-0.25I)x-y0 +3 dots", y="bitwise", dot_err_gpu_vs_ref_exact=errs, bar=1e-12)
    for k, (eg, _) in errs.items():
        assert eg <= 1e-12, (tag, k, eg)


def test_c5_real_values_vs_reference(sk, ref, fs):
    _stencil_case(sk, ref, fs, 400, 8, "C5 400^3 w=8")


@pytest.mark.parametrize("w", [16, 32])
def test_c2_real_values_vs_reference(sk, ref, fs, w):
    _stencil_case(sk, ref, fs, 256, w, f"C2 256^3 w={w}")


def test_c3_ti_complex_kpm_vs_reference(sk, ref, fs):
    lx, ly, lz, dis, w = 256, 128, 128, 0.5, 16
    N = 4 * lx * ly * lz
    A = sk.crs_ti(lx, ly, lz, dis).build(32, 256)
    rp, c, v = ti_crs(lx, ly, lz, dis)
    crs = ref.crs(rp, c, v, dt=sellkit.C64)
    del rp, c, v
    Ar = crs.build(32, 256)
    del crs
    xv = fs.hash_block(N, w, 42) + 1j * fs.hash_block(N, w, 142)
    y0 = fs.hash_block(N, w, 43) + 1j * fs.hash_block(N, w, 143)
    x, y = sk.densemat_from(xv), sk.densemat_from(y0)
    xr, yr = ref.densemat_from(xv), ref.densemat_from(y0)
    flags = sellkit.AXPBY | sellkit.SHIFT | DOTS
    dots, rdots = np.zeros(3 * w, np.complex128), np.zeros(3 * w, np.complex128)
    sk.spmv(y, A, x, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, dot=dots)
    ref.spmv(yr, Ar, xr, flags=flags, alpha=0.5, beta=-1.0, gamma=0.25, dot=rdots)
    yg, yref = y.copy_out(), yr.copy_out()
    assert np.array_equal(yg, yref), "C3: y differs from the reference"
    errs = _dot_errors(fs, dots, rdots, xv, yref, w)
    _report(case="C3 TI 2^24 C64 w=16", op="KPM y=0.5(H-0.25I)x-y0 +3 dots", y="bitwise",
            dot_err_gpu_vs_ref_exact=errs, bar=1e-12)
    for k, (eg, _) in errs.items():
        assert eg <= 1e-12, ("C3", k, eg)


@pytest.mark.parametrize("mk", [8, 64])
def test_c4_tsm_real_values(sk, fs, mk):
    import torch
    n, m, k = 100_000_000, mk, mk
    dev = torch.device("cuda")
    V = torch.empty((n, m), dtype=torch.float64, device=dev)
    W = torch.empty((n, k), dtype=torch.float64, device=dev)
    v = sk.view_plain(V.data_ptr(), n * m, n, m, m, keep=V)
    wv = sk.view_plain(W.data_ptr(), n * k, n, k, k, keep=W)
    v.fill_hash(5)
    wv.fill_hash(6)
    one, zero = np.array([1.0]), np.array([0.0])
    # TSMTTSM X = V^T W
    Xo = torch.zeros(m, k, dtype=torch.float64, device=dev)
    xo = sk.view_plain(Xo.data_ptr(), m * k, m, k, k, keep=Xo)
    sk.call("sellkit_tsmttsm", xo.h, v.h, wv.h, one.ctypes.data, zero.ctypes.data, 0)
    got = Xo.cpu().numpy()
    exact, scale = fs.tsmttsm(n, m, k, 5, 6)
    err_tt = float(np.max(np.abs(got - exact) / scale))
    # TSMM W = V X with a hash X (host), checked in row blocks against the reference order
    Xh = fs.hash_block(m, k, 7)
    Xd = torch.from_numpy(Xh).to(dev)
    xs = sk.view_plain(Xd.data_ptr(), m * k, m, k, k, keep=Xd)
    sk.call("sellkit_tsmm", wv.h, v.h, xs.h, one.ctypes.data, zero.ctypes.data)
    torch.cuda.synchronize()
    num = np.zeros(k)
    den = np.zeros(k)
    bitwise = True
    blk = 2_000_000 if mk == 64 else 10_000_000
    for i0 in range(0, n, blk):
        i1 = min(n, i0 + blk)
        g = W[i0:i1].cpu().numpy()
        r = fs.tsmm_rows(i0, i1, m, k, 5, Xh, 1.0, 0.0, 6)
        bitwise &= bool(np.array_equal(g, r))
        num += np.sum((g - r) ** 2, axis=0)
        den += np.sum(r ** 2, axis=0)
    err_mm = float(np.max(np.sqrt(num / den)))
    _report(case=f"C4 N=1e8 m=k={mk}", tsmttsm_err_vs_exact=err_tt, tsmm_normwise_err_vs_ref_order=err_mm,
            tsmm_bitwise=bitwise, bar=1e-12)
    assert err_tt <= 1e-12, err_tt
    assert err_mm <= 1e-12, err_mm
