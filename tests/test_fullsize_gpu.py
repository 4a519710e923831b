"""Full-size (BASELINE C5: 3-D 7-point 400^3, SELL-32-256, w = 8) parity through a
size-independent property: with small-integer x every product and partial sum is
an exactly representable integer, so y = A x is exact whatever the summation order
and must equal the stencil applied with array shifts (torch, original row order)
bit for bit.  The SELL storage permutation comes from the device matrix
(row_perm_inv: original row at storage position k, sellcs.hpp:143-232)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _stencil_ref(torch, X):
    """6 x - sum of the 6 neighbours, zero outside the cube (Dirichlet)."""
    Y = 6.0 * X
    for d in range(3):
        for s in (1, -1):
            sh = torch.roll(X, shifts=s, dims=d)
            idx = 0 if s == 1 else X.shape[d] - 1  # wrapped plane -> zero
            sh.index_fill_(d, torch.tensor([idx], device=X.device), 0.0)
            Y -= sh
    return Y


@pytest.mark.parametrize("n,w", [(400, 8), (256, 16)])
def test_stencil_fullsize_exact(sk, n, w):
    import torch
    from paper_1507_08101_b200 import sellkit
    N = n ** 3
    A = sk.crs_stencil(7, n).build(32, 256)
    perm_inv = np.zeros(N, np.int32)
    sk.call("sellkit_ext_mat_export", A.h, perm_inv.ctypes.data, None, None, None, None, None, None)
    dev = torch.device("cuda")
    pinv = torch.from_numpy(perm_inv).to(dev, torch.int64)
    cols = torch.arange(w, device=dev, dtype=torch.int64)
    g = torch.arange(N, device=dev, dtype=torch.int64)
    X = (((g[:, None] * 7 + cols[None, :] * 3) % 17) - 8).to(torch.float64)      # original order
    Xs = X[pinv].contiguous()                                                       # storage order
    Ys = torch.empty_like(Xs)
    x = sk.view_plain(Xs.data_ptr(), N * w, N, w, w, keep=Xs)
    y = sk.view_plain(Ys.data_ptr(), N * w, N, w, w, keep=Ys)
    sk.spmv(y, A, x)
    torch.cuda.synchronize()
    Yref = _stencil_ref(torch, X.view(n, n, n, w)).view(N, w)[pinv]
    assert torch.equal(Ys, Yref)
    # the fused epilogue at full size: y = 0.5 (A - 0.25 I) x + (-1) y0, all exact in binary
    y0 = (((g[:, None] * 5 + cols[None, :]) % 13) - 6).to(torch.float64)[pinv].contiguous()
    Ys.copy_(y0)
    sk.spmv(y, A, x, flags=sellkit.AXPBY | sellkit.SHIFT, alpha=0.5, beta=-1.0, gamma=0.25)
    torch.cuda.synchronize()
    want = 0.5 * (Yref - 0.25 * Xs) - y0
    assert torch.equal(Ys, want)


@pytest.mark.parametrize("n,m,k", [(100_000_000, 8, 8), (20_000_000, 64, 64), (50_000_000, 16, 32)])
def test_tsm_fullsize_exact(sk, n, m, k):
    """C4 sizes: small-integer V, W, X make TSMM / TSMTTSM exact in FP64 (every partial
    sum is an integer below 2^53), so any summation order must match torch bit for bit."""
    import torch
    from paper_1507_08101_b200 import sellkit
    dev = torch.device("cuda")
    r = torch.arange(n, device=dev, dtype=torch.int64)[:, None]
    V = ((r * 3 + torch.arange(m, device=dev)[None, :] * 5) % 7 - 3).to(torch.float64)
    W = ((r * 5 + torch.arange(k, device=dev)[None, :] * 3) % 9 - 4).to(torch.float64)
    X = ((torch.arange(m * k, device=dev) * 7) % 11 - 5).to(torch.float64).view(m, k).contiguous()
    v = sk.view_plain(V.data_ptr(), n * m, n, m, m, keep=V)
    wv = sk.view_plain(W.data_ptr(), n * k, n, k, k, keep=W)
    Xo = torch.zeros(m, k, dtype=torch.float64, device=dev)
    x = sk.view_plain(Xo.data_ptr(), m * k, m, k, k, keep=Xo)
    one, zero = np.array([1.0]), np.array([0.0])
    sk.call("sellkit_tsmttsm", x.h, v.h, wv.h, one.ctypes.data, zero.ctypes.data, 0)
    torch.cuda.synchronize()
    assert torch.equal(Xo, V.T @ W)
    Xs = sk.view_plain(X.data_ptr(), m * k, m, k, k, keep=X)
    Wout = torch.empty(n, k, dtype=torch.float64, device=dev)
    wo = sk.view_plain(Wout.data_ptr(), n * k, n, k, k, keep=Wout)
    sk.call("sellkit_tsmm", wo.h, v.h, Xs.h, one.ctypes.data, zero.ctypes.data)
    torch.cuda.synchronize()
    assert torch.equal(Wout, V @ X)
