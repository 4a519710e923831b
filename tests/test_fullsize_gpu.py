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
