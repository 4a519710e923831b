"""Sweep orders for structured-grid matrices (used with Mat.set_sweep_order /
sellkit_ext_mat_set_sweep_order).

A row-ordered sweep of a 3-D lattice re-reads the RHS of a z-plane after a
whole plane of rows: for the C3 topological-insulator lattice (2^24 rows, w=16,
complex) that window is 67 MB of x plus the y/matrix streams, more than L2 keeps,
so x comes from HBM three times.  A *pencil* order sweeps all z for a slab of
`yb` y-lines before moving on, shrinking the z-reuse window to yb x-lines.  The
result of the product does not depend on the order (each row is computed
independently); only the dot-product summation order changes.
"""
from __future__ import annotations

import numpy as np


def pencil_order(lx: int, ly: int, lz: int, per_site: int = 1, block_rows: int = 256, yb: int = 16) -> np.ndarray:
    """Block order for rows numbered row = per_site * ((z*ly + y)*lx + x) + orbital.

    Blocks of `block_rows` consecutive rows must not straddle an x-line:
    (lx * per_site) % block_rows == 0.  Returns the permutation of block indices
    for y-slabs of `yb` lines, z, y, x-blocks (innermost last)."""
    line = lx * per_site
    if line % block_rows:
        raise ValueError("block_rows must divide an x-line of rows")
    bpl = line // block_rows                      # blocks per x-line
    yb = max(1, min(yb, ly))
    order = []
    for y0 in range(0, ly, yb):
        ys = np.arange(y0, min(ly, y0 + yb))
        z, y, xq = np.meshgrid(np.arange(lz), ys, np.arange(bpl), indexing="ij")
        order.append(((z * ly + y) * bpl + xq).reshape(-1))
    return np.concatenate(order).astype(np.int32)
