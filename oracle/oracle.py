"""Python side of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module, and only as the checker or the timed reference.

* ``Oracle``: ctypes binding of oracle/liboracle.so, the C restatement of the
  reference's algorithms (sellkit_oracle.c, each function cites the
  reference file:line it follows).
* numpy generators producing CRS arrays identical to the device generators
  (stencils) and to the reference tests' random matrices
  (at least one entry per row, columns ascending; proj/tests/oracles.hpp:91-119).
* ``split_local_remote`` / ``build_context``: the distribution metadata of
  /root/reference/proj/src/partition.hpp:121-286 restated with numpy.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_LIB_PATH = os.path.join(HERE, "_ref", "libsellkit.so")
REFDUMP_PATH = os.path.join(HERE, "_ref", "refdump")

vp = C.c_void_p
i64 = C.c_int64
i32 = C.c_int32


class RefIO:
    """The reference's own file readers/writers (oracle/_ref/libsellkit.so, built
    from /root/reference/proj/src by oracle/Makefile.ref), bound through its C ABI
    (proj/include/sellkit.h:84-87).  Used as the parity checker for the I/O path:
    ``mm_to_gcrs`` / ``gcrs_to_gcrs`` return the reference's GCRS bytes, or the
    reference's error code (an int) when it rejects the file."""

    def __init__(self, path: str = REF_LIB_PATH):
        lib = C.CDLL(path)
        lib.sellkit_crs_read_mm.argtypes = [C.c_char_p, C.c_int, C.POINTER(vp)]
        lib.sellkit_crs_read_mm.restype = C.c_int
        lib.sellkit_crs_read_bin.argtypes = [C.c_char_p, C.POINTER(vp)]
        lib.sellkit_crs_read_bin.restype = C.c_int
        lib.sellkit_crs_write_bin.argtypes = [C.c_char_p, vp, C.c_int]
        lib.sellkit_crs_write_bin.restype = C.c_int
        lib.sellkit_crs_destroy.argtypes = [vp]
        lib.sellkit_crs_destroy.restype = None
        self.lib = lib

    def _write(self, h, out_path: str, wide: bool):
        err = self.lib.sellkit_crs_write_bin(os.fsencode(out_path), h, 1 if wide else 0)
        self.lib.sellkit_crs_destroy(h)
        if err:
            return err
        with open(out_path, "rb") as f:
            return f.read()

    def mm_to_gcrs(self, mm_path: str, dt: int, out_path: str, wide: bool = False):
        h = vp()
        err = self.lib.sellkit_crs_read_mm(os.fsencode(mm_path), dt, C.byref(h))
        return err if err else self._write(h, out_path, wide)

    def gcrs_to_gcrs(self, in_path: str, out_path: str, wide: bool = False):
        h = vp()
        err = self.lib.sellkit_crs_read_bin(os.fsencode(in_path), C.byref(h))
        return err if err else self._write(h, out_path, wide)


class OrSell(C.Structure):
    _fields_ = [("nrows", i32), ("ncols", i32), ("nrows_padded", i32), ("C", i32), ("sigma", i32),
                ("cols_permuted", i32), ("dt", i32), ("nnz", i64), ("nchunks", i64), ("slots", i64),
                ("row_perm_inv", C.POINTER(i32)), ("row_perm", C.POINTER(i32)), ("rowlen", C.POINTER(i32)),
                ("chunk_len", C.POINTER(i32)), ("chunk_offset", C.POINTER(i64)), ("val", C.POINTER(C.c_double)),
                ("col", C.POINTER(i32)), ("beta", C.c_double)]


def _p(a):
    return None if a is None else a.ctypes.data_as(vp)


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    if dtype == np.complex128:
        return np.ctypeslib.as_array(ptr, shape=(2 * n,)).copy().view(np.complex128)
    return np.ctypeslib.as_array(ptr, shape=(n,)).copy()


class SellLayout(dict):
    """SELL arrays as numpy (same keys as sellkit.Mat.export)."""


class Oracle:
    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -f oracle/Makefile`")
        self.lib = C.CDLL(path)
        L = self.lib
        L.or_sigma_permutation.argtypes = [vp, i64, i32, vp]
        L.or_sell_build.argtypes = [C.c_int, i64, i64, vp, vp, vp, i32, i32, C.c_int, vp, C.POINTER(C.POINTER(OrSell))]
        L.or_sell_build.restype = C.c_int
        L.or_sell_free.argtypes = [C.POINTER(OrSell)]
        L.or_spmv.argtypes = [C.POINTER(OrSell), vp, i64, i64, vp, i64, i64, vp, i64, i64, i32, C.c_uint32,
                              vp, vp, vp, vp, vp, vp, vp, C.c_int]
        L.or_tsmttsm.argtypes = [C.c_int, i64, i32, i32, vp, i64, i64, vp, i64, vp, i64, vp, vp, C.c_int, C.c_int]
        L.or_tsmm.argtypes = [C.c_int, i64, i32, i32, vp, i64, vp, i64, vp, i64, i64, vp, vp]
        L.or_tsmm_inplace.argtypes = [C.c_int, i64, i32, vp, i64, vp, i64, i64, vp, vp]
        L.or_dot.argtypes = [C.c_int, i64, i32, vp, i64, i64, vp, i64, i64, vp, C.c_int]
        L.or_partition.argtypes = [i64, vp, vp, C.c_int, C.c_int, vp]
        L.or_partition.restype = C.c_int

    # -- construction -----------------------------------------------------
    def sigma_permutation(self, lens, sigma):
        lens = np.ascontiguousarray(lens, np.int32)
        out = np.zeros(len(lens), np.int32)
        self.lib.or_sigma_permutation(_p(lens), len(lens), sigma, _p(out))
        return out

    def build(self, rowptr, col, val, C_, sigma, ncols=None, permute_columns=True, imposed_order=None):
        """Returns (handle, layout dict).  Raises ValueError(code) on a build error."""
        rowptr = np.ascontiguousarray(rowptr, np.int64)
        col = np.ascontiguousarray(col, np.int64)
        val = np.ascontiguousarray(val)
        dt = 1 if np.iscomplexobj(val) else 0
        val = val.astype(np.complex128 if dt else np.float64)
        nrows = len(rowptr) - 1
        ncols = nrows if ncols is None else ncols
        imp = None if imposed_order is None else np.ascontiguousarray(imposed_order, np.int32)
        out = C.POINTER(OrSell)()
        rc = self.lib.or_sell_build(dt, nrows, ncols, _p(rowptr), _p(col), _p(val), C_, sigma,
                                    1 if permute_columns else 0, _p(imp), C.byref(out))
        if rc != 0:
            raise ValueError(rc)
        return OracleSell(self, out)

    # -- spmv -------------------------------------------------------------
    def spmv(self, A: "OracleSell", x, y=None, z=None, flags=0, alpha=None, beta=None, gamma=None,
             gamma_list=None, delta=None, eta=None, workers=1):
        """Storage-space spmv on row-major numpy blocks (copies); returns (y, z, dots)."""
        cplx = A.s.dt == 1
        dtype = np.complex128 if cplx else np.float64
        x = np.ascontiguousarray(np.atleast_2d(x.T).T if x.ndim == 1 else x, dtype)
        w = x.shape[1]
        y = np.zeros((A.s.nrows, w), dtype) if y is None else np.array(y, dtype, copy=True).reshape(A.s.nrows, w)
        z = None if z is None else np.array(z, dtype, copy=True).reshape(A.s.nrows, w)
        dots = np.zeros(3 * w, dtype)

        def sc(v):
            return None if v is None else np.ascontiguousarray(np.atleast_1d(v), dtype)
        keep = [sc(alpha), sc(beta), sc(gamma), sc(gamma_list), sc(delta), sc(eta)]
        self.lib.or_spmv(A.h, _p(y), w, 1, _p(x), w, 1, _p(z), w, 1, w, flags, *[_p(k) for k in keep],
                         _p(dots), workers)
        return y, z, dots

    def tsmttsm(self, v, w, x=None, alpha=None, beta=None, kahan=False, workers=1):
        cplx = np.iscomplexobj(v)
        dtype = np.complex128 if cplx else np.float64
        v = np.ascontiguousarray(v, dtype)
        w = np.ascontiguousarray(w, dtype)
        n, m = v.shape
        k = w.shape[1]
        x = np.zeros((m, k), dtype) if x is None else np.array(x, dtype, copy=True)
        a = None if alpha is None else np.atleast_1d(np.asarray(alpha, dtype))
        b = None if beta is None else np.atleast_1d(np.asarray(beta, dtype))
        self.lib.or_tsmttsm(1 if cplx else 0, n, m, k, _p(x), k, 1, _p(v), m, _p(w), k, _p(a), _p(b),
                            1 if kahan else 0, workers)
        return x

    def tsmm(self, v, x, w=None, alpha=None, beta=None):
        cplx = np.iscomplexobj(v)
        dtype = np.complex128 if cplx else np.float64
        v = np.ascontiguousarray(v, dtype)
        x = np.ascontiguousarray(x, dtype)
        n, m = v.shape
        k = x.shape[1]
        w = np.zeros((n, k), dtype) if w is None else np.array(w, dtype, copy=True)
        a = None if alpha is None else np.atleast_1d(np.asarray(alpha, dtype))
        b = None if beta is None else np.atleast_1d(np.asarray(beta, dtype))
        self.lib.or_tsmm(1 if cplx else 0, n, m, k, _p(w), k, _p(v), m, _p(x), k, 1, _p(a), _p(b))
        return w

    def tsmm_inplace(self, v, x, alpha=None, beta=None):
        cplx = np.iscomplexobj(v)
        dtype = np.complex128 if cplx else np.float64
        v = np.array(v, dtype, copy=True)
        x = np.ascontiguousarray(x, dtype)
        n, m = v.shape
        a = None if alpha is None else np.atleast_1d(np.asarray(alpha, dtype))
        b = None if beta is None else np.atleast_1d(np.asarray(beta, dtype))
        self.lib.or_tsmm_inplace(1 if cplx else 0, n, m, _p(v), m, _p(x), m, 1, _p(a), _p(b))
        return v

    def dot(self, a, b, workers=1):
        cplx = np.iscomplexobj(a)
        dtype = np.complex128 if cplx else np.float64
        a = np.ascontiguousarray(a, dtype)
        b = np.ascontiguousarray(b, dtype)
        n, w = a.shape
        out = np.zeros(w, dtype)
        self.lib.or_dot(1 if cplx else 0, n, w, _p(a), w, 1, _p(b), w, 1, _p(out), workers)
        return out

    def partition(self, n, k, weights=None, by_nnz=False, rowlens=None):
        w = np.ones(k) if weights is None else np.ascontiguousarray(weights, np.float64)
        rl = None if rowlens is None else np.ascontiguousarray(rowlens, np.int32)
        out = np.zeros(k + 1, np.int64)
        rc = self.lib.or_partition(n, _p(rl), _p(w), k, 1 if by_nnz else 0, _p(out))
        if rc != 0:
            raise ValueError(rc)
        return out


class OracleSell:
    def __init__(self, orc: Oracle, h):
        self.orc, self.h = orc, h
        self.s = h.contents

    def layout(self) -> SellLayout:
        s = self.s
        vdt = np.complex128 if s.dt == 1 else np.float64
        return SellLayout(
            row_perm_inv=_arr(s.row_perm_inv, s.nrows, np.int32), row_perm=_arr(s.row_perm, s.nrows, np.int32),
            rowlen=_arr(s.rowlen, s.nrows_padded, np.int32), chunk_len=_arr(s.chunk_len, s.nchunks, np.int32),
            chunk_offset=_arr(s.chunk_offset, s.nchunks + 1, np.int64), val=_arr(s.val, s.slots, vdt),
            col=_arr(s.col, s.slots, np.int32), beta=s.beta, nrows_padded=s.nrows_padded, nchunks=s.nchunks,
            slots=s.slots, C=s.C, sigma=s.sigma, cols_permuted=s.cols_permuted)

    def __del__(self):
        try:
            if self.h:
                self.orc.lib.or_sell_free(self.h)
                self.h = None
        except Exception:
            pass


# ------------------------------------------------------------ generators --

def stencil_crs(points: int, n: int, row_begin: int = 0, row_end: Optional[int] = None):
    """2-D 5-point / 3-D 7-point Laplacian rows [row_begin, row_end), global columns
    (same matrix as sellkit_ext_crs_stencil)."""
    N = n * n if points == 5 else n ** 3
    row_end = N if row_end is None else row_end
    r = np.arange(row_begin, row_end, dtype=np.int64)
    if points == 5:
        x, y = r % n, r // n
        offs = [(-n, y > 0), (-1, x > 0), (0, np.ones_like(r, bool)), (1, x + 1 < n), (n, y + 1 < n)]
        diag = 4.0
    else:
        n2 = n * n
        x, y, z = r % n, (r // n) % n, r // n2
        offs = [(-n2, z > 0), (-n, y > 0), (-1, x > 0), (0, np.ones_like(r, bool)), (1, x + 1 < n),
                (n, y + 1 < n), (n2, z + 1 < n)]
        diag = 6.0
    mask = np.stack([m for _, m in offs], axis=1)
    cols = np.stack([r + o for o, _ in offs], axis=1)
    lens = mask.sum(axis=1)
    rowptr = np.zeros(len(r) + 1, np.int64)
    np.cumsum(lens, out=rowptr[1:])
    col = cols[mask]
    val = np.where(col == np.repeat(r, lens), diag, -1.0)
    return rowptr, col.astype(np.int64), val.astype(np.float64)


def stencil_box(nx: int, ny: int, nz: int):
    """3-D 7-point Laplacian on an nx x ny x nz box (row = (z*ny + y)*nx + x), the
    per-row structure of the cube stencil; used for bounded CPU samples."""
    r = np.arange(nx * ny * nz, dtype=np.int64)
    x, y, z = r % nx, (r // nx) % ny, r // (nx * ny)
    pl = nx * ny
    offs = [(-pl, z > 0), (-nx, y > 0), (-1, x > 0), (0, np.ones_like(r, bool)), (1, x + 1 < nx),
            (nx, y + 1 < ny), (pl, z + 1 < nz)]
    mask = np.stack([m for _, m in offs], axis=1)
    cols = np.stack([r + o for o, _ in offs], axis=1)
    lens = mask.sum(axis=1)
    rowptr = np.zeros(len(r) + 1, np.int64)
    np.cumsum(lens, out=rowptr[1:])
    col = cols[mask]
    val = np.where(col == np.repeat(r, lens), 6.0, -1.0)
    return rowptr, col.astype(np.int64), val.astype(np.float64)


def ti_crs(lx: int, ly: int, lz: int, disorder: float = 0.0):
    """Numpy restatement of the synthetic topological-insulator Hamiltonian of
    sellkit_ext_crs_ti: 4 orbitals per periodic site, 13 nonzeros per
    row: on-site 2*G1 + V*I and hoppings (G1 -/+ i*G_{a+2})/2, G1 = tau_z(x)I,
    G2..4 = tau_x(x)sigma_{x,y,z}."""
    nsite = lx * ly * lz
    rows = np.arange(4 * nsite, dtype=np.int64)
    site, o = rows >> 2, rows & 3
    x, y, z = site % lx, (site // lx) % ly, site // (lx * ly)
    g1 = np.where(o < 2, 1.0, -1.0)
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(0x51) ^ site.astype(np.uint64))
    u = (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 - 0.5
    cols = [rows]
    vals = [2.0 * g1 + disorder * u + 0j]
    to, so = o ^ 2, o & 1
    for a in range(3):
        for s in (-1, 1):
            nx, ny, nz = x.copy(), y.copy(), z.copy()
            if a == 0:
                nx = (x + s) % lx
            elif a == 1:
                ny = (y + s) % ly
            else:
                nz = (z + s) % lz
            ns = (nz * ly + ny) * lx + nx
            cols.append(ns * 4 + o)
            vals.append(0.5 * g1 + 0j)
            if a == 0:
                op, mr, mi = to ^ 1, np.ones(len(rows)), np.zeros(len(rows))
            elif a == 1:
                op, mr, mi = to ^ 1, np.zeros(len(rows)), np.where(so == 0, -1.0, 1.0)
            else:
                op, mr, mi = to, np.where(so == 0, 1.0, -1.0), np.zeros(len(rows))
            cols.append(ns * 4 + op)
            vals.append((-s * (-mi) * 0.5) + 1j * (-s * mr * 0.5))
    C_ = np.stack(cols, 1)
    V_ = np.stack(vals, 1)
    order = np.argsort(C_, axis=1, kind="stable")
    C_ = np.take_along_axis(C_, order, 1)
    V_ = np.take_along_axis(V_, order, 1)
    rowptr = np.arange(0, 13 * len(rows) + 1, 13, dtype=np.int64)
    return rowptr, C_.reshape(-1), V_.reshape(-1)


def random_crs(rng: np.random.Generator, nrows: int, ncols: int, density: float, cplx: bool = False):
    """Random CRS with >= 1 entry per row, columns ascending, values U(-1,1)
    (the shape of proj/tests/oracles.hpp:91-119)."""
    mask = rng.random((nrows, ncols)) < density
    empty = ~mask.any(axis=1)
    mask[np.nonzero(empty)[0], rng.integers(0, ncols, empty.sum())] = True
    lens = mask.sum(axis=1)
    rowptr = np.zeros(nrows + 1, np.int64)
    np.cumsum(lens, out=rowptr[1:])
    col = np.nonzero(mask)[1].astype(np.int64)
    val = rng.uniform(-1, 1, len(col))
    if cplx:
        val = val + 1j * rng.uniform(-1, 1, len(col))
    return rowptr, col, val


def splitmix64(z: np.ndarray) -> np.ndarray:
    z = (z + np.uint64(0x9E3779B97F4A7C15)) & np.uint64(0xFFFFFFFFFFFFFFFF)
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & np.uint64(0xFFFFFFFFFFFFFFFF)
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & np.uint64(0xFFFFFFFFFFFFFFFF)
    return z ^ (z >> np.uint64(31))


def hash_block(nrows: int, ncols: int, seed: int) -> np.ndarray:
    """U(-1,1) block from the counter hash of sellkit_ext_densemat_fill_hash."""
    with np.errstate(over="ignore"):
        idx = np.arange(nrows * ncols, dtype=np.uint64)
        h = splitmix64(np.uint64(seed) ^ idx)
    return ((h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 * 2.0 - 1.0).reshape(nrows, ncols)


# ----------------------------------------------------------- distribution --

def split_local_remote(rowptr, col, val, row_offset, rank, C_, sigma, orc: Oracle):
    """partition.hpp:136-220 for one rank; returns a dict of metadata and oracle SELL parts."""
    r0, r1 = int(row_offset[rank]), int(row_offset[rank + 1])
    b, e = rowptr[r0], rowptr[r1]
    rp = rowptr[r0:r1 + 1] - b
    cl = col[b:e]
    vl = val[b:e]
    nloc = r1 - r0
    is_local = (cl >= r0) & (cl < r1)
    halo_cols = np.unique(cl[~is_local])
    owners = np.searchsorted(row_offset, halo_cols, side="right") - 1
    rows_of = np.repeat(np.arange(nloc), np.diff(rp))
    lrp = np.zeros(nloc + 1, np.int64)
    np.cumsum(np.bincount(rows_of[is_local], minlength=nloc), out=lrp[1:])
    rrp = np.zeros(nloc + 1, np.int64)
    np.cumsum(np.bincount(rows_of[~is_local], minlength=nloc), out=rrp[1:])
    lcol = cl[is_local] - r0
    rcol = np.searchsorted(halo_cols, cl[~is_local]).astype(np.int64)
    lens = np.diff(rp).astype(np.int32)
    order = orc.sigma_permutation(lens, sigma)
    local = orc.build(lrp, lcol, vl[is_local], C_, sigma, ncols=nloc, permute_columns=True, imposed_order=order)
    remote = None
    if len(halo_cols):
        remote = orc.build(rrp, rcol, vl[~is_local], C_, sigma, ncols=max(1, len(halo_cols)),
                           permute_columns=False, imposed_order=order)
    recv_owner, recv_count = (np.unique(owners, return_counts=True) if len(owners) else
                              (np.zeros(0, np.int64), np.zeros(0, np.int64)))
    return dict(rank=rank, first_row=r0, nrows=nloc, halo_cols=halo_cols, halo_owner=owners,
                recv_owner=recv_owner, recv_count=recv_count, local=local, remote=remote, lens=lens,
                local_crs=(lrp, lcol, vl[is_local]), remote_crs=(rrp, rcol, vl[~is_local]))


def build_context(rowptr, col, val, k, C_, sigma, orc: Oracle, weights=None, by_nnz=False):
    """partition.hpp:250-286: all ranks' parts plus send lists."""
    n = len(rowptr) - 1
    lens = np.diff(rowptr).astype(np.int32)
    row_offset = orc.partition(n, k, weights, by_nnz, lens)
    ranks = [split_local_remote(rowptr, col, val, row_offset, r, C_, sigma, orc) for r in range(k)]
    for r in range(k):
        ranks[r]["send_to"], ranks[r]["send_rows"] = [], []
    for r in range(k):
        sm = ranks[r]
        for owner in np.unique(sm["halo_owner"]):
            gcols = sm["halo_cols"][sm["halo_owner"] == owner]
            perm = ranks[owner]["local"].layout()["row_perm"]
            ranks[owner]["send_to"].append(r)
            ranks[owner]["send_rows"].append(perm[gcols - row_offset[owner]].astype(np.int32))
    return row_offset, ranks


# ------------------------------------------------------------ full size --

FULLSIZE_PATH = os.path.join(HERE, "libfullsize.so")


class FullSize:
    """ctypes binding of oracle/libfullsize.so (fullsize.c): OpenMP generators and
    checkers for the BASELINE-size parity tests and the reference arm's input."""

    def __init__(self, path: str = FULLSIZE_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -f oracle/Makefile`")
        L = self.lib = C.CDLL(path)
        L.fs_hash_block.argtypes = [i64, i32, C.c_uint64, vp]
        L.fs_stencil7_crs.argtypes = [i64, i64, i64, vp, vp, vp]
        L.fs_tsmm_rows.argtypes = [i64, i64, i32, i32, C.c_uint64, vp, C.c_double, C.c_double, C.c_uint64, vp]
        L.fs_tsmttsm.argtypes = [i64, i32, i32, C.c_uint64, C.c_uint64, vp, vp]
        L.fs_dot_cols.argtypes = [i64, i32, vp, vp, vp, vp]
        L.fs_zdot_cols.argtypes = [i64, i32, vp, vp, vp, vp]

    def hash_block(self, nrows: int, ncols: int, seed: int) -> np.ndarray:
        out = np.empty((nrows, ncols), np.float64)
        self.lib.fs_hash_block(nrows, ncols, seed, _p(out))
        return out

    def stencil7_crs(self, n: int, r0: int = 0, r1: Optional[int] = None):
        r1 = n ** 3 if r1 is None else r1
        rows = r1 - r0
        rowptr = np.empty(rows + 1, np.int64)
        nnz_max = 7 * rows
        col = np.empty(nnz_max, np.int64)
        val = np.empty(nnz_max, np.float64)
        self.lib.fs_stencil7_crs(n, r0, r1, _p(rowptr), _p(col), _p(val))
        nnz = int(rowptr[-1])
        return rowptr, col[:nnz], val[:nnz]

    def tsmm_rows(self, i0: int, i1: int, m: int, k: int, seed_v: int, x: np.ndarray, alpha: float, beta: float,
                  seed_w: int) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty((i1 - i0, k), np.float64)
        self.lib.fs_tsmm_rows(i0, i1, m, k, seed_v, _p(x), alpha, beta, seed_w, _p(out))
        return out

    def tsmttsm(self, n: int, m: int, k: int, seed_v: int, seed_w: int):
        x, sc = np.empty((m, k), np.float64), np.empty((m, k), np.float64)
        self.lib.fs_tsmttsm(n, m, k, seed_v, seed_w, _p(x), _p(sc))
        return x, sc

    def dot_cols(self, a: np.ndarray, b: np.ndarray):
        """long-double column dots of two row-major blocks: (dots, sum |a b|) per column."""
        if np.iscomplexobj(a):
            a, b = np.ascontiguousarray(a, np.complex128), np.ascontiguousarray(b, np.complex128)
            out, sc = np.empty(a.shape[1], np.complex128), np.empty(a.shape[1], np.float64)
            self.lib.fs_zdot_cols(a.shape[0], a.shape[1], _p(a), _p(b), _p(out), _p(sc))
            return out, sc
        a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
        out, sc = np.empty(a.shape[1], np.float64), np.empty(a.shape[1], np.float64)
        self.lib.fs_dot_cols(a.shape[0], a.shape[1], _p(a), _p(b), _p(out), _p(sc))
        return out, sc
