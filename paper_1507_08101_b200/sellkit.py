"""ctypes mirror of the sellkit C ABI (include/sellkit.h + include/sellkit_ext.h).

The same binding drives any library that exports the reference's interface
(/root/reference/proj/include/sellkit.h): the B200 library
``paper_1507_08101_b200/lib/libsellkit_b200.so`` (the product) and, in tests and
the bench's reference arm only, the reference's own CPU build.  Function names,
argument meaning and error behaviour are the reference's; errors surface as
:class:`SellkitError` carrying the ``sellkit_error`` code.

There is no CPU fallback: :func:`load` raises if the CUDA library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

# --------------------------------------------------------------- constants --
OK, ERR_INVALID_ARG, ERR_OVERFLOW, ERR_SHAPE, ERR_PATTERN, ERR_IO = 0, 1, 2, 3, 4, 5
ERR_CAPACITY, ERR_STATE, ERR_ALLOC, ERR_TRANSPORT, ERR_UNSUPPORTED, ERR_NUMERIC = 6, 7, 8, 9, 10, 11

R32, R64, C32, C64 = 0, 1, 2, 3
ROW_MAJOR, COL_MAJOR = 0, 1
BY_ROWS, BY_NNZ = 0, 1
NO_OVERLAP, NAIVE_OVERLAP, TASK_OVERLAP = 0, 1, 2
TRANS_NONE, TRANS_T, TRANS_C = 0, 1, 2

AXPBY, SHIFT, VSHIFT, DOT_YY, DOT_XY, DOT_XX, CHAIN_AXPBY = 0x01, 0x02, 0x04, 0x08, 0x10, 0x20, 0x40

NP_DTYPE = {R32: np.float32, R64: np.float64, C32: np.complex64, C64: np.complex128}
DT_OF = {np.dtype(np.float32): R32, np.dtype(np.float64): R64,
         np.dtype(np.complex64): C32, np.dtype(np.complex128): C64}

gidx = C.c_int64
lidx = C.c_int32
err_t = C.c_int
vp = C.c_void_p
ROW_FN = C.CFUNCTYPE(C.c_int, gidx, C.POINTER(lidx), C.POINTER(gidx), vp, vp)


class SellkitError(RuntimeError):
    def __init__(self, code: int, where: str, name: str = "", detail: str = ""):
        super().__init__(f"{where} failed: sellkit_error {code} ({name})" + (f": {detail}" if detail else ""))
        self.code = code
        self.detail = detail


class spmv_opts(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("alpha", vp), ("beta", vp), ("gamma", vp),
                ("delta", vp), ("eta", vp), ("z", vp), ("dot", vp)]


# (name, restype, argtypes) of every entry point of include/sellkit.h
_API = [
    ("sellkit_error_name", C.c_char_p, [err_t]),
    ("sellkit_narrow_index", err_t, [gidx, C.POINTER(lidx)]),
    ("sellkit_buildconfig_chunk_heights", err_t, [C.POINTER(C.POINTER(C.c_int)), C.POINTER(C.c_size_t)]),
    ("sellkit_buildconfig_block_widths", err_t, [C.POINTER(C.POINTER(C.c_int)), C.POINTER(C.c_size_t)]),
    ("sellkit_set_num_workers", err_t, [C.c_int]),
    ("sellkit_num_workers", C.c_int, []),
    ("sellkit_now_seconds", C.c_double, []),
    ("sellkit_set_timer_override", None, [vp, vp]),
    ("sellkit_crs_create", err_t, [C.c_int, gidx, gidx, vp, vp, vp, C.POINTER(vp)]),
    ("sellkit_crs_from_rowfunc", err_t, [C.c_int, gidx, gidx, lidx, ROW_FN, vp, C.POINTER(vp)]),
    ("sellkit_crs_read_mm", err_t, [C.c_char_p, C.c_int, C.POINTER(vp)]),
    ("sellkit_crs_read_bin", err_t, [C.c_char_p, C.POINTER(vp)]),
    ("sellkit_crs_write_bin", err_t, [C.c_char_p, vp, C.c_int]),
    ("sellkit_crs_dims", err_t, [vp, C.POINTER(gidx), C.POINTER(gidx), C.POINTER(gidx)]),
    ("sellkit_crs_datatype", C.c_int, [vp]),
    ("sellkit_crs_destroy", None, [vp]),
    ("sellkit_mat_build", err_t, [vp, C.c_int, C.c_int, C.POINTER(vp)]),
    ("sellkit_mat_build_rowfunc", err_t, [C.c_int, gidx, gidx, lidx, ROW_FN, vp, C.c_int, C.c_int, C.POINTER(vp)]),
    ("sellkit_mat_stats", err_t, [vp, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]),
    ("sellkit_mat_update_values", err_t, [vp, vp]),
    ("sellkit_mat_to_crs", err_t, [vp, C.POINTER(vp)]),
    ("sellkit_mat_dims", err_t, [vp, C.POINTER(lidx), C.POINTER(lidx), C.POINTER(gidx)]),
    ("sellkit_mat_destroy", None, [vp]),
    ("sellkit_densemat_create", err_t, [C.c_int, lidx, lidx, C.c_int, C.POINTER(vp)]),
    ("sellkit_densemat_view_plain", err_t, [C.c_int, vp, C.c_size_t, lidx, lidx, lidx, C.c_int, C.POINTER(vp)]),
    ("sellkit_densemat_view", err_t, [vp, lidx, lidx, C.POINTER(lidx), lidx, C.POINTER(vp)]),
    ("sellkit_densemat_compact_clone", err_t, [vp, C.POINTER(vp)]),
    ("sellkit_densemat_convert_order", err_t, [vp, C.c_int, C.c_int, C.POINTER(vp)]),
    ("sellkit_densemat_is_scattered", C.c_int, [vp]),
    ("sellkit_densemat_dims", err_t, [vp, C.POINTER(lidx), C.POINTER(lidx)]),
    ("sellkit_densemat_copy_in", err_t, [vp, vp, C.c_size_t]),
    ("sellkit_densemat_copy_out", err_t, [vp, vp, C.c_size_t]),
    ("sellkit_densemat_destroy", None, [vp]),
    ("sellkit_axpby", err_t, [vp, vp, vp, vp]),
    ("sellkit_vaxpby", err_t, [vp, vp, vp, vp]),
    ("sellkit_scal", err_t, [vp, vp]),
    ("sellkit_vscal", err_t, [vp, vp]),
    ("sellkit_dot", err_t, [vp, vp, vp]),
    ("sellkit_tsmttsm", err_t, [vp, vp, vp, vp, vp, C.c_int]),
    ("sellkit_tsmm", err_t, [vp, vp, vp, vp, vp]),
    ("sellkit_tsmm_inplace", err_t, [vp, vp, vp, vp]),
    ("sellkit_gemm", err_t, [vp, vp, vp, vp, vp, C.c_int, C.c_int]),
    ("sellkit_spmv_opts_init", None, [C.POINTER(spmv_opts)]),
    ("sellkit_spmv", err_t, [vp, vp, vp, C.POINTER(spmv_opts)]),
    ("sellkit_select_kernel", err_t, [C.c_int, lidx, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.POINTER(C.c_int)]),
    ("sellkit_partition_compute", err_t, [gidx, vp, vp, C.c_int, C.c_int, vp]),
    ("sellkit_ctx_create", err_t, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    ("sellkit_ctx_rank_range", err_t, [vp, C.c_int, C.POINTER(gidx), C.POINTER(gidx)]),
    ("sellkit_ctx_halo_size", err_t, [vp, C.c_int, C.POINTER(lidx)]),
    ("sellkit_ctx_comm_stats", err_t, [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("sellkit_ctx_reset_comm_stats", err_t, [vp]),
    ("sellkit_ctx_destroy", None, [vp]),
    ("sellkit_dvec_create", err_t, [vp, lidx, C.c_int, C.POINTER(vp)]),
    ("sellkit_dvec_scatter", err_t, [vp, vp, vp]),
    ("sellkit_dvec_gather", err_t, [vp, vp, vp]),
    ("sellkit_dvec_destroy", None, [vp]),
    ("sellkit_dist_spmv", err_t, [vp, vp, vp, C.POINTER(spmv_opts), C.c_int, vp, C.c_int]),
    ("sellkit_spmv_nocomm", err_t, [vp, vp, vp, C.POINTER(spmv_opts), vp]),
    ("sellkit_pool_create", err_t, [C.c_int, vp, C.c_int, C.POINTER(vp)]),
    ("sellkit_task_create", err_t, [vp, vp, vp, C.c_int, C.c_int, C.c_uint32, C.POINTER(vp)]),
    ("sellkit_task_add_dependency", err_t, [vp, vp]),
    ("sellkit_task_enqueue", err_t, [vp, vp]),
    ("sellkit_task_spawn_child", err_t, [vp, vp]),
    ("sellkit_task_wait", err_t, [vp, vp, C.POINTER(vp)]),
    ("sellkit_pool_current_task", err_t, [vp, C.POINTER(vp)]),
    ("sellkit_task_state_of", err_t, [vp, C.POINTER(C.c_int)]),
    ("sellkit_task_destroy", err_t, [vp, vp]),
    ("sellkit_pool_shutdown", err_t, [vp]),
    ("sellkit_pool_npus", C.c_int, [vp]),
    ("sellkit_pool_num_numa_nodes", C.c_int, [vp]),
    ("sellkit_pool_numa_node_of", err_t, [vp, C.c_int, C.POINTER(C.c_int)]),
    ("sellkit_pool_trace", err_t, [vp, C.POINTER(vp)]),
    ("sellkit_pool_destroy", None, [vp]),
    ("sellkit_string_free", None, [vp]),
    ("sellkit_spmv_code_balance", err_t, [C.c_int, C.c_int, C.c_int, C.c_double, C.POINTER(C.c_double)]),
    ("sellkit_index_width_saving", err_t, [C.c_int, C.POINTER(C.c_double)]),
    ("sellkit_roofline_bound", err_t, [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]),
    ("sellkit_crs_refresh_cost", err_t, [gidx, C.c_int, C.c_double, C.POINTER(C.c_double)]),
    ("sellkit_region_create", err_t, [C.c_char_p, C.POINTER(vp)]),
    ("sellkit_region_record", err_t, [vp, C.c_double]),
    ("sellkit_region_p_max", err_t, [vp, C.POINTER(C.c_double)]),
    ("sellkit_region_p_skip10", err_t, [vp, C.POINTER(C.c_double)]),
    ("sellkit_region_table", err_t, [vp, C.c_int, C.POINTER(vp)]),
    ("sellkit_region_destroy", None, [vp]),
]

# include/sellkit_ext.h (B200 library only)
_EXT = [
    ("sellkit_ext_last_error", C.c_char_p, []),
    ("sellkit_ext_set_sync", err_t, [C.c_int]),
    ("sellkit_ext_synchronize", err_t, []),
    ("sellkit_ext_release_cached", err_t, []),
    ("sellkit_ext_stream", err_t, [C.POINTER(vp)]),
    ("sellkit_ext_device_info", err_t, [C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_size_t)]),
    ("sellkit_ext_crs_create_device", err_t, [C.c_int, gidx, gidx, vp, vp, vp, C.POINTER(vp)]),
    ("sellkit_ext_crs_stencil", err_t, [C.c_int, C.c_int, gidx, gidx, gidx, C.POINTER(vp)]),
    ("sellkit_ext_crs_ti", err_t, [C.c_int, gidx, gidx, gidx, C.c_double, gidx, gidx, C.POINTER(vp)]),
    ("sellkit_ext_mat_info", err_t, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(lidx), C.POINTER(gidx),
                                     C.POINTER(gidx), C.POINTER(C.c_int)]),
    ("sellkit_ext_mat_export", err_t, [vp, vp, vp, vp, vp, vp, vp, vp]),
    ("sellkit_ext_mat_set_sweep_order", err_t, [vp, lidx, vp, gidx]),
    ("sellkit_ext_mat_set_apply_override", err_t, [vp, vp, vp]),
    ("sellkit_ext_densemat_storage", err_t, [vp, C.POINTER(vp), C.POINTER(lidx), C.POINTER(C.c_int),
                                             C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("sellkit_ext_densemat_fill_hash", err_t, [vp, C.c_uint64]),
    ("sellkit_ext_ctx_set_trace", err_t, [vp, C.c_int]),
    ("sellkit_ext_ctx_timeline", err_t, [vp, vp, C.POINTER(C.c_int)]),
    ("sellkit_ext_nccl_unique_id", err_t, [vp]),
    ("sellkit_ext_rankctx_create", err_t, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    ("sellkit_ext_rankctx_recv_count", err_t, [vp, C.POINTER(C.c_int)]),
    ("sellkit_ext_rankctx_recv", err_t, [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(lidx), vp]),
    ("sellkit_ext_rankctx_set_sends", err_t, [vp, C.c_int, vp, lidx]),
    ("sellkit_ext_rankctx_send", err_t, [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(lidx), vp]),
    ("sellkit_ext_rankctx_connect", err_t, [vp, vp]),
    ("sellkit_ext_rankctx_ipc_export", err_t, [vp, C.c_int, vp, C.POINTER(C.c_size_t)]),
    ("sellkit_ext_rankctx_ipc_connect", err_t, [vp, vp, C.c_size_t]),
    ("sellkit_ext_rankctx_transport", err_t, [vp, C.POINTER(C.c_int)]),
    ("sellkit_ext_rankctx_set_options", err_t, [vp, C.c_int, C.c_int]),
    ("sellkit_ext_rank_spmv", err_t, [vp, vp, vp, C.POINTER(spmv_opts), vp, C.c_int]),
    ("sellkit_ext_rankctx_stats", err_t, [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(lidx),
                                          C.POINTER(C.c_uint64), C.POINTER(gidx), C.POINTER(gidx)]),
    ("sellkit_ext_rankctx_row_perm", err_t, [vp, vp]),
    ("sellkit_ext_rankctx_destroy", None, [vp]),
    ("sellkit_ext_rankplan_create", err_t, [C.c_int, vp, vp, vp, lidx, vp, C.c_int, C.c_int, C.POINTER(vp)]),
    ("sellkit_ext_rankplan_recv_count", err_t, [vp, C.POINTER(C.c_int)]),
    ("sellkit_ext_rankplan_recv", err_t, [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(lidx), vp]),
    ("sellkit_ext_rankplan_set_sends", err_t, [vp, C.c_int, vp, lidx]),
    ("sellkit_ext_rankplan_nsends", err_t, [vp, C.POINTER(C.c_int)]),
    ("sellkit_ext_rankplan_send", err_t, [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(lidx), vp]),
    ("sellkit_ext_rankplan_destroy", None, [vp]),
]

API_NAMES = [n for n, _, _ in _API]
EXT_NAMES = [n for n, _, _ in _EXT]

_HERE = os.path.dirname(os.path.abspath(__file__))
DEFAULT_LIB = os.path.join(_HERE, "lib", "libsellkit_b200.so")


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(vp)


class Sellkit:
    """Binding of one library exporting the sellkit C ABI."""

    def __init__(self, path: str, ext: bool = True, strict: bool = True):
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"sellkit library not found at {path}; build it with "
                "`python -m paper_1507_08101_b200.build` (there is no CPU fallback)")
        self.path = path
        self.lib = C.CDLL(path, mode=C.RTLD_LOCAL)
        self.missing = []
        for name, res, args in _API + (_EXT if ext else []):
            try:
                f = getattr(self.lib, name)
            except AttributeError:
                self.missing.append(name)
                continue
            f.restype = res
            f.argtypes = args
        if strict and self.missing:
            raise ImportError(f"{path} lacks {self.missing}")
        self.has_ext = ext and not any(n in self.missing for n in EXT_NAMES)

    # -- plumbing -----------------------------------------------------------
    def check(self, code: int, where: str):
        if code != OK:
            detail = ""
            if self.has_ext:
                detail = (self.lib.sellkit_ext_last_error() or b"").decode(errors="replace")
            raise SellkitError(code, where, self.lib.sellkit_error_name(code).decode(), detail)

    def call(self, name: str, *args):
        """Call `name`; handle objects may be passed directly and stay alive for the call."""
        raw = [a.h if isinstance(a, _Handle) else a for a in args]
        code = getattr(self.lib, name)(*raw)
        self.check(code, name)

    # -- objects ------------------------------------------------------------
    def crs(self, rowptr, col, val, ncols=None, dt=None) -> "Crs":
        rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
        col = np.ascontiguousarray(col, dtype=np.int64)
        if dt is None:
            dt = DT_OF[np.asarray(val).dtype]
        val = np.ascontiguousarray(val, dtype=NP_DTYPE[dt])
        nrows = len(rowptr) - 1
        ncols = nrows if ncols is None else ncols
        out = vp()
        self.call("sellkit_crs_create", dt, nrows, ncols, _ptr(rowptr), _ptr(col), _ptr(val), C.byref(out))
        return Crs(self, out, dt)

    def crs_read_mm(self, path: str, dt=R64) -> "Crs":
        """Matrix Market file -> device CRS (reference io.cpp:206-301)."""
        out = vp()
        self.call("sellkit_crs_read_mm", os.fsencode(path), dt, C.byref(out))
        return Crs(self, out, dt)

    def crs_read_bin(self, path: str) -> "Crs":
        """GCRS binary file -> device CRS; the element type comes from the header (io.cpp:303-333)."""
        out = vp()
        self.call("sellkit_crs_read_bin", os.fsencode(path), C.byref(out))
        return Crs(self, out, self.lib.sellkit_crs_datatype(out))

    def crs_stencil(self, points: int, n: int, row_begin: int = 0, row_end: Optional[int] = None, dt=R64) -> "Crs":
        N = n * n if points == 5 else n ** 3
        out = vp()
        self.call("sellkit_ext_crs_stencil", dt, points, n, row_begin, N if row_end is None else row_end, C.byref(out))
        return Crs(self, out, dt)

    def crs_ti(self, lx: int, ly: int, lz: int, disorder: float = 0.0, row_begin: int = 0,
               row_end: Optional[int] = None, dt=C64) -> "Crs":
        N = 4 * lx * ly * lz
        out = vp()
        self.call("sellkit_ext_crs_ti", dt, lx, ly, lz, disorder, row_begin, N if row_end is None else row_end,
                  C.byref(out))
        return Crs(self, out, dt)

    def densemat(self, nrows: int, ncols: int, dt=R64, order=ROW_MAJOR) -> "DenseMat":
        out = vp()
        self.call("sellkit_densemat_create", dt, nrows, ncols, order, C.byref(out))
        return DenseMat(self, out, dt)

    def densemat_from(self, arr: np.ndarray, order=ROW_MAJOR) -> "DenseMat":
        arr = np.asarray(arr)
        if arr.ndim == 1:
            arr = arr[:, None]
        dt = DT_OF[arr.dtype]
        d = self.densemat(arr.shape[0], arr.shape[1], dt, order)
        d.copy_in(arr)
        return d

    def view_plain(self, buf_ptr: int, nelems: int, nrows: int, ncols: int, stride: int, order=ROW_MAJOR,
                   dt=R64, keep=None) -> "DenseMat":
        out = vp()
        self.call("sellkit_densemat_view_plain", dt, vp(buf_ptr), nelems, nrows, ncols, stride, order, C.byref(out))
        d = DenseMat(self, out, dt)
        d._keep = keep
        return d

    def spmv(self, y, A, x, flags=0, alpha=None, beta=None, gamma=None, delta=None, eta=None, z=None,
             dot: Optional[np.ndarray] = None):
        o = spmv_opts()
        self.lib.sellkit_spmv_opts_init(C.byref(o))
        keep = []

        def scal(v):
            if v is None:
                return None
            a = np.ascontiguousarray(np.atleast_1d(v), dtype=NP_DTYPE[y.dt])
            keep.append(a)
            return _ptr(a)

        o.flags = flags
        o.alpha, o.beta, o.gamma, o.delta, o.eta = scal(alpha), scal(beta), scal(gamma), scal(delta), scal(eta)
        o.z = z.h if z is not None else None
        o.dot = _ptr(dot)
        self.call("sellkit_spmv", y.h, A.h, x.h, C.byref(o))

    def select_kernel(self, C_, W, order=ROW_MAJOR):
        c, w, v = C.c_int(), C.c_int(), C.c_int()
        self.call("sellkit_select_kernel", C_, W, order, C.byref(c), C.byref(w), C.byref(v))
        return c.value, w.value, v.value

    # -- ext ----------------------------------------------------------------
    def set_sync(self, sync: bool):
        self.call("sellkit_ext_set_sync", 1 if sync else 0)

    def synchronize(self):
        self.call("sellkit_ext_synchronize")

    def stream(self) -> int:
        s = vp()
        self.call("sellkit_ext_stream", C.byref(s))
        return s.value or 0


class _Handle:
    _destroy = ""

    def __init__(self, sk: Sellkit, h, dt):
        self.sk, self.h, self.dt = sk, h, dt
        self._keep = None

    def close(self):
        if self.h:
            getattr(self.sk.lib, self._destroy)(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Crs(_Handle):
    _destroy = "sellkit_crs_destroy"

    def dims(self):
        r, c, n = gidx(), gidx(), gidx()
        self.sk.call("sellkit_crs_dims", self.h, C.byref(r), C.byref(c), C.byref(n))
        return r.value, c.value, n.value

    def build(self, chunk_height: int, sigma: int) -> "Mat":
        out = vp()
        self.sk.call("sellkit_mat_build", self.h, chunk_height, sigma, C.byref(out))
        return Mat(self.sk, out, self.dt)

    def write_bin(self, path: str, wide_cols: bool = False):
        self.sk.call("sellkit_crs_write_bin", os.fsencode(path), self.h, 1 if wide_cols else 0)


class Mat(_Handle):
    _destroy = "sellkit_mat_destroy"

    def dims(self):
        r, c, n = lidx(), lidx(), gidx()
        self.sk.call("sellkit_mat_dims", self.h, C.byref(r), C.byref(c), C.byref(n))
        return r.value, c.value, n.value

    def stats(self):
        b, t = C.c_double(), C.c_uint64()
        self.sk.call("sellkit_mat_stats", self.h, C.byref(b), C.byref(t))
        return b.value, t.value

    def info(self):
        ch, sg, nrp, nch, sl, cp = C.c_int(), C.c_int(), lidx(), gidx(), gidx(), C.c_int()
        self.sk.call("sellkit_ext_mat_info", self.h, C.byref(ch), C.byref(sg), C.byref(nrp), C.byref(nch),
                     C.byref(sl), C.byref(cp))
        return dict(C=ch.value, sigma=sg.value, nrows_padded=nrp.value, nchunks=nch.value, slots=sl.value,
                    cols_permuted=cp.value)

    def set_sweep_order(self, block_rows: int, order: Optional[np.ndarray]):
        """Sweep blocks of `block_rows` stored rows in `order` (None: natural order)."""
        if order is None:
            self.sk.call("sellkit_ext_mat_set_sweep_order", self.h, block_rows, None, 0)
            return
        o = np.ascontiguousarray(order, np.int32)
        self.sk.call("sellkit_ext_mat_set_sweep_order", self.h, block_rows, _ptr(o), len(o))

    def export(self) -> dict:
        """SELL arrays (sellkit_ext_mat_export)."""
        info = self.info()
        nrows, _, _ = self.dims()
        out = dict(
            row_perm_inv=np.zeros(nrows, np.int32), row_perm=np.zeros(nrows, np.int32),
            rowlen=np.zeros(info["nrows_padded"], np.int32), chunk_len=np.zeros(info["nchunks"], np.int32),
            chunk_offset=np.zeros(info["nchunks"] + 1, np.int64),
            val=np.zeros(info["slots"], NP_DTYPE[self.dt]), col=np.zeros(info["slots"], np.int32))
        self.sk.call("sellkit_ext_mat_export", self.h, *[_ptr(out[k]) for k in
                     ("row_perm_inv", "row_perm", "rowlen", "chunk_len", "chunk_offset", "val", "col")])
        out.update(info)
        return out


class DenseMat(_Handle):
    _destroy = "sellkit_densemat_destroy"

    def dims(self):
        r, c = lidx(), lidx()
        self.sk.call("sellkit_densemat_dims", self.h, C.byref(r), C.byref(c))
        return r.value, c.value

    def copy_in(self, arr: np.ndarray):
        a = np.ascontiguousarray(arr, dtype=NP_DTYPE[self.dt])
        self.sk.call("sellkit_densemat_copy_in", self.h, _ptr(a), a.size)

    def copy_out(self) -> np.ndarray:
        r, c = self.dims()
        out = np.empty((r, c), dtype=NP_DTYPE[self.dt])
        self.sk.call("sellkit_densemat_copy_out", self.h, _ptr(out), out.size)
        return out

    def fill_hash(self, seed: int):
        self.sk.call("sellkit_ext_densemat_fill_hash", self.h, seed)

    def storage(self):
        d, s, o, dev, on = vp(), lidx(), C.c_int(), C.c_int(), C.c_int()
        self.sk.call("sellkit_ext_densemat_storage", self.h, C.byref(d), C.byref(s), C.byref(o), C.byref(dev),
                     C.byref(on))
        return dict(data=d.value, stride=s.value, order=o.value, device=dev.value, on_device=bool(on.value))


_LIB: Optional[Sellkit] = None


def load(path: Optional[str] = None) -> Sellkit:
    """The B200 library (cached).  Raises if it is missing -- no fallback."""
    global _LIB
    if path is not None:
        return Sellkit(path)
    if _LIB is None:
        _LIB = Sellkit(os.environ.get("SELLKIT_B200_LIB", DEFAULT_LIB))
    return _LIB
