"""Host side of the row-distributed SpMMV (reference: proj/src/partition.hpp).

Two entry points over the C ABI:

* :class:`DistContext` -- the reference's single-process API
  (``sellkit_ctx_create`` / ``sellkit_dvec_*`` / ``sellkit_dist_spmv``): all
  ranks driven from one process, ranks mapped round-robin onto the visible GPUs.
* :func:`setup_rank` -- one process per GPU (torchrun).  The C library builds
  this rank's local/remote SELL parts and moves the halo with NCCL; the only
  host-side protocol is the exchange of halo requests (each rank tells every
  owner which of its rows it needs), done here over ``torch.distributed``
  (gloo or NCCL object collectives) -- :func:`exchange_requests` is also what
  the CPU (gloo) tests exercise through the host-only ``sellkit_ext_rankplan``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional

import numpy as np

from . import sellkit
from .sellkit import R64, Sellkit, _ptr, vp


def partition(sk: Sellkit, n: int, nranks: int, weights=None, by_nnz: bool = False, rowlens=None) -> np.ndarray:
    """sellkit_partition_compute (partition.hpp:45-94)."""
    w = np.ones(nranks) if weights is None else np.ascontiguousarray(weights, np.float64)
    rl = None if rowlens is None else np.ascontiguousarray(rowlens, np.int32)
    out = np.zeros(nranks + 1, np.int64)
    sk.call("sellkit_partition_compute", n, _ptr(rl), _ptr(w), nranks, 1 if by_nnz else 0, _ptr(out))
    return out


# ------------------------------------------------------- single process

class DistContext:
    """sellkit_ctx: all ranks in this process (reference C ABI, sellkit.h:219-249)."""

    def __init__(self, sk: Sellkit, crs, nranks: int, chunk_height: int, sigma: int, weights=None,
                 by_nnz: bool = False, record: bool = True):
        self.sk, self.nranks, self.dt = sk, nranks, crs.dt
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        h = vp()
        sk.call("sellkit_ctx_create", crs.h, _ptr(w), nranks, 1 if by_nnz else 0, chunk_height, sigma,
                1 if record else 0, C.byref(h))
        self.h = h

    def rank_range(self, r):
        f, c = sellkit.gidx(), sellkit.gidx()
        self.sk.call("sellkit_ctx_rank_range", self.h, r, C.byref(f), C.byref(c))
        return f.value, c.value

    def halo_size(self, r):
        n = sellkit.lidx()
        self.sk.call("sellkit_ctx_halo_size", self.h, r, C.byref(n))
        return n.value

    def comm_stats(self):
        b, m = C.c_uint64(), C.c_uint64()
        self.sk.call("sellkit_ctx_comm_stats", self.h, C.byref(b), C.byref(m))
        return b.value, m.value

    def reset_comm_stats(self):
        self.sk.call("sellkit_ctx_reset_comm_stats", self.h)

    def vec(self, width: int, order=sellkit.ROW_MAJOR) -> "DistVec":
        h = vp()
        self.sk.call("sellkit_dvec_create", self.h, width, order, C.byref(h))
        return DistVec(self, h, width)

    def scatter(self, global_mat, v: "DistVec"):
        self.sk.call("sellkit_dvec_scatter", self.h, global_mat.h, v.h)

    def gather(self, v: "DistVec", out):
        self.sk.call("sellkit_dvec_gather", self.h, v.h, out.h)

    def spmv(self, y: "DistVec", x: "DistVec", flags=0, alpha=None, beta=None, gamma=None, delta=None, eta=None,
             z: Optional["DistVec"] = None, dot: Optional[np.ndarray] = None, mode=sellkit.NO_OVERLAP,
             nocomm: bool = False):
        o = sellkit.spmv_opts()
        keep = []

        def sc(v):
            if v is None:
                return None
            a = np.ascontiguousarray(np.atleast_1d(v), dtype=sellkit.NP_DTYPE[self.dt])
            keep.append(a)
            return _ptr(a)
        o.flags = flags
        o.alpha, o.beta, o.gamma, o.delta, o.eta = sc(alpha), sc(beta), sc(gamma), sc(delta), sc(eta)
        o.dot = _ptr(dot)
        if nocomm:
            self.sk.call("sellkit_spmv_nocomm", y.h, self.h, x.h, C.byref(o), z.h if z is not None else None)
        else:
            self.sk.call("sellkit_dist_spmv", y.h, self.h, x.h, C.byref(o), mode, z.h if z is not None else None, 4)

    def close(self):
        if self.h:
            self.sk.lib.sellkit_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistVec:
    def __init__(self, ctx: DistContext, h, width):
        self.ctx, self.h, self.width = ctx, h, width

    def close(self):
        if self.h:
            self.ctx.sk.lib.sellkit_dvec_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------- one process per GPU

def exchange_requests(my_requests: Dict[int, np.ndarray], rank: int, world: int, group=None) -> Dict[int, np.ndarray]:
    """All-to-all of halo requests: returns {requester: global columns it needs from `rank`}."""
    import torch.distributed as tdist
    gathered: List[Optional[Dict[int, np.ndarray]]] = [None] * world
    tdist.all_gather_object(gathered, {int(k): np.asarray(v, np.int64) for k, v in my_requests.items()}, group=group)
    return {r: gathered[r][rank] for r in range(world) if r != rank and rank in gathered[r]}


def _requests(sk: Sellkit, h, prefix: str) -> Dict[int, np.ndarray]:
    n = C.c_int()
    sk.call(f"sellkit_ext_{prefix}_recv_count", h, C.byref(n))
    out = {}
    for q in range(n.value):
        owner, cnt = C.c_int(), sellkit.lidx()
        sk.call(f"sellkit_ext_{prefix}_recv", h, q, C.byref(owner), C.byref(cnt), None)
        cols = np.zeros(cnt.value, np.int64)
        sk.call(f"sellkit_ext_{prefix}_recv", h, q, None, None, _ptr(cols))
        out[owner.value] = cols
    return out


class RankPlan:
    """Host-only plan of one rank (sellkit_ext_rankplan_*; no GPU needed)."""

    def __init__(self, sk: Sellkit, rowptr, col, val, row_offsets, rank: int, dt=R64):
        self.sk = sk
        self._keep = [np.ascontiguousarray(rowptr, np.int64), np.ascontiguousarray(col, np.int64),
                      np.ascontiguousarray(val, sellkit.NP_DTYPE[dt]), np.ascontiguousarray(row_offsets, np.int64)]
        rp, cl, vl, off = self._keep
        h = vp()
        sk.call("sellkit_ext_rankplan_create", dt, _ptr(rp), _ptr(cl), _ptr(vl), len(rp) - 1, _ptr(off),
                len(off) - 1, rank, C.byref(h))
        self.h = h

    def requests(self) -> Dict[int, np.ndarray]:
        return _requests(self.sk, self.h, "rankplan")

    def set_sends(self, to: int, cols: np.ndarray):
        cols = np.ascontiguousarray(cols, np.int64)
        self.sk.call("sellkit_ext_rankplan_set_sends", self.h, to, _ptr(cols), len(cols))

    def sends(self) -> Dict[int, np.ndarray]:
        n = C.c_int()
        self.sk.call("sellkit_ext_rankplan_nsends", self.h, C.byref(n))
        out = {}
        for s in range(n.value):
            to, cnt = C.c_int(), sellkit.lidx()
            self.sk.call("sellkit_ext_rankplan_send", self.h, s, C.byref(to), C.byref(cnt), None)
            rows = np.zeros(cnt.value, np.int32)
            self.sk.call("sellkit_ext_rankplan_send", self.h, s, None, None, _ptr(rows))
            out[to.value] = rows
        return out

    def __del__(self):
        try:
            if self.h:
                self.sk.lib.sellkit_ext_rankplan_destroy(self.h)
                self.h = None
        except Exception:
            pass


class RankContext:
    """sellkit_ext_rankctx: this process's rank of a distributed matrix."""

    def __init__(self, sk: Sellkit, rows_crs, row_offsets, rank: int, chunk_height: int, sigma: int):
        self.sk = sk
        self.row_offsets = np.ascontiguousarray(row_offsets, np.int64)
        self.rank, self.world = rank, len(self.row_offsets) - 1
        self.dt = rows_crs.dt
        self.nrows = int(self.row_offsets[rank + 1] - self.row_offsets[rank])
        h = vp()
        sk.call("sellkit_ext_rankctx_create", rows_crs.h, _ptr(self.row_offsets), self.world, rank, chunk_height,
                sigma, C.byref(h))
        self.h = h

    def requests(self) -> Dict[int, np.ndarray]:
        return _requests(self.sk, self.h, "rankctx")

    def set_sends(self, to: int, cols: np.ndarray):
        cols = np.ascontiguousarray(cols, np.int64)
        self.sk.call("sellkit_ext_rankctx_set_sends", self.h, to, _ptr(cols), len(cols))

    def connect(self, nccl_id: bytes):
        buf = (C.c_char * 128).from_buffer_copy(nccl_id)
        self.sk.call("sellkit_ext_rankctx_connect", self.h, C.cast(buf, vp))

    def ipc_export(self, max_width: int) -> bytes:
        """Export this rank's IPC send slots / dot slot / flags (sellkit_ext_rankctx_ipc_export)."""
        n = C.c_size_t(0)
        self.sk.call("sellkit_ext_rankctx_ipc_export", self.h, max_width, None, C.byref(n))
        buf = (C.c_char * n.value)()
        self.sk.call("sellkit_ext_rankctx_ipc_export", self.h, max_width, C.cast(buf, vp), C.byref(n))
        return bytes(buf.raw)

    def ipc_connect(self, blobs: List[bytes]):
        """Open every rank's exported buffers (blobs in rank order)."""
        size = len(blobs[0])
        assert all(len(b) == size for b in blobs) and len(blobs) == self.world
        raw = (C.c_char * (size * len(blobs))).from_buffer_copy(b"".join(blobs))
        self.sk.call("sellkit_ext_rankctx_ipc_connect", self.h, C.cast(raw, vp), size)

    @property
    def transport(self) -> str:
        t = C.c_int()
        self.sk.call("sellkit_ext_rankctx_transport", self.h, C.byref(t))
        return {0: "none", 1: "nccl", 2: "ipc"}[t.value]

    def set_options(self, graphs: int = -1, reserve_sms: int = -1):
        self.sk.call("sellkit_ext_rankctx_set_options", self.h, graphs, reserve_sms)

    def row_perm(self) -> np.ndarray:
        out = np.zeros(self.nrows, np.int32)
        self.sk.call("sellkit_ext_rankctx_row_perm", self.h, _ptr(out))
        return out

    def stats(self):
        b, m, nh, br, ln, rn = (C.c_uint64(), C.c_uint64(), sellkit.lidx(), C.c_uint64(), sellkit.gidx(),
                                sellkit.gidx())
        self.sk.call("sellkit_ext_rankctx_stats", self.h, C.byref(b), C.byref(m), C.byref(nh), C.byref(br),
                     C.byref(ln), C.byref(rn))
        return dict(bytes=b.value, msgs=m.value, n_halo=nh.value, boundary_rows=br.value, local_nnz=ln.value,
                    remote_nnz=rn.value)

    def spmv(self, y, x, flags=0, alpha=None, beta=None, gamma=None, delta=None, eta=None, z=None,
             dot: Optional[np.ndarray] = None, nocomm: bool = False, opts=None):
        if opts is None:
            opts = sellkit.spmv_opts()
            keep = []

            def sc(v):
                if v is None:
                    return None
                a = np.ascontiguousarray(np.atleast_1d(v), dtype=sellkit.NP_DTYPE[self.dt])
                keep.append(a)
                return _ptr(a)
            opts.flags = flags
            opts.alpha, opts.beta, opts.gamma, opts.delta, opts.eta = sc(alpha), sc(beta), sc(gamma), sc(delta), sc(eta)
            opts.dot = _ptr(dot)
        self.sk.call("sellkit_ext_rank_spmv", y.h, self.h, x.h, C.byref(opts), z.h if z is not None else None,
                     1 if nocomm else 0)

    def close(self, group=None):
        """Collective when connected: every rank must have finished its last step before
        any rank frees the buffers the others map (CUDA IPC) or leaves the NCCL
        communicator, so the ranks synchronise their device and meet at a barrier first."""
        if self.h:
            if self.world > 1 and self.transport != "none":
                import torch
                import torch.distributed as tdist
                torch.cuda.synchronize()
                if tdist.is_available() and tdist.is_initialized():
                    tdist.barrier(group=group if group is not None else getattr(self, "group", None))
            self.sk.lib.sellkit_ext_rankctx_destroy(self.h)
            self.h = None

    def __del__(self):
        # interpreter shutdown: no collective possible any more; just release
        try:
            if self.h:
                self.sk.lib.sellkit_ext_rankctx_destroy(self.h)
                self.h = None
        except Exception:
            pass


def default_transport(world: int) -> str:
    """IPC when every rank runs on this node (torchrun's LOCAL_WORLD_SIZE), else NCCL;
    SELLKIT_HALO_TRANSPORT=ipc|nccl overrides."""
    import os
    t = os.environ.get("SELLKIT_HALO_TRANSPORT", "auto")
    if t != "auto":
        return t
    local = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    return "ipc" if local == world else "nccl"


def setup_rank(sk: Sellkit, rows_crs, row_offsets, rank: int, world: int, chunk_height: int, sigma: int,
               group=None, transport: Optional[str] = None, max_width: int = 64) -> RankContext:
    """Build this rank's parts, exchange halo requests, connect the halo transport.

    transport: "ipc" (CUDA-IPC slots + copy-engine pulls, one node) or "nccl"
    (send/recv over NCCL); default :func:`default_transport`.  Only the setup
    handshake (requests, IPC blobs / NCCL id) goes through ``torch.distributed``."""
    import torch.distributed as tdist
    rc = RankContext(sk, rows_crs, row_offsets, rank, chunk_height, sigma)
    rc.group = group
    if world > 1:
        incoming = exchange_requests(rc.requests(), rank, world, group)
        for to in sorted(incoming):
            rc.set_sends(to, incoming[to])
        transport = transport or default_transport(world)
        if transport == "ipc":
            blobs: List[Optional[bytes]] = [None] * world
            tdist.all_gather_object(blobs, rc.ipc_export(max_width), group=group)
            rc.ipc_connect(blobs)
        elif transport == "nccl":
            idbuf = bytearray(128)
            if rank == 0:
                raw = (C.c_char * 128)()
                sk.call("sellkit_ext_nccl_unique_id", C.cast(raw, vp))
                idbuf = bytearray(raw.raw)
            obj = [bytes(idbuf)]
            tdist.broadcast_object_list(obj, src=0, group=group)
            rc.connect(obj[0])
        else:
            raise ValueError(f"unknown halo transport {transport!r}")
        tdist.barrier(group=group)  # every rank connected before the first step
    else:
        rc.connect(bytes(128))
    return rc


# ------------------------------------------------------------------ bench

@dataclass
class BenchJob:
    step: Callable[[], None]
    e2e_step: Callable[[], None]
    rows_local: int
    nnz_local: int
    halo_bytes: int
    launches_per_step: int
    h2d_bytes: int
    d2h_bytes: int
    keep: list = field(default_factory=list)
    e2e_flush: Optional[Callable[[], None]] = None

    def kernel_ms(self, per_step: List[float]) -> float:
        return float(np.mean(per_step))

    def close(self):
        """Collective: release the rank context after every rank finished (see RankContext.close)."""
        for obj in self.keep:
            if isinstance(obj, RankContext):
                obj.close()


def bench_setup(sk: Sellkit, n: int, w: int, chunk_height: int, sigma: int, rank: int, world: int,
                transport: Optional[str] = None) -> BenchJob:
    """This rank's z-slab of the n^3 7-point stencil (BY_ROWS, equal weights), x hashed on the device."""
    import torch
    N = n ** 3
    off = partition(sk, N, world)
    r0, r1 = int(off[rank]), int(off[rank + 1])
    rows = sk.crs_stencil(7, n, r0, r1)
    _, _, nnz_local = rows.dims()
    rc = setup_rank(sk, rows, off, rank, world, chunk_height, sigma, transport=transport, max_width=w)
    del rows
    nloc = r1 - r0
    # rank vectors in HBM (torch allocations viewed by the library: the e2e copies below
    # run on torch copy streams)
    xt = torch.empty((nloc, w), dtype=torch.float64, device="cuda")
    yt = torch.empty((nloc, w), dtype=torch.float64, device="cuda")
    x = sk.view_plain(xt.data_ptr(), nloc * w, nloc, w, w, keep=xt)
    y = sk.view_plain(yt.data_ptr(), nloc * w, nloc, w, w, keep=yt)
    x.fill_hash(42 + rank)
    st = rc.stats()
    opts = sellkit.spmv_opts()
    sk.lib.sellkit_spmv_opts_init(C.byref(opts))

    def step():
        sk.call("sellkit_ext_rank_spmv", y.h, rc.h, x.h, C.byref(opts), None, 0)

    xh = torch.empty((nloc, w), dtype=torch.float64, pin_memory=True)
    yh = torch.empty((nloc, w), dtype=torch.float64, pin_memory=True)
    xh.copy_(xt)

    # e2e step: H2D of x (copy stream), the distributed sweep (library stream), D2H of y
    # (second copy stream).  Consecutive steps pipeline: step i+1's x upload overlaps
    # step i's y download (the two directions of the link); the sweep waits for its x and
    # for the previous download to release y.
    lib = torch.cuda.ExternalStream(sk.stream())
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev_x, ev_sweep, ev_y = torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()

    def e2e_step():
        s_in.wait_event(ev_sweep)           # previous sweep finished reading x
        with torch.cuda.stream(s_in):
            xt.copy_(xh, non_blocking=True)
            ev_x.record(s_in)
        lib.wait_event(ev_x)
        lib.wait_event(ev_y)                # previous download finished reading y
        sk.set_sync(False)
        step()
        ev_sweep.record(lib)
        s_out.wait_event(ev_sweep)
        with torch.cuda.stream(s_out):
            yh.copy_(yt, non_blocking=True)
            ev_y.record(s_out)

    def e2e_flush():
        lib.wait_event(ev_y)                # the timed region ends after the last download

    # our kernels per step: pack (one per send list) + local sweep + remote sweep; the stencil
    # coupling is symmetric, so we send to exactly the owners we receive from
    nsend = len(rc.requests())
    launches = 1 + (1 + nsend if world > 1 and st["boundary_rows"] > 0 else 0)
    halo_bytes = st["n_halo"] * w * 8
    return BenchJob(step=step, e2e_step=e2e_step, rows_local=nloc, nnz_local=nnz_local, halo_bytes=halo_bytes,
                    launches_per_step=launches, h2d_bytes=nloc * w * 8, d2h_bytes=nloc * w * 8,
                    keep=[rc, x, y, xt, yt, xh, yh, opts, s_in, s_out], e2e_flush=e2e_flush)


# ------------------------------------------------------- tall-skinny, sharded
# TSMM is row-sharded with no communication (X replicated); TSMTTSM
# is row-sharded with one exchange of the m x k partials.  The reference has no
# distributed TSMTTSM; here every rank gathers all partials and sums them in rank
# order with the library's axpby, so every rank holds the identical (deterministic)
# result, as the reference's rank-ordered allreduce of dots does (partition.hpp:379-394).

def gather_in_rank_order(t, group=None) -> list:
    """[t_0, ..., t_{k-1}] from every rank (all_gather; works for gloo CPU and NCCL GPU tensors)."""
    import torch
    import torch.distributed as tdist
    if not (tdist.is_available() and tdist.is_initialized()) or tdist.get_world_size(group) == 1:
        return [t]
    parts = [torch.empty_like(t) for _ in range(tdist.get_world_size(group))]
    tdist.all_gather(parts, t.contiguous(), group=group)
    return parts


def tsmm(sk: Sellkit, w, v, x, alpha=1.0, beta=0.0):
    """W_r = alpha V_r X + beta W_r on this rank's rows (X replicated): no communication."""
    dt = w.dt
    a = np.atleast_1d(np.asarray(alpha, sellkit.NP_DTYPE[dt]))
    b = np.atleast_1d(np.asarray(beta, sellkit.NP_DTYPE[dt]))
    sk.call("sellkit_tsmm", w, v, x, _ptr(a), _ptr(b))


def tsmttsm(sk: Sellkit, x, v, w, alpha=1.0, beta=0.0, kahan: bool = False, group=None):
    """X = alpha * sum_r V_r^H W_r + beta X over row-sharded V, W (one shard per rank)."""
    import torch
    dt = x.dt
    npdt = sellkit.NP_DTYPE[dt]
    tdt = {sellkit.R32: torch.float32, sellkit.R64: torch.float64, sellkit.C32: torch.complex64,
           sellkit.C64: torch.complex128}[dt]
    m, k = x.dims()
    one, zero = np.ones(1, npdt), np.zeros(1, npdt)
    part = torch.zeros((m, k), dtype=tdt, device="cuda")
    pv = sk.view_plain(part.data_ptr(), m * k, m, k, k, dt=dt, keep=part)
    sk.call("sellkit_tsmttsm", pv, v, w, _ptr(one), _ptr(zero), 1 if kahan else 0)  # V_r^H W_r
    parts = gather_in_rank_order(part, group)
    acc = parts[0].clone()
    av = sk.view_plain(acc.data_ptr(), m * k, m, k, k, dt=dt, keep=acc)
    for p in parts[1:]:
        sk.call("sellkit_axpby", av, sk.view_plain(p.data_ptr(), m * k, m, k, k, dt=dt, keep=p), _ptr(one),
                _ptr(one))
    a = np.atleast_1d(np.asarray(alpha, npdt))
    b = np.atleast_1d(np.asarray(beta, npdt))
    sk.call("sellkit_axpby", x, av, _ptr(a), _ptr(b))  # X = alpha * sum + beta * X
