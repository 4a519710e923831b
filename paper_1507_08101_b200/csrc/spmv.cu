// Fused SELL-C-sigma SpMV driver: validation (spmv.hpp:98-125), staging of
// host-resident vectors, kernel dispatch and the ordered dot reduction.
#include "spmv_kernels.cuh"

#include <algorithm>

namespace skb {

using namespace spmv_detail;

namespace {

template <class T>
T scalar_of(const unsigned char* b) {
    T v;
    std::memcpy(&v, b, sizeof(T));
    return v;
}

// Every row segment a specialised kernel touches with one vector access must be
// aligned to the access width: min(32 B, width * element bytes) (widths are powers of 2).
bool aligned_for_vectors(const DenseMat& m) {
    const std::size_t req = std::min<std::size_t>(32, std::size_t(m.ncols) * m.esize());
    if (req & (req - 1)) return false;
    return (reinterpret_cast<std::uintptr_t>(m.data) % req == 0) && ((std::size_t(m.stride) * m.esize()) % req == 0);
}

// largest column index of each block of row groups [rgb[b], rgb[b+1])
__global__ void watermark_kernel(const lidx* col, const gidx* chunk_offset, const gidx* cbeg, int nb, lidx* out) {
    const int b = blockIdx.y;
    if (b >= nb) return;
    const gidx s0 = chunk_offset[cbeg[b]], s1 = chunk_offset[cbeg[b + 1]];
    lidx m = 0;
    for (gidx s = s0 + blockIdx.x * gidx(blockDim.x) + threadIdx.x; s < s1; s += gidx(gridDim.x) * blockDim.x)
        m = max(m, col[s]);
    m = lidx(__reduce_max_sync(0xffffffffu, unsigned(m)));
    if ((threadIdx.x & 31) == 0) atomicMax(&out[b], m);
}

bool pinned_host(const DenseMat& m) {
    if (m.mem != MemKind::host || m.scattered() || m.order != Order::row_major || m.stride != m.ncols) return false;
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, m.data) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeHost;
}

// farthest |column - stored row| over the real entries of each row group (32 stored rows)
__global__ void coupling_kernel(const lidx* col, const gidx* chunk_offset, const lidx* rowlen, lidx C, lidx nrows,
                                gidx ngroups, lidx* out) {
    const gidx g = blockIdx.x * gidx(blockDim.x / 32) + threadIdx.x / 32;
    if (g >= ngroups) return;
    const int lane = threadIdx.x & 31;
    const lidx row = lidx(g * 32 + lane);
    lidx m = 0;
    if (row < nrows) {
        const gidx c = row / C;
        const int i = row - lidx(c * C);
        const gidx off = chunk_offset[c] + i;
        const lidx len = rowlen[row];
        for (lidx j = 0; j < len; ++j) {
            const lidx d = col[off + gidx(j) * C] - row;
            m = max(m, d < 0 ? -d : d);
        }
    }
    m = lidx(__reduce_max_sync(0xffffffffu, unsigned(m)));
    if (lane == 0) out[g] = m;
}

// Coupling distance of a square matrix swept by the row-contiguous kernels: the median
// over row groups of the farthest |column - row| (a lattice's largest stride).
gidx coupling_distance(const SellMat& A) {
    if (A.coupling >= 0) return A.coupling;
    A.coupling = 0;
    if (A.nrows != A.ncols || A.nrows < 64 || A.C > 32 || 32 % A.C != 0) return 0;
    auto& rt = runtime(A.device);
    const gidx ngroups = (gidx(A.nrows) + 31) / 32;
    DeviceBuffer d(std::size_t(ngroups) * sizeof(lidx), A.device);
    coupling_kernel<<<int((ngroups + 7) / 8), 256, 0, rt.stream>>>(A.col.as<lidx>(), A.chunk_offset.as<gidx>(),
                                                                    A.rowlen.as<lidx>(), A.C, A.nrows, ngroups,
                                                                    d.as<lidx>());
    CK(cudaGetLastError());
    std::vector<lidx> h(static_cast<std::size_t>(ngroups));
    CK(cudaMemcpyAsync(h.data(), d.get(), h.size() * sizeof(lidx), cudaMemcpyDeviceToHost, rt.stream));
    CK(cudaStreamSynchronize(rt.stream));
    std::nth_element(h.begin(), h.begin() + h.size() / 2, h.end());
    A.coupling = h[h.size() / 2];
    return A.coupling;
}

}  // namespace

// Automatic locality order of a full sweep (no caller order): a row-ordered sweep
// re-reads x[r + D] from HBM when the coupling distance D times the bytes streamed
// per row (x row, matrix entries, y / z rows) exceeds what L2 keeps -- the z-plane
// reuse of a 3-D lattice (C3: D = 131072 rows, 135 MB at w = 16 complex).  Then the
// rows are swept in slabs walked along D: for each slab offset p, blocks p, p + D,
// p + 2D, ... (a "pencil" through the lattice), so x[r + D] is reused a slab later.
// The slab is sized so that three slabs of streams (planes z-1, z, z+1) fit a quarter
// of L2.  Returns the device order and its block size in row groups, or nullptr.
static const int* auto_sweep_order(const SellMat& A, lidx w, std::uint32_t flags, int& block_rgs, gidx& nblocks) {
    const char* e_off = std::getenv("SELLKIT_AUTO_ORDER");
    if ((e_off && std::string(e_off) == "0") || A.sweep_policy != 0) return nullptr;
    const gidx D = coupling_distance(A);
    if (D <= 0) return nullptr;
    auto& rt = runtime(A.device);
    const double es = double(value_bytes(A.dt));
    const double nnz_row = double(A.nnz) / double(std::max<lidx>(1, A.nrows));
    const double vec = es * w;
    const double row_bytes = vec + nnz_row * (es + 4.0) + vec * (1.0 + ((flags & kFlagAxpby) ? 1.0 : 0.0) +
                                                                 ((flags & kFlagChain) ? 2.0 : 0.0));
    // 64-byte RHS rows (double w = 8) stream more matrix than x per row: there the slab
    // orders measured slower at every slab size (400^3: 2.38 -> 2.56-2.63 ms; 320^3:
    // 1.08 -> 1.21-1.35 ms), so they keep the row order
    if (vec < 128.0) return nullptr;
    const char* e_l2 = std::getenv("SELLKIT_AUTO_ORDER_L2");  // cache size the decision assumes (tests)
    // what the sweep can count on keeping: about half the L2 (measured best over
    // 1/8 ... 1 L2 on C2 w = 16/32, 320^3 / 400^3 w = 16 and C3 C64/R64, profiles r2s)
    const double l2 = 0.476 * (e_l2 ? std::atof(e_l2) : double(rt.l2_bytes));
    if (double(D) * row_bytes <= 0.5 * l2) return nullptr;  // the reuse window already fits L2
    constexpr int kBlockRgs = 8;                              // 256-row blocks
    const gidx brows = 32 * kBlockRgs;
    const gidx Db = std::max<gidx>(1, (D + brows / 2) / brows);  // plane stride in blocks
    const gidx slab_rows = gidx(0.25 * l2 / (3.0 * row_bytes));
    const int Sb = int(std::max<gidx>(1, slab_rows / brows));
    block_rgs = kBlockRgs;
    nblocks = (gidx(A.nrows_padded) + brows - 1) / brows;
    for (auto& o : A.auto_orders)
        if (o.slab_blocks == Sb && o.nblocks == nblocks) return o.order.get() ? o.order.as<int>() : nullptr;
    SellMat::AutoOrder ao;
    ao.slab_blocks = Sb;
    ao.nblocks = nblocks;
    if (Sb < Db) {
        std::vector<int> ord;
        ord.reserve(std::size_t(nblocks));
        const gidx planes = (nblocks + Db - 1) / Db;
        for (gidx p0 = 0; p0 < Db; p0 += Sb)
            for (gidx q = 0; q < planes; ++q)
                for (gidx p = p0; p < std::min<gidx>(p0 + Sb, Db); ++p) {
                    const gidx b = q * Db + p;
                    if (b < nblocks) ord.push_back(int(b));
                }
        ao.order = DeviceBuffer(ord.size() * sizeof(int), A.device);
        CK(cudaMemcpyAsync(ao.order.get(), ord.data(), ord.size() * sizeof(int), cudaMemcpyHostToDevice, rt.stream));
        CK(cudaStreamSynchronize(rt.stream));
        if (std::getenv("SELLKIT_VERBOSE"))
            std::fprintf(stderr, "[sellkit] auto sweep order: coupling %lld rows, %.0f B/row, slabs of %d x 256 rows\n",
                         (long long)D, row_bytes, Sb);
    }
    A.auto_orders.push_back(std::move(ao));
    return A.auto_orders.back().order.get() ? A.auto_orders.back().order.as<int>() : nullptr;
}

// Streamed spmv on pinned host buffers: x arrives in row slabs on one copy engine,
// each block of row groups is swept as soon as the x rows up to its largest column
// index are resident (column watermark), and its y rows leave on the other copy
// engine -- H2D, sweep and D2H overlap instead of running back to back.
// Row blocks of the streamed sweep: the transfer of the first x slab(s) and of
// the last y block are not overlapped, so finer blocks shorten fill and drain
// (per block: one sweep launch + 2-3 copies, ~10 us).  SELLKIT_STREAM_BLOCKS overrides.
static int stream_blocks() {
    static const int nb = [] {
        const char* e = std::getenv("SELLKIT_STREAM_BLOCKS");
        return e ? std::max(2, std::atoi(e)) : 64;
    }();
    return nb;
}

static bool spmv_host_streamed(DenseMat& y, const SellMat& A, const DenseMat& x, const SpmvOptions& o) {
    const int kStreamBlocks = stream_blocks();
    const bool chain = (o.flags & kFlagChain) != 0;
    const bool ok = pinned_host(x) && pinned_host(y) && (!chain || pinned_host(*o.z));
    if (std::getenv("SELLKIT_VERBOSE"))
        std::fprintf(stderr, "[sellkit] host-buffer spmv: %s\n", ok ? "streamed" : "staged (buffers not pinned)");
    if (!ok) return false;
    auto& rt = runtime(A.device);
    rt.copy_streams();
    const gidx ngroups = (gidx(A.nrows_padded) + 31) / 32;
    const int nb = int(std::min<gidx>(kStreamBlocks, ngroups));
    if (nb < 2) return false;
    const std::size_t es = value_bytes(A.dt);
    const lidx w = x.ncols;
    const std::size_t xrow = std::size_t(w) * es;
    std::vector<gidx> rgb(std::size_t(nb) + 1);
    for (int b = 0; b <= nb; ++b) rgb[b] = ngroups * b / nb;
    if (A.watermark_blocks != nb) {
        const int cpr = A.C >= 32 ? 1 : 32 / A.C;  // chunks per row group (C divides 32 or C >= 32)
        std::vector<gidx> cbeg(std::size_t(nb) + 1);
        for (int b = 0; b <= nb; ++b)
            cbeg[b] = A.C <= 32 && 32 % A.C == 0 ? std::min<gidx>(A.nchunks, rgb[b] * cpr)
                                                 : std::min<gidx>(A.nchunks, (rgb[b] * 32 + A.C - 1) / A.C);
        DeviceBuffer d_cb(cbeg.size() * sizeof(gidx), A.device), d_wm(std::size_t(nb) * sizeof(lidx), A.device);
        CK(cudaMemcpyAsync(d_cb.get(), cbeg.data(), cbeg.size() * sizeof(gidx), cudaMemcpyHostToDevice, rt.stream));
        CK(cudaMemsetAsync(d_wm.get(), 0, std::size_t(nb) * sizeof(lidx), rt.stream));
        watermark_kernel<<<dim3(64, nb), 256, 0, rt.stream>>>(A.col.as<lidx>(), A.chunk_offset.as<gidx>(),
                                                             d_cb.as<gidx>(), nb, d_wm.as<lidx>());
        CK(cudaGetLastError());
        A.watermark.assign(std::size_t(nb), 0);
        CK(cudaMemcpyAsync(A.watermark.data(), d_wm.get(), std::size_t(nb) * sizeof(lidx), cudaMemcpyDeviceToHost,
                           rt.stream));
        CK(cudaStreamSynchronize(rt.stream));
        A.watermark_blocks = nb;
    }
    auto* xd = static_cast<unsigned char*>(rt.stage_bytes(0, std::size_t(x.nrows) * xrow));
    auto* yd = static_cast<unsigned char*>(rt.stage_bytes(1, std::size_t(y.nrows) * xrow));
    unsigned char* zd = chain ? static_cast<unsigned char*>(rt.stage_bytes(2, std::size_t(y.nrows) * xrow)) : nullptr;
    DenseMat xdev = densemat_view_plain(A.dt, xd, std::size_t(x.nrows) * w, x.nrows, w, w, Order::row_major);
    DenseMat ydev = densemat_view_plain(A.dt, yd, std::size_t(y.nrows) * w, y.nrows, w, w, Order::row_major);
    DenseMat zdev;
    if (chain) zdev = densemat_view_plain(A.dt, zd, std::size_t(y.nrows) * w, y.nrows, w, w, Order::row_major);

    std::vector<cudaEvent_t> ev(3 * std::size_t(nb));
    for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEvent_t* ev_x = ev.data();
    cudaEvent_t* ev_in = ev.data() + nb;
    cudaEvent_t* ev_c = ev.data() + 2 * nb;
    const auto* xh = reinterpret_cast<const unsigned char*>(x.data);
    auto* yh = reinterpret_cast<unsigned char*>(y.data);
    auto* zh = chain ? reinterpret_cast<unsigned char*>(o.z->data) : nullptr;
    const bool need_y = (o.flags & kFlagAxpby) != 0;
    auto rows_of = [&](int b, gidx& r0, gidx& r1) {
        r0 = std::min<gidx>(y.nrows, rgb[b] * 32);
        r1 = std::min<gidx>(y.nrows, rgb[b + 1] * 32);
    };
    // x slabs (same row split as the blocks) and the per-block y/z inputs, in order
    gidx xdone = 0;
    std::vector<int> slab_for(static_cast<std::size_t>(nb));
    for (int s = 0; s < nb; ++s) {
        const gidx x1 = (s == nb - 1) ? gidx(x.nrows) : std::min<gidx>(x.nrows, gidx(x.nrows) * (s + 1) / nb);
        if (x1 > xdone)
            CK(cudaMemcpyAsync(xd + std::size_t(xdone) * xrow, xh + std::size_t(xdone) * xrow,
                               std::size_t(x1 - xdone) * xrow, cudaMemcpyHostToDevice, rt.h2d));
        CK(cudaEventRecord(ev_x[s], rt.h2d));
        gidx r0, r1;
        rows_of(s, r0, r1);
        if (need_y && r1 > r0)
            CK(cudaMemcpyAsync(yd + std::size_t(r0) * xrow, yh + std::size_t(r0) * xrow, std::size_t(r1 - r0) * xrow,
                               cudaMemcpyHostToDevice, rt.h2d));
        if (chain && r1 > r0)
            CK(cudaMemcpyAsync(zd + std::size_t(r0) * xrow, zh + std::size_t(r0) * xrow, std::size_t(r1 - r0) * xrow,
                               cudaMemcpyHostToDevice, rt.h2d));
        CK(cudaEventRecord(ev_in[s], rt.h2d));
        xdone = x1;
    }
    // SHIFT/VSHIFT/DOT_XY/DOT_XX also read x at the block's own rows: those must be
    // resident too, whatever the block's column watermark
    const bool need_x = (o.flags & (kFlagShift | kFlagVshift | kFlagDotXY | kFlagDotXX)) != 0;
    for (int b = 0; b < nb; ++b) {
        gidx need = gidx(A.watermark[b]);  // largest x row the block reads
        if (need_x) {
            gidx r0, r1;
            rows_of(b, r0, r1);
            if (r1 > r0) need = std::max(need, std::min<gidx>(x.nrows, r1) - 1);
        }
        int s = 0;  // first slab that contains row `need`
        while (s < nb - 1 && std::min<gidx>(x.nrows, gidx(x.nrows) * (s + 1) / nb) <= need) ++s;
        slab_for[b] = std::max(s, b);  // y/z inputs of block b arrive with slab b
    }
    const bool dots = (o.flags & kFlagDots) != 0;
    SpmvOptions run = o;
    run.z = chain ? &zdev : nullptr;
    run.dot = nullptr;
    DeviceBuffer dots_buf(dots ? 3 * std::size_t(w) * es : 16, A.device);
    if (dots) CK(cudaMemsetAsync(dots_buf.get(), 0, 3 * std::size_t(w) * es, rt.stream));
    for (int b = 0; b < nb; ++b) {
        CK(cudaStreamWaitEvent(rt.stream, ev_in[slab_for[b]], 0));
        SpmvHooks h;
        h.rg0 = rgb[b];
        h.rg1 = rgb[b + 1];
        h.accumulate_dots = dots;
        h.dot_accum = dots_buf.get();
        spmv_device(ydev, A, xdev, run, h);
        CK(cudaEventRecord(ev_c[b], rt.stream));
        CK(cudaStreamWaitEvent(rt.d2h, ev_c[b], 0));
        gidx r0, r1;
        rows_of(b, r0, r1);
        if (r1 > r0) {
            CK(cudaMemcpyAsync(yh + std::size_t(r0) * xrow, yd + std::size_t(r0) * xrow, std::size_t(r1 - r0) * xrow,
                               cudaMemcpyDeviceToHost, rt.d2h));
            if (chain)
                CK(cudaMemcpyAsync(zh + std::size_t(r0) * xrow, zd + std::size_t(r0) * xrow,
                                   std::size_t(r1 - r0) * xrow, cudaMemcpyDeviceToHost, rt.d2h));
        }
    }
    if (dots) {
        for (int s = 0; s < 3; ++s)
            if (o.flags & (kFlagDotYY << s))
                CK(cudaMemcpyAsync(static_cast<unsigned char*>(o.dot) + std::size_t(s) * w * es,
                                   static_cast<unsigned char*>(dots_buf.get()) + std::size_t(s) * w * es, w * es,
                                   cudaMemcpyDefault, rt.stream));
    }
    CK(cudaStreamSynchronize(rt.stream));
    CK(cudaStreamSynchronize(rt.d2h));
    CK(cudaStreamSynchronize(rt.h2d));
    for (auto& e : ev) cudaEventDestroy(e);
    return true;
}

void spmv_options_from(Datatype dt, std::uint32_t flags, const void* alpha, const void* beta, const void* gamma,
                       const void* delta, const void* eta, SpmvOptions& o) {
    visit_dt(dt, [&]<class T>() {
        auto put = [&](unsigned char* dst, const void* src, T dflt) {
            T v = dflt;
            if (src) std::memcpy(&v, src, sizeof(T));
            std::memcpy(dst, &v, sizeof(T));
        };
        o.flags = flags;
        put(o.alpha, alpha, Ops<T>::one());
        put(o.beta, beta, Ops<T>::zero());
        put(o.delta, delta, Ops<T>::zero());
        put(o.eta, eta, Ops<T>::zero());
        if (flags & kFlagVshift) {
            o.gamma_list = gamma;
            put(o.gamma, nullptr, Ops<T>::zero());
        } else {
            put(o.gamma, gamma, Ops<T>::zero());
        }
        return 0;
    });
}

KernelVariant select_kernel(lidx chunk_height, lidx block_width, Order order) {
    std::size_t nc = 0, nw = 0;
    const int* cs = config_chunk_heights(&nc);
    const int* ws = config_block_widths(&nw);
    bool c_ok = false, w_ok = false;
    for (std::size_t i = 0; i < nc; ++i) c_ok |= cs[i] == chunk_height;
    for (std::size_t i = 0; i < nw; ++i) w_ok |= ws[i] == block_width;
    if (order == Order::row_major) {
        if (c_ok && w_ok) return {chunk_height, block_width, true};
        if (c_ok) return {chunk_height, 0, true};
        if (w_ok) return {0, block_width, true};
    }
    return {0, 0, false};
}

std::size_t spmv_scratch_bytes(Datatype dt, lidx width, int num_sms) {
    const std::size_t W = std::size_t(width);
    const std::size_t max_parts = std::size_t(num_sms) * 32 * ((W + kGW - 1) / kGW + 1);
    // + 256 B of alignment slack + 256 B holding the dynamic-tile counter
    return (W + 3 * W + max_parts * 3 * std::max<std::size_t>(W, kGW)) * value_bytes(dt) + 512;
}

void spmv_device(DenseMat& y, const SellMat& A, const DenseMat& x, const SpmvOptions& o, const SpmvHooks& hooks) {
    auto& rt = runtime(A.device);
    cudaStream_t st = hooks.stream ? hooks.stream : rt.stream;
    const lidx W = x.ncols;
    const std::size_t es = value_bytes(A.dt);
    const bool want_dots = (o.flags & kFlagDots) != 0;
    const bool rm = y.order == Order::row_major && x.order == Order::row_major &&
                    (!o.z || o.z->order == Order::row_major);
    const bool spec = rm && aligned_for_vectors(x) && aligned_for_vectors(y) && (!o.z || aligned_for_vectors(*o.z));

    visit_dt(A.dt, [&]<class T>() {
        KArgs<T> a{};
        a.chunk_offset = A.chunk_offset.as<gidx>();
        a.chunk_len = A.chunk_len.as<lidx>();
        a.val = A.val.as<T>();
        a.col = A.col.as<lidx>();
        a.nrows = A.nrows;
        a.nrows_padded = A.nrows_padded;
        a.nchunks = A.nchunks;
        a.C = A.C;
        a.y = reinterpret_cast<T*>(y.data);
        a.y_rs = y.row_stride();
        a.y_cs = y.col_step();
        a.x = reinterpret_cast<const T*>(x.data);
        a.x_rs = x.row_stride();
        a.x_cs = x.col_step();
        a.xs = a.x;
        a.xs_rs = a.x_rs;
        a.xs_cs = a.x_cs;
        if (hooks.x_self) {
            a.xs = reinterpret_cast<const T*>(hooks.x_self->data);
            a.xs_rs = hooks.x_self->row_stride();
            a.xs_cs = hooks.x_self->col_step();
        }
        if (o.z) {
            a.z = reinterpret_cast<T*>(o.z->data);
            a.z_rs = o.z->row_stride();
            a.z_cs = o.z->col_step();
        }
        a.width = W;
        a.flags = o.flags;
        a.alpha = scalar_of<T>(o.alpha);
        a.beta = scalar_of<T>(o.beta);
        a.gamma = scalar_of<T>(o.gamma);
        a.delta = scalar_of<T>(o.delta);
        a.eta = scalar_of<T>(o.eta);
        a.defer_mask = hooks.defer_mask;
        a.row_map = hooks.row_map;
        a.rg0 = hooks.rg0;
        a.rg1 = hooks.rg1 < 0 ? (gidx(A.nrows_padded) + 31) / 32 : hooks.rg1;
        if (hooks.rg0 == 0 && hooks.rg1 < 0 && hooks.row_map == nullptr) {  // full sweep
            if (A.sweep_policy == 2 && A.sweep_block_rgs > 0) {
                a.sweep_order = A.sweep_order.as<int>();  // the caller's block order
                a.sweep_brg = A.sweep_block_rgs;
            } else if (spec && A.sweep_policy == 0) {
                int brg = 0;
                gidx nb = 0;
                if (const int* ord = auto_sweep_order(A, W, o.flags, brg, nb)) {
                    a.sweep_order = ord;
                    a.sweep_brg = brg;
                }
            }
        }

        // scratch: [gamma_list W][final dots 3W][partials]
        const std::size_t need = spmv_scratch_bytes(A.dt, W, rt.num_sms);
        auto* sc = static_cast<unsigned char*>(hooks.scratch && hooks.scratch_size >= need ? hooks.scratch
                                                                                        : rt.scratch_bytes(need));
        if (hooks.reserve_sms > 0) a.grid_sms = std::max(1, rt.num_sms - hooks.reserve_sms);
        T* gl = reinterpret_cast<T*>(sc);
        T* res = gl + W;
        a.partial = res + 3 * W;
        a.tile_counter = reinterpret_cast<int*>(sc + need - 256);  // zeroed per launch when used
#if SK_CHECK
        a.xrows = x.nrows;
        a.slots = A.slots;
#endif
        if (o.flags & kFlagVshift) {
            CK(cudaMemcpyAsync(gl, o.gamma_list, W * es, cudaMemcpyDefault, st));
            a.gamma_list = gl;
        }
        const LaunchShape ls = launch_spmv<T>(a, spec, rt, st, A.max_chunk_len);
        CK(cudaGetLastError());
        if (want_dots) {
            T* dst = hooks.accumulate_dots ? static_cast<T*>(hooks.dot_accum) : res;
            dot_final_kernel<T><<<(3 * W + 127) / 128, 128, 0, st>>>(a.partial, ls.nparts, W, ls.layout, o.flags,
                                                                    dst, hooks.accumulate_dots ? 1 : 0);
            CK(cudaGetLastError());
            if (!hooks.accumulate_dots && o.dot) {
                for (int s = 0; s < 3; ++s)
                    if (o.flags & (kFlagDotYY << s))
                        CK(cudaMemcpyAsync(static_cast<unsigned char*>(o.dot) + std::size_t(s) * W * es,
                                           res + std::size_t(s) * W, W * es, cudaMemcpyDefault, st));
            }
        }
        return 0;
    });
}

// spmv.hpp:98-125
void spmv_validate(const DenseMat& y, const SellMat& A, const DenseMat& x, const SpmvOptions& o) {
    SK_REQUIRE(!y.scattered() && !x.scattered(), errc::unsupported,
               "scattered views are not supported by spmv; make a compact clone first");
    SK_REQUIRE(x.nrows == A.ncols, errc::shape_mismatch, "x rows must equal matrix columns");
    SK_REQUIRE(y.nrows == A.nrows, errc::shape_mismatch, "y rows must equal matrix rows");
    SK_REQUIRE(x.ncols == y.ncols, errc::shape_mismatch, "x and y must have the same width");
    SK_REQUIRE(y.data != x.data, errc::invalid_arg, "y must not alias x");
    const auto f = o.flags;
    SK_REQUIRE((f & ~kFlagAll) == 0, errc::invalid_arg, "unknown spmv flag");
    SK_REQUIRE(!((f & kFlagShift) && (f & kFlagVshift)), errc::invalid_arg, "SHIFT and VSHIFT are mutually exclusive");
    if (f & (kFlagShift | kFlagVshift))
        SK_REQUIRE(A.nrows == A.ncols, errc::shape_mismatch, "shift requires a square matrix");
    if (f & kFlagVshift) SK_REQUIRE(o.gamma_list != nullptr, errc::invalid_arg, "VSHIFT requires a gamma list");
    if (f & kFlagDots) SK_REQUIRE(o.dot != nullptr, errc::invalid_arg, "dot flags require a dot buffer");
    if (f & (kFlagDotXY | kFlagDotXX))
        SK_REQUIRE(x.nrows == y.nrows, errc::shape_mismatch, "<x,y> and <x,x> require equal x and y row counts");
    if (f & kFlagChain) {
        SK_REQUIRE(o.z != nullptr, errc::invalid_arg, "CHAIN_AXPBY requires z");
        SK_REQUIRE(o.z->same_shape(y), errc::shape_mismatch, "z must have the shape of y");
        SK_REQUIRE(!o.z->scattered(), errc::unsupported, "z must be compact");
    }
    SK_REQUIRE(x.dt == A.dt && y.dt == A.dt && (!o.z || o.z->dt == A.dt), errc::invalid_arg,
               "datatype mismatch between y and A");
}

// spmv.hpp:129-202
void spmv(DenseMat& y, const SellMat& A, const DenseMat& x_in, const SpmvOptions& o) {
    DenseMat x = x_in;
    spmv_validate(y, A, x, o);
    const auto f = o.flags;
    DeviceGuard g(A.device);
    auto& rt = runtime(A.device);
    if (x.mem == MemKind::host && y.mem == MemKind::host && spmv_host_streamed(y, A, x, o)) return;
    // host operands go through the runtime's reusable staging buffers (slots 0..2)
    Staged xs(x, true, 0);
    Staged ys(y, (f & kFlagAxpby) != 0, 1);
    DenseMat zdummy;
    std::unique_ptr<Staged> zs;
    SpmvOptions run = o;
    if (f & kFlagChain) {
        zs = std::make_unique<Staged>(*o.z, true, 2);
        run.z = &zs->dev;
    } else {
        run.z = nullptr;
    }
    for (DenseMat* m : {&xs.dev, &ys.dev})
        SK_REQUIRE(m->device == A.device, errc::invalid_arg, "vectors must live on the matrix's device");
    spmv_device(ys.dev, A, xs.dev, run, SpmvHooks{});
    if (ys.staged) ys.write_back();
    if (zs && zs->staged) zs->write_back();
    finish(rt);
    if (xs.staged || ys.staged || (zs && zs->staged)) CK(cudaStreamSynchronize(rt.stream));
}

}  // namespace skb
