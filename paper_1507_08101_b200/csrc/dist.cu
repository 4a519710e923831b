// Row-distributed SpMMV with halo exchange.  Design: dist.cuh.
// Reference: /root/reference/proj/src/partition.hpp.
#include <cuda.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <functional>
#include <numeric>

#include "dist.cuh"
#include "handles.cuh"
#include "ops.cuh"

namespace skb {

void exclusive_scan_i64(const gidx* in, gidx* out, gidx n, DeviceRuntime& rt);

namespace {

#define NCK(call)                                                                                  \
    do {                                                                                           \
        ncclResult_t _r = (call);                                                                  \
        if (_r != ncclSuccess) fail(errc::transport, std::string("NCCL: ") + ncclGetErrorString(_r)); \
    } while (0)

// sigma_permutation (sellcs.hpp:80-91) on the host
std::vector<lidx> sigma_permutation_host(const std::vector<lidx>& lens, lidx sigma) {
    const gidx n = gidx(lens.size());
    std::vector<lidx> order(lens.size());
    std::iota(order.begin(), order.end(), 0);
    if (sigma <= 1) return order;
    for (gidx s = 0; s < n; s += sigma) {
        const gidx e = std::min<gidx>(n, s + sigma);
        std::stable_sort(order.begin() + s, order.begin() + e, [&](lidx a, lidx b) { return lens[a] > lens[b]; });
    }
    return order;
}

int owner_of(const std::vector<gidx>& row_offset, gidx row) {
    int lo = 0, hi = int(row_offset.size()) - 2;
    while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (row < row_offset[mid + 1]) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

template <class T>
__global__ void pack_kernel(const T* x, gidx x_rs, gidx x_cs, const lidx* rows, lidx count, lidx w, T* out) {
    const gidx total = gidx(count) * w;
    for (gidx t = blockIdx.x * gidx(blockDim.x) + threadIdx.x; t < total; t += gidx(gridDim.x) * blockDim.x) {
        const gidx i = t / w;
        const lidx j = lidx(t - i * w);
        out[t] = x[gidx(rows[i]) * x_rs + gidx(j) * x_cs];
    }
}

template <class T>
__global__ void rank_sum_kernel(const T* all, int nranks, int n, T* out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    T s = all[t];
    for (int r = 1; r < nranks; ++r) s = Ops<T>::add(s, all[gidx(r) * n + t]);
    out[t] = s;
}

int pack_grid(gidx work) { return int(std::max<gidx>(1, std::min<gidx>((work + 255) / 256, 4096))); }

std::unique_ptr<Crs> crs_upload(Datatype dt, gidx nrows, gidx ncols, const std::vector<gidx>& rowptr,
                                const std::vector<gidx>& col, const std::vector<unsigned char>& val) {
    auto a = std::make_unique<Crs>();
    a->dt = dt;
    a->nrows = nrows;
    a->ncols = ncols;
    a->nnz = rowptr.back();
    a->device = current_device();
    auto& rt = runtime(a->device);
    a->rowptr = DeviceBuffer(rowptr.size() * sizeof(gidx), a->device);
    a->col = DeviceBuffer(std::max<std::size_t>(col.size() * sizeof(gidx), 8), a->device);
    a->val = DeviceBuffer(std::max<std::size_t>(val.size(), 16), a->device);
    CK(cudaMemcpyAsync(a->rowptr.get(), rowptr.data(), rowptr.size() * sizeof(gidx), cudaMemcpyHostToDevice, rt.stream));
    if (!col.empty()) {
        CK(cudaMemcpyAsync(a->col.get(), col.data(), col.size() * sizeof(gidx), cudaMemcpyHostToDevice, rt.stream));
        CK(cudaMemcpyAsync(a->val.get(), val.data(), val.size(), cudaMemcpyHostToDevice, rt.stream));
    }
    CK(cudaStreamSynchronize(rt.stream));
    return a;
}

ncclDataType_t nccl_type(Datatype dt, std::size_t& mult) {
    switch (dt) {
        case Datatype::r32: mult = 1; return ncclFloat32;
        case Datatype::r64: mult = 1; return ncclFloat64;
        case Datatype::c32: mult = 2; return ncclFloat32;
        case Datatype::c64: mult = 2; return ncclFloat64;
    }
    mult = 1;
    return ncclFloat64;
}

}  // namespace

// ------------------------------------------------------------------ planning

// partition.hpp:45-94
std::vector<gidx> compute_partition(gidx n, const lidx* rowlens, const std::vector<double>& weights, bool by_nnz) {
    const int k = int(weights.size());
    SK_REQUIRE(n > 0, errc::invalid_arg, "empty matrix");
    SK_REQUIRE(k >= 1, errc::invalid_arg, "need at least one rank");
    SK_REQUIRE(gidx(k) <= n, errc::invalid_arg, "more ranks than rows");
    double total_w = 0.0;
    for (double w : weights) {
        SK_REQUIRE(w > 0.0, errc::invalid_arg, "weights must be positive");
        total_w += w;
    }
    std::vector<gidx> prefix;
    gidx total_nnz = 0;
    if (by_nnz) {
        SK_REQUIRE(rowlens != nullptr, errc::invalid_arg, "ByNnz partitioning needs per-row lengths");
        prefix.assign(std::size_t(n) + 1, 0);
        for (gidx r = 0; r < n; ++r) prefix[r + 1] = prefix[r] + rowlens[r];
        total_nnz = prefix[n];
    }
    std::vector<gidx> off(std::size_t(k) + 1, 0);
    off[k] = n;
    double cum = 0.0;
    for (int i = 1; i < k; ++i) {
        cum += weights[i - 1];
        const double share = cum / total_w;
        gidx b;
        if (!by_nnz || total_nnz == 0) {
            b = static_cast<gidx>(std::floor(double(n) * share + 0.5));
        } else {
            const double target = double(total_nnz) * share;
            gidx p = 0;
            while (p < n && double(prefix[p]) < target) ++p;
            if (p > 0 && std::abs(double(prefix[p - 1]) - target) <= std::abs(double(prefix[p]) - target)) b = p - 1;
            else b = p;
        }
        b = std::max(b, off[i - 1] + 1);
        b = std::min(b, n - (k - i));
        off[i] = b;
    }
    return off;
}

// partition.hpp:136-220
RankPlan plan_rank(Datatype dt, const gidx* rowptr, const gidx* col, const void* val, lidx nrows,
                   const std::vector<gidx>& row_offset, int rank) {
    RankPlan p;
    p.dt = dt;
    p.rank = rank;
    p.nranks = int(row_offset.size()) - 1;
    SK_REQUIRE(rank >= 0 && rank < p.nranks, errc::invalid_arg, "rank out of range");
    p.row_offset = row_offset;
    const gidx r0 = row_offset[rank], r1 = row_offset[rank + 1];
    SK_REQUIRE(gidx(nrows) == r1 - r0, errc::shape_mismatch, "row block does not match the partition plan");
    const gidx n = row_offset.back();
    p.first_row = r0;
    p.nrows = nrows;
    const std::size_t es = value_bytes(dt);
    const auto* vb = static_cast<const unsigned char*>(val);
    const gidx base = rowptr[0];

    std::vector<gidx> halo;
    for (gidx k = rowptr[0]; k < rowptr[nrows]; ++k) {
        const gidx c = col[k - base];
        SK_REQUIRE(c >= 0 && c < n, errc::invalid_arg, "column index out of range");
        if (c < r0 || c >= r1) halo.push_back(c);
    }
    std::sort(halo.begin(), halo.end());
    halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
    p.halo_cols = halo;
    p.halo_owner.resize(halo.size());
    for (std::size_t i = 0; i < halo.size(); ++i) p.halo_owner[i] = owner_of(row_offset, halo[i]);

    p.lrowptr.assign(std::size_t(nrows) + 1, 0);
    p.rrowptr.assign(std::size_t(nrows) + 1, 0);
    p.lens.resize(std::size_t(nrows));
    for (lidx r = 0; r < nrows; ++r) {
        const gidx b = rowptr[r] - base, e = rowptr[r + 1] - base;
        p.lens[r] = lidx(e - b);
        for (gidx k = b; k < e; ++k) {
            const gidx c = col[k];
            if (c >= r0 && c < r1) {
                p.lcol.push_back(c - r0);
                p.lval.insert(p.lval.end(), vb + k * es, vb + (k + 1) * es);
            } else {
                p.rcol.push_back(gidx(std::lower_bound(halo.begin(), halo.end(), c) - halo.begin()));
                p.rval.insert(p.rval.end(), vb + k * es, vb + (k + 1) * es);
            }
        }
        p.lrowptr[r + 1] = gidx(p.lcol.size());
        p.rrowptr[r + 1] = gidx(p.rcol.size());
    }
    int cur = -1;
    for (std::size_t i = 0; i < halo.size(); ++i) {
        if (p.halo_owner[i] != cur) {
            cur = p.halo_owner[i];
            p.recv_owner.push_back(cur);
            p.recv_count.push_back(0);
            p.recv_offset.push_back(lidx(i));
        }
        p.recv_count.back()++;
    }
    return p;
}

void plan_set_sends(RankPlan& p, int to, const gidx* cols, lidx count) {
    SK_REQUIRE(to >= 0 && to < p.nranks && to != p.rank, errc::invalid_arg, "bad send destination");
    std::vector<lidx> rows(static_cast<std::size_t>(count));
    for (lidx i = 0; i < count; ++i) {
        const gidx c = cols[i];
        SK_REQUIRE(c >= p.first_row && c < p.first_row + p.nrows, errc::invalid_arg, "requested column not owned");
        rows[i] = lidx(c - p.first_row);
    }
    // keep send lists ordered by destination rank (partition.hpp:268-277)
    auto it = std::lower_bound(p.send_to.begin(), p.send_to.end(), to);
    const std::size_t pos = std::size_t(it - p.send_to.begin());
    if (it != p.send_to.end() && *it == to) {
        p.send_local_rows[pos] = std::move(rows);
    } else {
        p.send_to.insert(it, to);
        p.send_local_rows.insert(p.send_local_rows.begin() + pos, std::move(rows));
    }
}

RankPart::~RankPart() {
    if (comm) cudaStreamDestroy(comm);
    if (ev_x) cudaEventDestroy(ev_x);
    if (ev_halo) cudaEventDestroy(ev_halo);
    if (ev_done) cudaEventDestroy(ev_done);
}

// Local part (permute_columns = true) and the boundary-row remote part, both with
// the sigma order of the combined row lengths (partition.hpp:193-209).
void rank_build_device(RankPart& part, lidx C, lidx sigma) {
    RankPlan& p = part.plan;
    DeviceGuard g(part.device);
    auto& rt = runtime(part.device);
    const std::vector<lidx> order = sigma_permutation_host(p.lens, sigma);
    DeviceBuffer d_order(std::max<std::size_t>(order.size() * sizeof(lidx), 4), part.device);
    CK(cudaMemcpyAsync(d_order.get(), order.data(), order.size() * sizeof(lidx), cudaMemcpyHostToDevice, rt.stream));
    {
        auto lcrs = crs_upload(p.dt, p.nrows, p.nrows, p.lrowptr, p.lcol, p.lval);
        BuildOptions opt;
        opt.permute_columns = true;
        opt.imposed_order = d_order.as<lidx>();
        part.local = sell_build(*lcrs, C, sigma, opt);
    }
    // stored order -> rows with remote entries
    std::vector<lidx> rrows;
    std::vector<gidx> rp{0};
    std::vector<gidx> rc;
    std::vector<unsigned char> rv;
    const std::size_t es = value_bytes(p.dt);
    std::vector<std::uint32_t> mask((std::size_t(p.nrows) + 31) / 32, 0u);
    for (lidx k = 0; k < p.nrows; ++k) {
        const lidx o = order[k];
        const gidx b = p.rrowptr[o], e = p.rrowptr[o + 1];
        if (e == b) continue;
        rrows.push_back(k);
        mask[std::size_t(k) >> 5] |= 1u << (k & 31);
        rc.insert(rc.end(), p.rcol.begin() + b, p.rcol.begin() + e);
        rv.insert(rv.end(), p.rval.begin() + b * es, p.rval.begin() + e * es);
        rp.push_back(gidx(rc.size()));
    }
    part.defer_mask = DeviceBuffer(std::max<std::size_t>(mask.size() * 4, 4), part.device);
    CK(cudaMemcpyAsync(part.defer_mask.get(), mask.data(), mask.size() * 4, cudaMemcpyHostToDevice, rt.stream));
    if (!rrows.empty()) {
        // the remote part keeps each row's entries in CRS order, so its per-row sums
        // are the reference's whatever the chunking; sigma = 1 keeps row_map monotone
        auto rcrs = crs_upload(p.dt, gidx(rrows.size()), gidx(std::max<std::size_t>(1, p.halo_cols.size())), rp, rc, rv);
        BuildOptions opt;
        opt.permute_columns = false;
        part.remote = sell_build(*rcrs, C, 1, opt);
        part.row_map = DeviceBuffer(rrows.size() * sizeof(lidx), part.device);
        CK(cudaMemcpyAsync(part.row_map.get(), rrows.data(), rrows.size() * sizeof(lidx), cudaMemcpyHostToDevice,
                           rt.stream));
    }
    if (!part.comm) {
        // highest priority: the small pack kernels get SMs ahead of the persistent local sweep
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&part.comm, cudaStreamNonBlocking, hi));
        CK(cudaEventCreateWithFlags(&part.ev_x, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&part.ev_halo, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&part.ev_done, cudaEventDisableTiming));
    }
    CK(cudaStreamSynchronize(rt.stream));
}

namespace {

std::vector<lidx> download_perm_uncached(const SellMat& m) {
    std::vector<lidx> h(std::size_t(m.nrows));
    DeviceGuard g(m.device);
    CK(cudaMemcpy(h.data(), m.row_perm.get(), h.size() * sizeof(lidx), cudaMemcpyDeviceToHost));
    return h;
}

// original local row -> stored row of a rank's local part, downloaded once
const std::vector<lidx>& rank_perm(const RankPart& part) {
    if (part.perm_host.size() != std::size_t(part.plan.nrows)) part.perm_host = download_perm_uncached(*part.local);
    return part.perm_host;
}

// send rows in the owner's stored space (partition.hpp:274-275)
void build_send_rows(RankPart& part) {
    const std::vector<lidx>& perm = rank_perm(part);
    DeviceGuard g(part.device);
    auto& rt = runtime(part.device);
    part.send_rows.clear();
    for (auto& rows : part.plan.send_local_rows) {
        std::vector<lidx> stored(rows.size());
        for (std::size_t i = 0; i < rows.size(); ++i) stored[i] = perm[rows[i]];
        DeviceBuffer b(std::max<std::size_t>(stored.size() * sizeof(lidx), 4), part.device);
        CK(cudaMemcpyAsync(b.get(), stored.data(), stored.size() * sizeof(lidx), cudaMemcpyHostToDevice, rt.stream));
        part.send_rows.push_back(std::move(b));
    }
    CK(cudaStreamSynchronize(rt.stream));
}

void ensure_scratch(RankScratch& s, const RankPart& part, lidx w) {
    if (s.width == w && s.dots.get()) return;
    DeviceGuard g(part.device);
    CK(cudaDeviceSynchronize());
    const std::size_t es = value_bytes(part.plan.dt);
    std::size_t nsend = 0;
    for (auto& r : part.plan.send_local_rows) nsend += r.size();
    s.width = w;
    s.halo = DeviceBuffer(std::max<std::size_t>(part.plan.halo_cols.size() * w * es, 32), part.device);
    s.sendbuf = DeviceBuffer(std::max<std::size_t>(nsend * w * es, 32), part.device);
    s.dots = DeviceBuffer(std::max<std::size_t>(3 * std::size_t(w) * es, 32), part.device);
}

// local sweep (+ deferred-row hooks) and remote sweep of one rank; dots -> scratch.dots
// `extra` supplies the sweeps' scratch (graph-stable, rank-owned) and the SMs the
// local sweep leaves to a concurrent halo pack; stream/dot fields are set here.
void rank_sweeps(RankPart& part, RankScratch& sc, DenseMat& y, const DenseMat& x, const SpmvOptions& o, DenseMat* z,
                 bool nocomm, cudaStream_t st, const std::function<void()>& before_remote,
                 const SpmvHooks& extra = SpmvHooks{}) {
    const std::uint32_t dots = o.flags & kFlagDots;
    const bool chain = (o.flags & kFlagChain) != 0;
    const bool has_remote = part.remote != nullptr && !nocomm;
    SpmvOptions base = o;
    base.dot = nullptr;
    base.z = chain ? z : nullptr;
    SpmvHooks hl;
    hl.scratch = extra.scratch;
    hl.scratch_size = extra.scratch_size;
    hl.reserve_sms = extra.reserve_sms;
    hl.stream = st;
    hl.accumulate_dots = true;
    hl.dot_accum = sc.dots.get();
    // rows finished by the remote sweep contribute their dots/chain there; without dots
    // or chain the mask is not needed and the local sweep runs the plain y = A x kernel
    if (has_remote && (dots || chain)) hl.defer_mask = part.defer_mask.as<std::uint32_t>();
    CK(cudaMemsetAsync(sc.dots.get(), 0, 3 * std::size_t(x.ncols) * value_bytes(part.plan.dt), st));
    spmv_device(y, *part.local, x, base, hl);
    if (!has_remote) return;
    before_remote();
    // accum opts (partition.hpp:454-457): alpha, beta = 1, AXPBY, plus the deferred dots/chain
    SpmvOptions acc = o;
    acc.flags = kFlagAxpby | dots | (chain ? kFlagChain : 0u);
    visit_dt(part.plan.dt, [&]<class T>() {
        T one = Ops<T>::one();
        std::memcpy(acc.beta, &one, sizeof(T));
        return 0;
    });
    acc.dot = nullptr;
    acc.z = chain ? z : nullptr;
    DenseMat halo = densemat_view_plain(part.plan.dt, sc.halo.get(), part.plan.halo_cols.size() * x.ncols,
                                        lidx(part.plan.halo_cols.size()), x.ncols, x.ncols, Order::row_major);
    SpmvHooks hr;
    hr.scratch = extra.scratch;
    hr.scratch_size = extra.scratch_size;
    hr.stream = st;
    hr.row_map = part.row_map.as<lidx>();
    hr.accumulate_dots = true;
    hr.dot_accum = sc.dots.get();
    hr.x_self = &x;
    spmv_device(y, *part.remote, halo, acc, hr);
}

}  // namespace

// ---------------------------------------------------------- single process

std::unique_ptr<DistContext> dist_context_create(const Crs& a, const std::vector<double>& weights, bool by_nnz,
                                                 lidx C, lidx sigma, bool record) {
    crs_validate(a);
    SK_REQUIRE(a.nrows == a.ncols, errc::invalid_arg, "row-wise distribution requires a square matrix");
    std::vector<gidx> rowptr, col;
    std::vector<unsigned char> val;
    {
        DeviceGuard g(a.device);
        crs_download(a, rowptr, col, val);
    }
    auto ctx = std::make_unique<DistContext>();
    ctx->dt = a.dt;
    ctx->n = a.nrows;
    ctx->nnz = a.nnz;
    ctx->C = C;
    ctx->sigma = sigma;
    ctx->record = record;
    std::vector<lidx> lens(std::size_t(a.nrows));
    for (gidx r = 0; r < a.nrows; ++r) lens[r] = lidx(rowptr[r + 1] - rowptr[r]);
    ctx->row_offset = compute_partition(a.nrows, lens.data(), weights, by_nnz);
    const int k = int(weights.size());
    int ndev = 1;
    CK(cudaGetDeviceCount(&ndev));
    const std::size_t es = value_bytes(a.dt);
    for (int r = 0; r < k; ++r) {
        auto part = std::make_unique<RankPart>();
        part->device = (a.device + r) % ndev;
        const gidx r0 = ctx->row_offset[r], r1 = ctx->row_offset[r + 1];
        part->plan = plan_rank(a.dt, rowptr.data() + r0, col.data() + rowptr[r0], val.data() + rowptr[r0] * es,
                               lidx(r1 - r0), ctx->row_offset, r);
        ctx->ranks.push_back(std::move(part));
    }
    // send lists: ascending requesting rank, within that ascending global column (partition.hpp:268-277)
    for (int r = 0; r < k; ++r) {
        const RankPlan& p = ctx->ranks[r]->plan;
        for (std::size_t q = 0; q < p.recv_owner.size(); ++q) {
            const int owner = p.recv_owner[q];
            plan_set_sends(ctx->ranks[owner]->plan, r, p.halo_cols.data() + p.recv_offset[q], p.recv_count[q]);
        }
    }
    for (int r = 0; r < k; ++r) {
        rank_build_device(*ctx->ranks[r], C, sigma);
        build_send_rows(*ctx->ranks[r]);
    }
    // peer access between the devices the ranks use (halo stores go straight into the
    // peer's buffer); the pairs that were enabled decide the direct-store path
    ctx->ndev = ndev;
    ctx->peer_ok.assign(std::size_t(ndev) * ndev, 0);
    std::vector<int> used;
    for (auto& part : ctx->ranks)
        if (std::find(used.begin(), used.end(), part->device) == used.end()) used.push_back(part->device);
    for (int i : used)
        for (int j : used) {
            if (i == j) continue;
            int ok = 0;
            if (cudaDeviceCanAccessPeer(&ok, i, j) != cudaSuccess) ok = 0;
            if (ok) {
                DeviceGuard g(i);
                const cudaError_t e = cudaDeviceEnablePeerAccess(j, 0);
                ok = e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled;
                cudaGetLastError();
            }
            ctx->peer_ok[std::size_t(i) * ndev + j] = char(ok);
        }
    ctx->scratch.resize(std::size_t(k));
    return ctx;
}

std::unique_ptr<DistVec> dist_vec_create(const DistContext& ctx, lidx width, Order order) {
    auto v = std::make_unique<DistVec>();
    v->width = width;
    v->order = order;
    for (auto& part : ctx.ranks) {
        DeviceGuard g(part->device);
        v->parts.push_back(densemat_create(ctx.dt, part->plan.nrows, width, order));
    }
    return v;
}

// partition.hpp:302-326 (parts live in each rank's stored / permuted space)
void dist_scatter(const DistContext& ctx, const DenseMat& global, DistVec& v) {
    SK_REQUIRE(global.nrows == ctx.n && global.ncols == v.width, errc::shape_mismatch, "global vector shape mismatch");
    SK_REQUIRE(global.dt == ctx.dt, errc::invalid_arg, "datatype mismatch between context and vector");
    const std::size_t es = value_bytes(ctx.dt);
    const lidx w = v.width;
    std::vector<unsigned char> host(std::size_t(ctx.n) * w * es);
    densemat_copy_out(global, host.data(), std::size_t(ctx.n) * w);
    for (std::size_t r = 0; r < ctx.ranks.size(); ++r) {
        const auto& part = *ctx.ranks[r];
        const std::vector<lidx>& perm = rank_perm(part);
        std::vector<unsigned char> buf(std::size_t(part.plan.nrows) * w * es);
        for (lidx i = 0; i < part.plan.nrows; ++i)
            std::memcpy(&buf[std::size_t(perm[i]) * w * es], &host[std::size_t(part.plan.first_row + i) * w * es],
                        w * es);
        DeviceGuard g(part.device);
        densemat_copy_in(v.parts[r], buf.data(), std::size_t(part.plan.nrows) * w);
    }
}

void dist_gather(const DistContext& ctx, const DistVec& v, DenseMat& out) {
    SK_REQUIRE(out.nrows == ctx.n && out.ncols == v.width, errc::shape_mismatch, "global vector shape mismatch");
    SK_REQUIRE(out.dt == ctx.dt, errc::invalid_arg, "datatype mismatch between context and vector");
    const std::size_t es = value_bytes(ctx.dt);
    const lidx w = v.width;
    std::vector<unsigned char> host(std::size_t(ctx.n) * w * es);
    for (std::size_t r = 0; r < ctx.ranks.size(); ++r) {
        const auto& part = *ctx.ranks[r];
        const std::vector<lidx>& perm = rank_perm(part);
        std::vector<unsigned char> buf(std::size_t(part.plan.nrows) * w * es);
        {
            DeviceGuard g(part.device);
            densemat_copy_out(v.parts[r], buf.data(), buf.size() / es);
        }
        for (lidx i = 0; i < part.plan.nrows; ++i)
            std::memcpy(&host[std::size_t(part.plan.first_row + i) * w * es], &buf[std::size_t(perm[i]) * w * es],
                        w * es);
    }
    densemat_copy_in(out, host.data(), host.size() / es);
}

// partition.hpp:423-600
void dist_spmv(DistVec& y, DistContext& ctx, const DistVec& x, const SpmvOptions& o, int mode, DistVec* z,
               bool nocomm) {
    const int k = int(ctx.ranks.size());
    SK_REQUIRE(x.width == y.width, errc::shape_mismatch, "x and y must have the same width");
    SK_REQUIRE(int(x.parts.size()) == k && int(y.parts.size()) == k, errc::invalid_arg, "vector/context mismatch");
    const bool chain = (o.flags & kFlagChain) != 0;
    SK_REQUIRE(!chain || z != nullptr, errc::invalid_arg, "CHAIN_AXPBY requires z");
    const std::uint32_t dots = o.flags & kFlagDots;
    SK_REQUIRE(!dots || o.dot != nullptr, errc::invalid_arg, "dot flags require a dot buffer");
    SK_REQUIRE((o.flags & ~kFlagAll) == 0, errc::invalid_arg, "unknown spmv flag");
    SK_REQUIRE(!((o.flags & kFlagShift) && (o.flags & kFlagVshift)), errc::invalid_arg,
               "SHIFT and VSHIFT are mutually exclusive");
    const lidx w = x.width;
    const std::size_t es = value_bytes(ctx.dt);
    for (int r = 0; r < k; ++r) ensure_scratch(ctx.scratch[r], *ctx.ranks[r], w);
    // optional timeline (sellkit_ext_ctx_set_trace): per rank, timing events at the
    // exchange start / end (comm stream) and the local-sweep start / end and remote-sweep
    // end (main stream), relative to one start event on rank 0's device
    const bool trace = ctx.trace;
    auto tev = [&](int r, int i) -> cudaEvent_t { return ctx.tev[std::size_t(r) * kTraceEvents + i + 1]; };
    if (trace) {
        if (ctx.tev.empty()) {
            ctx.tev.resize(std::size_t(k) * kTraceEvents + 1);
            for (std::size_t i = 0; i < ctx.tev.size(); ++i) {
                DeviceGuard g(ctx.ranks[i == 0 ? 0 : (i - 1) / kTraceEvents]->device);
                CK(cudaEventCreate(&ctx.tev[i]));
            }
        }
        DeviceGuard g(ctx.ranks[0]->device);
        CK(cudaEventRecord(ctx.tev[0], runtime(ctx.ranks[0]->device).stream));
    }

    // 1. halo exchange: each owner packs straight into the requester's halo block
    if (!nocomm) {
        for (int r = 0; r < k; ++r) {
            RankPart& part = *ctx.ranks[r];
            DeviceGuard g(part.device);
            auto& rt = runtime(part.device);
            CK(cudaEventRecord(part.ev_x, rt.stream));
            CK(cudaStreamWaitEvent(part.comm, part.ev_x, 0));
            if (trace) CK(cudaEventRecord(tev(r, 0), part.comm));
            for (std::size_t s = 0; s < part.plan.send_to.size(); ++s) {
                const int to = part.plan.send_to[s];
                RankPart& dst = *ctx.ranks[to];
                // previous remote sweep of `to` must have consumed its halo
                CK(cudaStreamWaitEvent(part.comm, dst.ev_done, 0));
                const RankPlan& dp = dst.plan;
                const auto it = std::find(dp.recv_owner.begin(), dp.recv_owner.end(), r);
                const std::size_t q = std::size_t(it - dp.recv_owner.begin());
                const lidx cnt = lidx(part.plan.send_local_rows[s].size());
                auto* dptr = static_cast<unsigned char*>(ctx.scratch[to].halo.get()) +
                             std::size_t(dp.recv_offset[q]) * w * es;
                const bool can = ctx.direct(part.device, dst.device);
                const DenseMat& xr = x.parts[r];
                visit_dt(ctx.dt, [&]<class T>() {
                    T* out = can ? reinterpret_cast<T*>(dptr) : ctx.scratch[r].sendbuf.as<T>();
                    pack_kernel<T><<<pack_grid(gidx(cnt) * w), 256, 0, part.comm>>>(
                        reinterpret_cast<const T*>(xr.data), xr.row_stride(), xr.col_step(),
                        part.send_rows[s].as<lidx>(), cnt, w, out);
                    return 0;
                });
                CK(cudaGetLastError());
                if (!can)
                    CK(cudaMemcpyPeerAsync(dptr, dst.device, ctx.scratch[r].sendbuf.get(), part.device,
                                           std::size_t(cnt) * w * es, part.comm));
                if (ctx.record) {
                    ctx.bytes += std::uint64_t(cnt) * w * es;
                    ctx.msgs += 1;
                }
            }
            if (trace) CK(cudaEventRecord(tev(r, 1), part.comm));
            CK(cudaEventRecord(part.ev_halo, part.comm));
        }
    }
    // 2. sweeps; remote sweeps wait for every owner that sends to them
    for (int r = 0; r < k; ++r) {
        RankPart& part = *ctx.ranks[r];
        DeviceGuard g(part.device);
        auto& rt = runtime(part.device);
        if (!nocomm && mode == 0) {  // NO_OVERLAP: the whole exchange precedes the sweeps
            for (int owner : part.plan.recv_owner) CK(cudaStreamWaitEvent(rt.stream, ctx.ranks[owner]->ev_halo, 0));
        }
        DenseMat* zr = chain ? &z->parts[r] : nullptr;
        if (trace) CK(cudaEventRecord(tev(r, 2), rt.stream));
        bool local_marked = false;
        rank_sweeps(part, ctx.scratch[r], const_cast<DenseMat&>(y.parts[r]), x.parts[r], o, zr, nocomm, rt.stream,
                    [&] {
                        if (trace) CK(cudaEventRecord(tev(r, 3), rt.stream));
                        local_marked = true;
                        for (int owner : part.plan.recv_owner)
                            CK(cudaStreamWaitEvent(rt.stream, ctx.ranks[owner]->ev_halo, 0));
                    });
        if (trace && !local_marked) CK(cudaEventRecord(tev(r, 3), rt.stream));
        if (trace) CK(cudaEventRecord(tev(r, 4), rt.stream));
        CK(cudaEventRecord(part.ev_done, rt.stream));
    }
    if (trace) {
        ctx.timeline.assign(std::size_t(k) * kTraceEvents, -1.0);
        for (int r = 0; r < k; ++r) {
            DeviceGuard g(ctx.ranks[r]->device);
            CK(cudaDeviceSynchronize());
        }
        for (int r = 0; r < k; ++r) {
            if (ctx.ranks[r]->device != ctx.ranks[0]->device) continue;  // one clock per device
            for (int i = 0; i < kTraceEvents; ++i) {
                if (nocomm && i < 2) continue;
                float ms = 0.f;
                if (cudaEventElapsedTime(&ms, ctx.tev[0], tev(r, i)) == cudaSuccess)
                    ctx.timeline[std::size_t(r) * kTraceEvents + i] = ms;
                cudaGetLastError();
            }
        }
    }
    // 3. dots: per-rank partials summed in rank order on rank 0's device
    //    (partition.hpp:379-394), one copy of the requested thirds to the caller
    if (dots) {
        RankPart& p0 = *ctx.ranks[0];
        DeviceGuard g(p0.device);
        auto& rt0 = runtime(p0.device);
        const std::size_t db = 3 * std::size_t(w) * es;
        if (ctx.dots_all.bytes() < std::size_t(k) * db) ctx.dots_all = DeviceBuffer(std::size_t(k) * db, p0.device);
        auto* all = static_cast<unsigned char*>(ctx.dots_all.get());
        for (int r = 0; r < k; ++r) {
            RankPart& part = *ctx.ranks[r];
            if (r > 0) CK(cudaStreamWaitEvent(rt0.stream, part.ev_done, 0));
            CK(cudaMemcpyPeerAsync(all + std::size_t(r) * db, p0.device, ctx.scratch[r].dots.get(), part.device, db,
                                   rt0.stream));
        }
        visit_dt(ctx.dt, [&]<class T>() {
            rank_sum_kernel<T><<<(3 * w + 127) / 128, 128, 0, rt0.stream>>>(ctx.dots_all.as<T>(), k, 3 * w,
                                                                           ctx.scratch[0].dots.as<T>());
            return 0;
        });
        CK(cudaGetLastError());
        for (int s = 0; s < 3; ++s)
            if (o.flags & (kFlagDotYY << s))
                CK(cudaMemcpyAsync(static_cast<unsigned char*>(o.dot) + std::size_t(s) * w * es,
                                   static_cast<unsigned char*>(ctx.scratch[0].dots.get()) + std::size_t(s) * w * es,
                                   w * es, cudaMemcpyDefault, rt0.stream));
        if (ctx.record && k > 1) {
            ctx.msgs += 2 * std::uint64_t(k - 1);
            ctx.bytes += 2 * std::uint64_t(k - 1) * 3 * w * es;
        }
    }
    if (sync_mode())
        for (auto& part : ctx.ranks) {
            DeviceGuard g(part->device);
            CK(cudaStreamSynchronize(runtime(part->device).stream));
        }
}

// ------------------------------------------------------ one process per GPU
//
// Transports of the per-process rank context:
//   nccl : pack -> ncclSend/ncclRecv pairs in one group on the comm stream; dots
//          all-gathered with NCCL and summed in rank order.
//   ipc  : every rank exports (CUDA IPC) a send buffer with one slot per
//          destination, a dot-partial slot and a flag block.  The owner packs its
//          send lists into its own slots (a local gather kernel), then raises the
//          receiver's "full" flag; the receiver pulls its slot with a copy-engine
//          peer copy (NVLink on a multi-GPU node, no SMs taken from the local sweep)
//          and raises the owner's "free" flag.  Flags are 0/1 handshakes written and
//          waited on by stream memory operations (cuStreamWriteValue32 /
//          cuStreamWaitValue32): no kernel ever waits on another rank, and the
//          values are the same every step, so the whole step can be captured in a
//          CUDA graph.  Dots travel the same way (a 3w slot per rank).

namespace {

// driver entry points resolved through the runtime (no link-time libcuda dependency)
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <class F>
F driver_fn(const char* name) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CK(cudaGetDriverEntryPointByVersion(name, &fn, 12000, cudaEnableDefault, &q));
    SK_REQUIRE(fn != nullptr && q == cudaDriverEntryPointSuccess, errc::unsupported,
               std::string("driver entry point unavailable: ") + name);
    return reinterpret_cast<F>(fn);
}

void cu_check(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS)
        fail(errc::transport, std::string("CUDA driver error ") + std::to_string(int(r)) + " in " + what);
}

void flag_wait(cudaStream_t st, const std::uint32_t* addr, std::uint32_t v) {
    static const WaitValueFn fn = driver_fn<WaitValueFn>("cuStreamWaitValue32");
    cu_check(fn(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), v, CU_STREAM_WAIT_VALUE_EQ),
             "cuStreamWaitValue32");
}

void flag_set(cudaStream_t st, std::uint32_t* addr, std::uint32_t v) {
    // default flags: the write is ordered after (and fenced against) the stream's earlier work
    static const WriteValueFn fn = driver_fn<WriteValueFn>("cuStreamWriteValue32");
    cu_check(fn(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), v, CU_STREAM_WRITE_VALUE_DEFAULT),
             "cuStreamWriteValue32");
}

constexpr char kIpcMagic[8] = {'S', 'K', 'I', 'P', 'C', '0', '1', 0};

struct IpcBlobHead {
    char magic[8];
    int rank, nranks, max_w, es, device, pad;
    cudaIpcMemHandle_t send, dots, flags;
};
// followed by gidx seg_row[nranks]: first row of destination d's slot in the send buffer (-1: none)

std::size_t ipc_blob_bytes(int nranks) { return sizeof(IpcBlobHead) + std::size_t(nranks) * sizeof(gidx); }

// 16-byte units of whole rows (row bytes and strides multiples of 16)
__global__ void pack16_kernel(const int4* x, gidx x_rs16, const lidx* rows, lidx count, int u, int4* out) {
    const gidx total = gidx(count) * u;
    for (gidx t = blockIdx.x * gidx(blockDim.x) + threadIdx.x; t < total; t += gidx(gridDim.x) * blockDim.x) {
        const gidx i = t / u;
        const int j = int(t - i * u);
        out[t] = x[gidx(__ldg(rows + i)) * x_rs16 + j];
    }
}

// gather x rows `rows[0..cnt)` (all `w` columns) into out[cnt x w]
void launch_pack(Datatype dt, const DenseMat& x, const lidx* rows, lidx cnt, lidx w, void* out, cudaStream_t st) {
    if (cnt == 0) return;
    const std::size_t es = value_bytes(dt);
    const std::size_t rb = std::size_t(w) * es;
    const bool vec = x.order == Order::row_major && rb % 16 == 0 &&
                     (std::size_t(x.row_stride()) * es) % 16 == 0 && reinterpret_cast<std::uintptr_t>(x.data) % 16 == 0 &&
                     reinterpret_cast<std::uintptr_t>(out) % 16 == 0;
    if (vec) {
        const int u = int(rb / 16);
        pack16_kernel<<<pack_grid(gidx(cnt) * u), 256, 0, st>>>(reinterpret_cast<const int4*>(x.data),
                                                                 gidx(std::size_t(x.row_stride()) * es / 16), rows,
                                                                 cnt, u, static_cast<int4*>(out));
    } else {
        visit_dt(dt, [&]<class T>() {
            pack_kernel<T><<<pack_grid(gidx(cnt) * w), 256, 0, st>>>(
                reinterpret_cast<const T*>(x.data), x.row_stride(), x.col_step(), rows, cnt, w, static_cast<T*>(out));
            return 0;
        });
    }
    CK(cudaGetLastError());
}

// identity of one step: everything a captured graph bakes in
struct StepKey {
    const void* y = nullptr;
    const void* x = nullptr;
    const void* z = nullptr;
    const void* gl = nullptr;
    const void* dot = nullptr;
    std::uint32_t flags = 0;
    lidx w = 0;
    int nocomm = 0;
    unsigned char sc[5][16] = {};
    bool operator==(const StepKey& o) const { return std::memcmp(this, &o, sizeof(StepKey)) == 0; }
};

StepKey make_key(const DenseMat& y, const DenseMat& x, const SpmvOptions& o, const DenseMat* z, bool nocomm) {
    StepKey k;
    std::memset(&k, 0, sizeof(k));  // padding bytes take part in the comparison
    k.y = y.data;
    k.x = x.data;
    k.z = z ? z->data : nullptr;
    k.gl = o.gamma_list;
    k.dot = o.dot;
    k.flags = o.flags;
    k.w = x.ncols;
    k.nocomm = nocomm ? 1 : 0;
    std::memcpy(k.sc[0], o.alpha, 16);
    std::memcpy(k.sc[1], o.beta, 16);
    std::memcpy(k.sc[2], o.gamma, 16);
    std::memcpy(k.sc[3], o.delta, 16);
    std::memcpy(k.sc[4], o.eta, 16);
    return k;
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

}  // namespace

struct RankContext {
    RankPart part;
    RankScratch sc;
    Transport transport = Transport::none;
    ncclComm_t comm = nullptr;
    lidx C = 1, sigma = 1;
    bool sends_ready = false;
    std::uint64_t bytes = 0, msgs = 0;
    DeviceBuffer dots_all;       // nranks x 3w partials
    DeviceBuffer sweep_scratch;  // the sweeps' scratch (graph-stable)
    lidx buf_width = 0;
    // ipc transport
    int ipc_max_w = 0;
    DeviceBuffer ipc_send, ipc_dots, ipc_flags;
    std::vector<gidx> seg_row;  // per destination rank: first row of its slot (-1: none)
    struct Peer {
        unsigned char* send = nullptr;
        unsigned char* dots = nullptr;
        std::uint32_t* flags = nullptr;
        gidx seg_for_me = -1;
    };
    std::vector<Peer> peers;
    // CUDA graphs of whole steps, keyed by StepKey (captured on the second use)
    struct Graph {
        StepKey key;
        cudaGraphExec_t exec = nullptr;
    };
    std::vector<Graph> graphs;
    bool graphs_on = env_int("SELLKIT_GRAPHS", 1) != 0;
    bool graphs_broken = false;
    int reserve_sms = env_int("SELLKIT_COMM_RESERVE_SMS", 0);
    cudaStream_t cap = nullptr;
    cudaEvent_t cev_x = nullptr, cev_halo = nullptr;  // fork/join events of captured steps
    ~RankContext();
    void drop_graphs() {
        for (auto& g : graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        graphs.clear();
    }
};

RankContext::~RankContext() {
    DeviceGuard g(part.device);
    cudaDeviceSynchronize();
    drop_graphs();
    for (auto& p : peers) {
        if (p.send) cudaIpcCloseMemHandle(p.send);
        if (p.dots) cudaIpcCloseMemHandle(p.dots);
        if (p.flags) cudaIpcCloseMemHandle(p.flags);
    }
    if (comm) ncclCommDestroy(comm);
    if (cap) cudaStreamDestroy(cap);
    if (cev_x) cudaEventDestroy(cev_x);
    if (cev_halo) cudaEventDestroy(cev_halo);
    cudaGetLastError();
}

RankContext* rankctx_create(const Crs& rows, const std::vector<gidx>& row_offset, int rank, lidx C, lidx sigma) {
    SK_REQUIRE(row_offset.size() >= 2, errc::invalid_arg, "partition needs at least one rank");
    std::vector<gidx> rowptr, col;
    std::vector<unsigned char> val;
    {
        DeviceGuard g(rows.device);
        crs_download(rows, rowptr, col, val);
    }
    SK_REQUIRE(rows.ncols == row_offset.back(), errc::shape_mismatch, "row block must carry global columns");
    auto* rc = new RankContext();
    try {
        rc->C = C;
        rc->sigma = sigma;
        rc->part.device = rows.device;
        rc->part.plan = plan_rank(rows.dt, rowptr.data(), col.data(), val.data(), lidx(rows.nrows), row_offset, rank);
        rank_build_device(rc->part, C, sigma);
    } catch (...) {
        delete rc;
        throw;
    }
    return rc;
}

RankPlan& rankctx_plan(RankContext* rc) { return rc->part.plan; }

void rankctx_finalize_sends(RankContext* rc) {
    build_send_rows(rc->part);
    rc->sends_ready = true;
}

void nccl_unique_id(void* out128) {
    ncclUniqueId id;
    NCK(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
}

void rankctx_connect(RankContext* rc, const void* nccl_id) {
    SK_REQUIRE(rc->transport == Transport::none, errc::state, "rank context is already connected");
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    DeviceGuard g(rc->part.device);
    NCK(ncclCommInitRank(&rc->comm, rc->part.plan.nranks, id, rc->part.plan.rank));
    rc->transport = Transport::nccl;
}

std::size_t rankctx_ipc_blob_bytes(RankContext* rc) { return ipc_blob_bytes(rc->part.plan.nranks); }

// allocate and export this rank's IPC buffers (send slots sized for max_w columns)
void rankctx_ipc_export(RankContext* rc, int max_w, void* blob) {
    RankPart& part = rc->part;
    const RankPlan& p = part.plan;
    SK_REQUIRE(rc->transport == Transport::none, errc::state, "rank context is already connected");
    SK_REQUIRE(max_w >= 1, errc::invalid_arg, "max_width must be positive");
    DeviceGuard g(part.device);
    const std::size_t es = value_bytes(p.dt);
    const int n = p.nranks;
    if (!rc->ipc_flags.get() || rc->ipc_max_w != max_w) {
        rc->seg_row.assign(std::size_t(n), -1);
        gidx rows = 0;
        for (std::size_t s = 0; s < p.send_to.size(); ++s) {
            rc->seg_row[p.send_to[s]] = rows;
            rows += gidx(p.send_local_rows[s].size());
        }
        rc->ipc_max_w = max_w;
        rc->ipc_send = DeviceBuffer(std::max<std::size_t>(std::size_t(rows) * max_w * es, 256), part.device);
        rc->ipc_dots = DeviceBuffer(std::max<std::size_t>(3 * std::size_t(max_w) * es, 256), part.device);
        rc->ipc_flags = DeviceBuffer(4 * std::size_t(n) * sizeof(std::uint32_t), part.device);
        // full = 0, free = 1, dots full = 0, dots free = 1
        std::vector<std::uint32_t> init(4 * std::size_t(n), 0u);
        for (int d = 0; d < n; ++d) init[n + d] = init[3 * n + d] = 1u;
        CK(cudaMemcpy(rc->ipc_flags.get(), init.data(), init.size() * sizeof(std::uint32_t), cudaMemcpyHostToDevice));
    }
    IpcBlobHead h;
    std::memset(&h, 0, sizeof(h));
    std::memcpy(h.magic, kIpcMagic, sizeof(kIpcMagic));
    h.rank = p.rank;
    h.nranks = n;
    h.max_w = max_w;
    h.es = int(es);
    h.device = part.device;
    CK(cudaIpcGetMemHandle(&h.send, rc->ipc_send.get()));
    CK(cudaIpcGetMemHandle(&h.dots, rc->ipc_dots.get()));
    CK(cudaIpcGetMemHandle(&h.flags, rc->ipc_flags.get()));
    std::memcpy(blob, &h, sizeof(h));
    std::memcpy(static_cast<unsigned char*>(blob) + sizeof(h), rc->seg_row.data(), std::size_t(n) * sizeof(gidx));
}

// open every peer's buffers (blobs of all ranks, in rank order)
void rankctx_ipc_connect(RankContext* rc, const void* blobs, std::size_t blob_bytes) {
    RankPart& part = rc->part;
    const RankPlan& p = part.plan;
    const int n = p.nranks;
    SK_REQUIRE(rc->transport == Transport::none, errc::state, "rank context is already connected");
    SK_REQUIRE(rc->ipc_flags.get() != nullptr, errc::state, "export the IPC buffers first");
    SK_REQUIRE(blob_bytes == ipc_blob_bytes(n), errc::invalid_arg, "IPC blob size mismatch");
    DeviceGuard g(part.device);
    rc->peers.assign(std::size_t(n), RankContext::Peer{});
    const auto* b = static_cast<const unsigned char*>(blobs);
    for (int r = 0; r < n; ++r) {
        IpcBlobHead h;
        std::memcpy(&h, b + std::size_t(r) * blob_bytes, sizeof(h));
        SK_REQUIRE(std::memcmp(h.magic, kIpcMagic, sizeof(kIpcMagic)) == 0 && h.rank == r && h.nranks == n,
                   errc::transport, "malformed IPC blob");
        SK_REQUIRE(h.max_w == rc->ipc_max_w && h.es == int(value_bytes(p.dt)), errc::transport,
                   "ranks disagree on the IPC slot geometry");
        if (r == p.rank) continue;
        std::vector<gidx> seg(static_cast<std::size_t>(n));
        std::memcpy(seg.data(), b + std::size_t(r) * blob_bytes + sizeof(h), std::size_t(n) * sizeof(gidx));
        auto& peer = rc->peers[r];
        void* ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, h.send, cudaIpcMemLazyEnablePeerAccess));
        peer.send = static_cast<unsigned char*>(ptr);
        CK(cudaIpcOpenMemHandle(&ptr, h.dots, cudaIpcMemLazyEnablePeerAccess));
        peer.dots = static_cast<unsigned char*>(ptr);
        CK(cudaIpcOpenMemHandle(&ptr, h.flags, cudaIpcMemLazyEnablePeerAccess));
        peer.flags = static_cast<std::uint32_t*>(ptr);
        peer.seg_for_me = seg[p.rank];
    }
    for (int owner : p.recv_owner)
        SK_REQUIRE(rc->peers[owner].seg_for_me >= 0, errc::transport, "an owner has no send slot for this rank");
    rc->transport = Transport::ipc;
}

namespace {

// width-dependent buffers; reallocation invalidates every captured graph
void ensure_rank_buffers(RankContext* rc, lidx w) {
    RankPart& part = rc->part;
    const RankPlan& p = part.plan;
    const std::size_t es = value_bytes(p.dt);
    ensure_scratch(rc->sc, part, w);
    if (rc->buf_width == w) return;
    auto& rt = runtime(part.device);
    CK(cudaDeviceSynchronize());
    rc->drop_graphs();
    rc->dots_all = DeviceBuffer(std::max<std::size_t>(std::size_t(p.nranks) * 3 * w * es, 256), part.device);
    const std::size_t ss = spmv_scratch_bytes(p.dt, w, rt.num_sms);
    rc->sweep_scratch = DeviceBuffer(ss, part.device);
    rc->buf_width = w;
}

void ipc_exchange(RankContext* rc, const DenseMat& x, lidx w) {
    RankPart& part = rc->part;
    const RankPlan& p = part.plan;
    const int n = p.nranks, me = p.rank;
    const std::size_t es = value_bytes(p.dt);
    const std::size_t slot_row = std::size_t(rc->ipc_max_w) * es;  // slot pitch per row
    std::uint32_t* flags = rc->ipc_flags.as<std::uint32_t>();
    cudaStream_t cs = part.comm;
    auto* mine = static_cast<unsigned char*>(rc->ipc_send.get());
    // 1. my slots are free once each receiver pulled the previous step's data
    for (int d : p.send_to) {
        flag_wait(cs, flags + n + d, 1u);
        flag_set(cs, flags + n + d, 0u);
    }
    // 2. pack each send list into its slot, 3. raise the receiver's full flag
    for (std::size_t s = 0; s < p.send_to.size(); ++s) {
        const int to = p.send_to[s];
        const lidx cnt = lidx(p.send_local_rows[s].size());
        launch_pack(p.dt, x, part.send_rows[s].as<lidx>(), cnt, w, mine + std::size_t(rc->seg_row[to]) * slot_row, cs);
        rc->bytes += std::uint64_t(cnt) * w * es;
        rc->msgs += 1;
    }
    for (int d : p.send_to) flag_set(cs, rc->peers[d].flags + me, 1u);
    // 4. pull every owner's slot into the halo block (copy engine), release the slot
    for (std::size_t q = 0; q < p.recv_owner.size(); ++q) {
        const int s = p.recv_owner[q];
        const auto& peer = rc->peers[s];
        flag_wait(cs, flags + s, 1u);
        CK(cudaMemcpyAsync(static_cast<unsigned char*>(rc->sc.halo.get()) + std::size_t(p.recv_offset[q]) * w * es,
                           peer.send + std::size_t(peer.seg_for_me) * slot_row, std::size_t(p.recv_count[q]) * w * es,
                           cudaMemcpyDeviceToDevice, cs));
        flag_set(cs, flags + s, 0u);
        flag_set(cs, peer.flags + n + me, 1u);
    }
}

void nccl_exchange(RankContext* rc, const DenseMat& x, lidx w) {
    RankPart& part = rc->part;
    const RankPlan& p = part.plan;
    const std::size_t es = value_bytes(p.dt);
    std::size_t mult = 1;
    const ncclDataType_t nt = nccl_type(p.dt, mult);
    std::size_t off = 0;
    std::vector<std::size_t> soff;
    for (std::size_t s = 0; s < p.send_to.size(); ++s) {
        const lidx cnt = lidx(p.send_local_rows[s].size());
        soff.push_back(off);
        launch_pack(p.dt, x, part.send_rows[s].as<lidx>(), cnt, w,
                    static_cast<unsigned char*>(rc->sc.sendbuf.get()) + off * es, part.comm);
        off += std::size_t(cnt) * w;
    }
    NCK(ncclGroupStart());
    for (std::size_t q = 0; q < p.recv_owner.size(); ++q)
        NCK(ncclRecv(static_cast<unsigned char*>(rc->sc.halo.get()) + std::size_t(p.recv_offset[q]) * w * es,
                     std::size_t(p.recv_count[q]) * w * mult, nt, p.recv_owner[q], rc->comm, part.comm));
    for (std::size_t s = 0; s < p.send_to.size(); ++s) {
        const std::size_t cnt = p.send_local_rows[s].size();
        NCK(ncclSend(static_cast<unsigned char*>(rc->sc.sendbuf.get()) + soff[s] * es, cnt * w * mult, nt,
                     p.send_to[s], rc->comm, part.comm));
        rc->bytes += cnt * w * es;
        rc->msgs += 1;
    }
    NCK(ncclGroupEnd());
}

// per-rank dot partials (sc.dots) -> every rank's dots_all in rank order -> rank-ordered sum
void combine_dots(RankContext* rc, lidx w, cudaStream_t st) {
    RankPart& part = rc->part;
    const RankPlan& p = part.plan;
    const int n = p.nranks, me = p.rank;
    const std::size_t es = value_bytes(p.dt);
    const std::size_t db = 3 * std::size_t(w) * es;
    auto* all = static_cast<unsigned char*>(rc->dots_all.get());
    if (rc->transport == Transport::nccl) {
        std::size_t mult = 1;
        const ncclDataType_t nt = nccl_type(p.dt, mult);
        NCK(ncclAllGather(rc->sc.dots.get(), all, 3 * std::size_t(w) * mult, nt, rc->comm, st));
    } else {
        std::uint32_t* flags = rc->ipc_flags.as<std::uint32_t>();
        for (int d = 0; d < n; ++d)
            if (d != me) {
                flag_wait(st, flags + 3 * n + d, 1u);
                flag_set(st, flags + 3 * n + d, 0u);
            }
        CK(cudaMemcpyAsync(rc->ipc_dots.get(), rc->sc.dots.get(), db, cudaMemcpyDeviceToDevice, st));
        for (int d = 0; d < n; ++d)
            if (d != me) flag_set(st, rc->peers[d].flags + 2 * n + me, 1u);
        for (int s = 0; s < n; ++s) {
            if (s == me) {
                CK(cudaMemcpyAsync(all + std::size_t(s) * db, rc->sc.dots.get(), db, cudaMemcpyDeviceToDevice, st));
                continue;
            }
            flag_wait(st, flags + 2 * n + s, 1u);
            CK(cudaMemcpyAsync(all + std::size_t(s) * db, rc->peers[s].dots, db, cudaMemcpyDeviceToDevice, st));
            flag_set(st, flags + 2 * n + s, 0u);
            flag_set(st, rc->peers[s].flags + 3 * n + me, 1u);
        }
    }
    visit_dt(p.dt, [&]<class T>() {
        rank_sum_kernel<T><<<(3 * w + 127) / 128, 128, 0, st>>>(rc->dots_all.as<T>(), n, 3 * w, rc->sc.dots.as<T>());
        return 0;
    });
    CK(cudaGetLastError());
    rc->msgs += 2 * std::uint64_t(n - 1);
    rc->bytes += 2 * std::uint64_t(n - 1) * db;
}

// enqueue one distributed step on `st` (+ the comm stream); `capturing`: inside a
// graph capture (consecutive graph launches are ordered by the stream instead of ev_done)
void rank_step(RankContext* rc, DenseMat& y, const DenseMat& x, const SpmvOptions& o, DenseMat* z, bool nocomm,
               cudaStream_t st, bool capturing) {
    RankPart& part = rc->part;
    const RankPlan& p = part.plan;
    const lidx w = x.ncols;
    const std::size_t es = value_bytes(p.dt);
    const std::uint32_t dots = o.flags & kFlagDots;
    const bool exchange = !nocomm && p.nranks > 1 && (!p.send_to.empty() || !p.recv_owner.empty());
    // events recorded inside a capture cannot be waited on outside it: captures use their own
    cudaEvent_t ev_x = capturing ? rc->cev_x : part.ev_x;
    cudaEvent_t ev_halo = capturing ? rc->cev_halo : part.ev_halo;
    if (exchange) {
        NvtxRange r("sellkit halo exchange (enqueue)");
        CK(cudaEventRecord(ev_x, st));
        CK(cudaStreamWaitEvent(part.comm, ev_x, 0));
        if (!capturing) CK(cudaStreamWaitEvent(part.comm, part.ev_done, 0));  // previous remote sweep used the halo
        if (rc->transport == Transport::ipc) ipc_exchange(rc, x, w);
        else nccl_exchange(rc, x, w);
        CK(cudaEventRecord(ev_halo, part.comm));
    }
    SpmvHooks extra;
    extra.scratch = rc->sweep_scratch.get();
    extra.scratch_size = rc->sweep_scratch.bytes();
    extra.reserve_sms = exchange && !p.send_to.empty() ? rc->reserve_sms : 0;
    {
        NvtxRange r("sellkit local + remote sweeps (enqueue)");
        rank_sweeps(part, rc->sc, y, x, o, z, !exchange && (nocomm || p.recv_owner.empty()), st,
                    [&] { CK(cudaStreamWaitEvent(st, ev_halo, 0)); }, extra);
    }
    if (exchange) CK(cudaStreamWaitEvent(st, ev_halo, 0));  // join the comm branch
    // (graph launches are ordered by the stream; only eager steps publish ev_done)
    if (!capturing) CK(cudaEventRecord(part.ev_done, st));
    if (dots) {
        NvtxRange r("sellkit dots (enqueue)");
        if (p.nranks > 1 && rc->transport != Transport::none) combine_dots(rc, w, st);
        for (int s = 0; s < 3; ++s)
            if (o.flags & (kFlagDotYY << s))
                CK(cudaMemcpyAsync(static_cast<unsigned char*>(o.dot) + std::size_t(s) * w * es,
                                   static_cast<unsigned char*>(rc->sc.dots.get()) + std::size_t(s) * w * es, w * es,
                                   cudaMemcpyDefault, st));
    }
}

void check_transport(RankContext* rc) {
    if (rc->transport != Transport::nccl || !rc->comm) return;
    ncclResult_t as = ncclSuccess;
    NCK(ncclCommGetAsyncError(rc->comm, &as));
    if (as != ncclSuccess && as != ncclInProgress)
        fail(errc::transport, std::string("NCCL asynchronous error: ") + ncclGetErrorString(as));
}

// a step may be captured when every host-side input is baked into device memory
bool graphable(const SpmvOptions& o) {
    if ((o.flags & kFlagVshift) && pointer_kind(o.gamma_list, nullptr) != MemKind::device) return false;
    if ((o.flags & kFlagDots) && pointer_kind(o.dot, nullptr) != MemKind::device) return false;
    return true;
}

bool capture_step(RankContext* rc, RankContext::Graph& g, DenseMat& y, const DenseMat& x, const SpmvOptions& o,
                  DenseMat* z, bool nocomm) {
    if (!rc->cap) {
        CK(cudaStreamCreateWithFlags(&rc->cap, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&rc->cev_x, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&rc->cev_halo, cudaEventDisableTiming));
    }
    CK(cudaStreamBeginCapture(rc->cap, cudaStreamCaptureModeThreadLocal));
    std::string why;
    const std::uint64_t bytes0 = rc->bytes, msgs0 = rc->msgs;  // capturing moves no data
    try {
        rank_step(rc, y, x, o, z, nocomm, rc->cap, true);
    } catch (const std::exception& e) {
        why = e.what();
    }
    rc->bytes = bytes0;
    rc->msgs = msgs0;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(rc->cap, &graph);
    if (why.empty() && e != cudaSuccess) why = cudaGetErrorString(e);
    cudaGraphExec_t exec = nullptr;
    if (why.empty()) {
        e = cudaGraphInstantiate(&exec, graph, 0);
        if (e != cudaSuccess) why = cudaGetErrorString(e);
    }
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    if (!why.empty()) {
        if (std::getenv("SELLKIT_VERBOSE"))
            std::fprintf(stderr, "[sellkit] rank step not capturable (%s); running eagerly\n", why.c_str());
        rc->graphs_broken = true;
        return false;
    }
    g.exec = exec;
    return true;
}

}  // namespace

void rankctx_spmv(RankContext* rc, DenseMat& y, const DenseMat& x, const SpmvOptions& o, DenseMat* z, bool nocomm) {
    RankPart& part = rc->part;
    const RankPlan& p = part.plan;
    SK_REQUIRE(rc->sends_ready || nocomm || p.nranks == 1, errc::state, "send lists were not finalised");
    SK_REQUIRE(rc->transport != Transport::none || nocomm || p.nranks == 1, errc::state,
               "rank context is not connected");
    SK_REQUIRE(x.nrows == p.nrows && y.nrows == p.nrows && x.ncols == y.ncols, errc::shape_mismatch,
               "x and y must hold this rank's rows");
    SK_REQUIRE(x.mem == MemKind::device && y.mem == MemKind::device, errc::unsupported,
               "rank vectors must be device-resident");
    SK_REQUIRE(y.data != x.data, errc::invalid_arg, "y must not alias x");
    const bool chain = (o.flags & kFlagChain) != 0;
    SK_REQUIRE(!chain || z != nullptr, errc::invalid_arg, "CHAIN_AXPBY requires z");
    SK_REQUIRE(!chain || (z->mem == MemKind::device && z->same_shape(y)), errc::shape_mismatch,
               "z must be a device block of y's shape");
    const std::uint32_t dots = o.flags & kFlagDots;
    SK_REQUIRE(!dots || o.dot != nullptr, errc::invalid_arg, "dot flags require a dot buffer");
    SK_REQUIRE((o.flags & ~kFlagAll) == 0, errc::invalid_arg, "unknown spmv flag");
    SK_REQUIRE(!((o.flags & kFlagShift) && (o.flags & kFlagVshift)), errc::invalid_arg,
               "SHIFT and VSHIFT are mutually exclusive");
    SK_REQUIRE(!(o.flags & kFlagVshift) || o.gamma_list != nullptr, errc::invalid_arg, "VSHIFT requires a gamma list");
    const lidx w = x.ncols;
    SK_REQUIRE(rc->transport != Transport::ipc || w <= rc->ipc_max_w, errc::capacity,
               "block width exceeds the IPC slots exported at connect time");
    DeviceGuard g(part.device);
    auto& rt = runtime(part.device);
    ensure_rank_buffers(rc, w);
    bool done = false;
    if (rc->graphs_on && !rc->graphs_broken && graphable(o)) {
        const StepKey key = make_key(y, x, o, z, nocomm);
        RankContext::Graph* hit = nullptr;
        for (auto& gr : rc->graphs)
            if (gr.key == key) hit = &gr;
        if (hit && !hit->exec) capture_step(rc, *hit, y, x, o, z, nocomm);  // second use: capture
        if (hit && hit->exec) {
            CK(cudaGraphLaunch(hit->exec, rt.stream));
            done = true;
            // the transport counters advance as if the step ran eagerly
            const bool exchange = !nocomm && p.nranks > 1 && (!p.send_to.empty() || !p.recv_owner.empty());
            if (exchange) {
                for (auto& rows : p.send_local_rows) rc->bytes += std::uint64_t(rows.size()) * w * value_bytes(p.dt);
                rc->msgs += p.send_to.size();
            }
            if (dots && p.nranks > 1 && rc->transport != Transport::none) {
                rc->msgs += 2 * std::uint64_t(p.nranks - 1);
                rc->bytes += 2 * std::uint64_t(p.nranks - 1) * 3 * w * value_bytes(p.dt);
            }
        } else if (!hit) {
            if (rc->graphs.size() >= 8) {
                if (rc->graphs.front().exec) cudaGraphExecDestroy(rc->graphs.front().exec);
                rc->graphs.erase(rc->graphs.begin());
            }
            rc->graphs.push_back(RankContext::Graph{key, nullptr});
        }
    }
    if (!done) rank_step(rc, y, x, o, z, nocomm, rt.stream, false);
    check_transport(rc);
    finish(rt);
}

void rankctx_set_options(RankContext* rc, int graphs, int reserve_sms) {
    if (graphs >= 0) {
        rc->graphs_on = graphs != 0;
        if (!rc->graphs_on) {
            DeviceGuard g(rc->part.device);
            CK(cudaDeviceSynchronize());
            rc->drop_graphs();
        }
        rc->graphs_broken = false;
    }
    if (reserve_sms >= 0) {
        rc->reserve_sms = reserve_sms;
        DeviceGuard g(rc->part.device);
        CK(cudaDeviceSynchronize());
        rc->drop_graphs();
    }
}

int rankctx_transport(RankContext* rc) { return int(rc->transport); }

void rankctx_stats(RankContext* rc, std::uint64_t* bytes, std::uint64_t* msgs, lidx* n_halo, std::uint64_t* halo_rows,
                   gidx* local_nnz, gidx* remote_nnz) {
    if (bytes) *bytes = rc->bytes;
    if (msgs) *msgs = rc->msgs;
    if (n_halo) *n_halo = lidx(rc->part.plan.halo_cols.size());
    if (halo_rows) *halo_rows = rc->part.remote ? std::uint64_t(rc->part.remote->nrows) : 0;
    if (local_nnz) *local_nnz = rc->part.local->nnz;
    if (remote_nnz) *remote_nnz = rc->part.remote ? rc->part.remote->nnz : 0;
}

const SellMat* rankctx_local(RankContext* rc) { return rc->part.local.get(); }

void rankctx_destroy(RankContext* rc) { delete rc; }

}  // namespace skb

// ======================================================================= C ABI

namespace sk = skb;

extern "C" {

sellkit_error sellkit_partition_compute(sellkit_gidx n, const sellkit_lidx* rowlens, const double* weights, int nranks,
                                        sellkit_weight_mode mode, sellkit_gidx* offsets_out) {
    return sk::guarded([&] {
        sk::require(weights && offsets_out, "null argument");
        std::vector<double> w(weights, weights + std::max(nranks, 0));
        const auto off = sk::compute_partition(n, rowlens, w, mode == SELLKIT_BY_NNZ);
        std::copy(off.begin(), off.end(), offsets_out);
    });
}

sellkit_error sellkit_ctx_create(const sellkit_crs* a, const double* weights, int nranks, sellkit_weight_mode mode,
                                 int chunk_height, int sigma, int record_transport, sellkit_ctx** out) {
    return sk::guarded([&] {
        sk::require(a && out && nranks >= 1, "null argument");
        std::vector<double> w = weights ? std::vector<double>(weights, weights + nranks) : std::vector<double>(nranks, 1.0);
        *out = new sellkit_ctx{sk::dist_context_create(*a->p, w, mode == SELLKIT_BY_NNZ, chunk_height, sigma,
                                                       record_transport != 0)};
    });
}

sellkit_error sellkit_ctx_rank_range(const sellkit_ctx* ctx, int rank, sellkit_gidx* first, sellkit_gidx* count) {
    return sk::guarded([&] {
        sk::require(ctx != nullptr, "null handle");
        const auto& c = *ctx->p;
        sk::require(rank >= 0 && rank < int(c.ranks.size()), "rank out of range");
        if (first) *first = c.row_offset[rank];
        if (count) *count = c.row_offset[rank + 1] - c.row_offset[rank];
    });
}

sellkit_error sellkit_ctx_halo_size(const sellkit_ctx* ctx, int rank, sellkit_lidx* n_halo) {
    return sk::guarded([&] {
        sk::require(ctx && n_halo, "null argument");
        const auto& c = *ctx->p;
        sk::require(rank >= 0 && rank < int(c.ranks.size()), "rank out of range");
        *n_halo = sk::lidx(c.ranks[rank]->plan.halo_cols.size());
    });
}

sellkit_error sellkit_ctx_comm_stats(const sellkit_ctx* ctx, uint64_t* total_bytes, uint64_t* total_messages) {
    return sk::guarded([&] {
        sk::require(ctx != nullptr, "null handle");
        SK_REQUIRE(ctx->p->record, sk::errc::state, "context was created without transport recording");
        if (total_bytes) *total_bytes = ctx->p->bytes;
        if (total_messages) *total_messages = ctx->p->msgs;
    });
}

sellkit_error sellkit_ctx_reset_comm_stats(sellkit_ctx* ctx) {
    return sk::guarded([&] {
        sk::require(ctx != nullptr, "null handle");
        SK_REQUIRE(ctx->p->record, sk::errc::state, "context was created without transport recording");
        ctx->p->bytes = ctx->p->msgs = 0;
    });
}

void sellkit_ctx_destroy(sellkit_ctx* ctx) { delete ctx; }

sellkit_error sellkit_ext_ctx_set_trace(sellkit_ctx* ctx, int on) {
    return sk::guarded([&] {
        sk::require(ctx != nullptr, "null handle");
        ctx->p->trace = on != 0;
    });
}

sellkit_error sellkit_ext_ctx_timeline(const sellkit_ctx* ctx, double* out, int* nvalues) {
    return sk::guarded([&] {
        sk::require(ctx && nvalues, "null argument");
        const auto& t = ctx->p->timeline;
        if (out) std::copy(t.begin(), t.begin() + std::min<std::size_t>(t.size(), std::size_t(*nvalues)), out);
        *nvalues = int(t.size());
    });
}

sellkit_error sellkit_dvec_create(const sellkit_ctx* ctx, sellkit_lidx width, sellkit_order order, sellkit_dvec** out) {
    return sk::guarded([&] {
        sk::require(ctx && out, "null argument");
        *out = new sellkit_dvec{sk::dist_vec_create(*ctx->p, width, sk::order_from(order))};
    });
}

sellkit_error sellkit_dvec_scatter(const sellkit_ctx* ctx, const sellkit_densemat* global, sellkit_dvec* v) {
    return sk::guarded([&] {
        sk::require(ctx && global && v, "null argument");
        sk::dist_scatter(*ctx->p, global->m, *v->p);
    });
}

sellkit_error sellkit_dvec_gather(const sellkit_ctx* ctx, const sellkit_dvec* v, sellkit_densemat* out) {
    return sk::guarded([&] {
        sk::require(ctx && v && out, "null argument");
        sk::dist_gather(*ctx->p, *v->p, out->m);
    });
}

void sellkit_dvec_destroy(sellkit_dvec* v) { delete v; }

sellkit_error sellkit_dist_spmv(sellkit_dvec* y, sellkit_ctx* ctx, const sellkit_dvec* x, const sellkit_spmv_opts* opts,
                                sellkit_dist_mode mode, sellkit_dvec* z, int pus_per_rank) {
    (void)pus_per_rank;
    return sk::guarded([&] {
        sk::require(y && ctx && x, "null argument");
        sk::require(!opts || opts->z == nullptr, "distributed chain target must be a sellkit_dvec");
        sk::SpmvOptions o;
        sk::options_from_c(ctx->p->dt, opts, o);
        sk::dist_spmv(*y->p, *ctx->p, *x->p, o, int(mode), z ? z->p.get() : nullptr, false);
    });
}

sellkit_error sellkit_spmv_nocomm(sellkit_dvec* y, sellkit_ctx* ctx, const sellkit_dvec* x, const sellkit_spmv_opts* opts,
                                  sellkit_dvec* z) {
    return sk::guarded([&] {
        sk::require(y && ctx && x, "null argument");
        sk::require(!opts || opts->z == nullptr, "distributed chain target must be a sellkit_dvec");
        sk::SpmvOptions o;
        sk::options_from_c(ctx->p->dt, opts, o);
        sk::dist_spmv(*y->p, *ctx->p, *x->p, o, 0, z ? z->p.get() : nullptr, true);
    });
}

/* ---------------------------------------------------- multi-process (ext) */

sellkit_error sellkit_ext_nccl_unique_id(void* id128) {
    return sk::guarded([&] {
        sk::require(id128 != nullptr, "null output");
        sk::nccl_unique_id(id128);
    });
}

sellkit_error sellkit_ext_rankctx_create(const sellkit_crs* rows, const sellkit_gidx* row_offsets, int nranks, int rank,
                                         int chunk_height, int sigma, sellkit_rankctx** out) {
    return sk::guarded([&] {
        sk::require(rows && row_offsets && out && nranks >= 1, "null argument");
        std::vector<sk::gidx> off(row_offsets, row_offsets + nranks + 1);
        *out = new sellkit_rankctx{sk::rankctx_create(*rows->p, off, rank, chunk_height, sigma)};
    });
}

sellkit_error sellkit_ext_rankctx_recv_count(const sellkit_rankctx* rc, int* nowners) {
    return sk::guarded([&] {
        sk::require(rc && nowners, "null argument");
        *nowners = int(sk::rankctx_plan(rc->p).recv_owner.size());
    });
}

sellkit_error sellkit_ext_rankctx_recv(const sellkit_rankctx* rc, int q, int* owner, sellkit_lidx* count,
                                       sellkit_gidx* cols) {
    return sk::guarded([&] {
        sk::require(rc != nullptr, "null handle");
        const auto& p = sk::rankctx_plan(rc->p);
        sk::require(q >= 0 && q < int(p.recv_owner.size()), "receive index out of range");
        if (owner) *owner = p.recv_owner[q];
        if (count) *count = p.recv_count[q];
        if (cols) std::copy_n(p.halo_cols.begin() + p.recv_offset[q], p.recv_count[q], cols);
    });
}

sellkit_error sellkit_ext_rankctx_set_sends(sellkit_rankctx* rc, int to, const sellkit_gidx* cols, sellkit_lidx count) {
    return sk::guarded([&] {
        sk::require(rc && (cols || count == 0), "null argument");
        sk::plan_set_sends(sk::rankctx_plan(rc->p), to, cols, count);
    });
}

sellkit_error sellkit_ext_rankctx_send(const sellkit_rankctx* rc, int s, int* to, sellkit_lidx* count,
                                       sellkit_lidx* local_rows) {
    return sk::guarded([&] {
        sk::require(rc != nullptr, "null handle");
        const auto& p = sk::rankctx_plan(rc->p);
        sk::require(s >= 0 && s < int(p.send_to.size()), "send index out of range");
        if (to) *to = p.send_to[s];
        if (count) *count = sk::lidx(p.send_local_rows[s].size());
        if (local_rows) std::copy(p.send_local_rows[s].begin(), p.send_local_rows[s].end(), local_rows);
    });
}

sellkit_error sellkit_ext_rankctx_connect(sellkit_rankctx* rc, const void* id128) {
    return sk::guarded([&] {
        sk::require(rc && id128, "null argument");
        sk::rankctx_finalize_sends(rc->p);
        if (sk::rankctx_plan(rc->p).nranks > 1) sk::rankctx_connect(rc->p, id128);
    });
}

sellkit_error sellkit_ext_rankctx_ipc_export(sellkit_rankctx* rc, int max_width, void* blob, size_t* blob_bytes) {
    return sk::guarded([&] {
        sk::require(rc && blob_bytes, "null argument");
        const std::size_t need = sk::rankctx_ipc_blob_bytes(rc->p);
        if (!blob) {
            *blob_bytes = need;
            return;
        }
        SK_REQUIRE(*blob_bytes >= need, sk::errc::capacity, "IPC blob buffer too small");
        sk::rankctx_finalize_sends(rc->p);
        sk::rankctx_ipc_export(rc->p, max_width, blob);
        *blob_bytes = need;
    });
}

sellkit_error sellkit_ext_rankctx_ipc_connect(sellkit_rankctx* rc, const void* blobs, size_t blob_bytes) {
    return sk::guarded([&] {
        sk::require(rc && blobs, "null argument");
        if (sk::rankctx_plan(rc->p).nranks == 1) return;
        sk::rankctx_ipc_connect(rc->p, blobs, blob_bytes);
    });
}

sellkit_error sellkit_ext_rankctx_transport(const sellkit_rankctx* rc, int* transport) {
    return sk::guarded([&] {
        sk::require(rc && transport, "null argument");
        *transport = sk::rankctx_transport(rc->p);
    });
}

sellkit_error sellkit_ext_rankctx_set_options(sellkit_rankctx* rc, int graphs, int reserve_sms) {
    return sk::guarded([&] {
        sk::require(rc != nullptr, "null handle");
        sk::rankctx_set_options(rc->p, graphs, reserve_sms);
    });
}

sellkit_error sellkit_ext_rank_spmv(sellkit_densemat* y, sellkit_rankctx* rc, const sellkit_densemat* x,
                                    const sellkit_spmv_opts* opts, sellkit_densemat* z, int nocomm) {
    return sk::guarded([&] {
        sk::require(y && rc && x, "null argument");
        sk::require(!opts || opts->z == nullptr, "pass the chain target as z");
        sk::same_dt(y->m.dt, x->m.dt, "y and x");
        sk::SpmvOptions o;
        sk::options_from_c(y->m.dt, opts, o);
        sk::rankctx_spmv(rc->p, y->m, x->m, o, z ? &z->m : nullptr, nocomm != 0);
    });
}

sellkit_error sellkit_ext_rankctx_stats(const sellkit_rankctx* rc, uint64_t* bytes, uint64_t* msgs, sellkit_lidx* n_halo,
                                        uint64_t* boundary_rows, sellkit_gidx* local_nnz, sellkit_gidx* remote_nnz) {
    return sk::guarded([&] {
        sk::require(rc != nullptr, "null handle");
        sk::rankctx_stats(rc->p, bytes, msgs, n_halo, boundary_rows, local_nnz, remote_nnz);
    });
}

sellkit_error sellkit_ext_rankctx_row_perm(const sellkit_rankctx* rc, sellkit_lidx* row_perm) {
    return sk::guarded([&] {
        sk::require(rc && row_perm, "null argument");
        const sk::SellMat* m = sk::rankctx_local(rc->p);
        sk::DeviceGuard g(m->device);
        CK(cudaMemcpy(row_perm, m->row_perm.get(), std::size_t(m->nrows) * sizeof(sk::lidx), cudaMemcpyDeviceToHost));
    });
}

void sellkit_ext_rankctx_destroy(sellkit_rankctx* rc) {
    if (rc) sk::rankctx_destroy(rc->p);
    delete rc;
}

/* host-only planning (no GPU needed): the halo / send-list logic of one rank */
struct sellkit_rankplan {
    sk::RankPlan p;
};

sellkit_error sellkit_ext_rankplan_create(sellkit_datatype dt, const sellkit_gidx* rowptr, const sellkit_gidx* col,
                                          const void* val, sellkit_lidx nrows, const sellkit_gidx* row_offsets,
                                          int nranks, int rank, sellkit_rankplan** out) {
    return sk::guarded([&] {
        sk::require(rowptr && row_offsets && out, "null argument");
        std::vector<sk::gidx> off(row_offsets, row_offsets + nranks + 1);
        *out = new sellkit_rankplan{sk::plan_rank(sk::dt_from(dt), rowptr, col, val, nrows, off, rank)};
    });
}

sellkit_error sellkit_ext_rankplan_recv_count(const sellkit_rankplan* rp, int* nowners) {
    return sk::guarded([&] {
        sk::require(rp && nowners, "null argument");
        *nowners = int(rp->p.recv_owner.size());
    });
}

sellkit_error sellkit_ext_rankplan_recv(const sellkit_rankplan* rp, int q, int* owner, sellkit_lidx* count,
                                        sellkit_gidx* cols) {
    return sk::guarded([&] {
        sk::require(rp != nullptr, "null handle");
        const auto& p = rp->p;
        sk::require(q >= 0 && q < int(p.recv_owner.size()), "receive index out of range");
        if (owner) *owner = p.recv_owner[q];
        if (count) *count = p.recv_count[q];
        if (cols) std::copy_n(p.halo_cols.begin() + p.recv_offset[q], p.recv_count[q], cols);
    });
}

sellkit_error sellkit_ext_rankplan_set_sends(sellkit_rankplan* rp, int to, const sellkit_gidx* cols,
                                             sellkit_lidx count) {
    return sk::guarded([&] {
        sk::require(rp && (cols || count == 0), "null argument");
        sk::plan_set_sends(rp->p, to, cols, count);
    });
}

sellkit_error sellkit_ext_rankplan_send(const sellkit_rankplan* rp, int s, int* to, sellkit_lidx* count,
                                        sellkit_lidx* local_rows) {
    return sk::guarded([&] {
        sk::require(rp != nullptr, "null handle");
        const auto& p = rp->p;
        sk::require(s >= 0 && s < int(p.send_to.size()), "send index out of range");
        if (to) *to = p.send_to[s];
        if (count) *count = sk::lidx(p.send_local_rows[s].size());
        if (local_rows) std::copy(p.send_local_rows[s].begin(), p.send_local_rows[s].end(), local_rows);
    });
}

sellkit_error sellkit_ext_rankplan_nsends(const sellkit_rankplan* rp, int* nsends) {
    return sk::guarded([&] {
        sk::require(rp && nsends, "null argument");
        *nsends = int(rp->p.send_to.size());
    });
}

void sellkit_ext_rankplan_destroy(sellkit_rankplan* rp) { delete rp; }

}  // extern "C"
