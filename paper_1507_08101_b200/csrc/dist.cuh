// Row-distributed SpMMV with halo exchange (reference:
// /root/reference/proj/src/partition.hpp:45-600).
//
// A rank owns the contiguous row block [first_row, first_row + nrows) of a
// square matrix.  Its rows are split into
//   local  : columns inside the block, shifted and sigma-permuted (SELL, device);
//   remote : columns outside, compressed to [0, n_halo) in ascending global column
//            order (= ascending (owner, column)).  Only rows WITH remote entries are
//            stored (in stored order, row_map -> stored row), so the remote sweep
//            touches the boundary rows only (partition.hpp:471 sweeps all rows).
// One sigma order from the combined row lengths is imposed on both parts
// (partition.hpp:193-209), so every array -- row_offset, halo columns, receive
// counts, send lists, both layouts -- equals the reference's.
//
// dist_spmv, per rank, on the rank's device:
//   comm stream : pack x rows of each send list -> deliver to the destination's
//                 halo block (peer store / device copy in one process, NCCL send /
//                 recv across processes)
//   main stream : local sweep with every flag except the dots/chain of rows that
//                 have remote entries (defer mask), concurrently with the exchange;
//                 then, after the halo arrived, the remote sweep over boundary rows:
//                 y = alpha * A_rem * halo + y (partition.hpp:454-457 accum) fused
//                 with the deferred dots and chain of those rows.
// Per-rank dot partials are combined in rank order (partition.hpp:379-394).
#pragma once

#include <array>

#include "objects.cuh"
#include "spmv.cuh"

namespace skb {

// partition.hpp:45-94
std::vector<gidx> compute_partition(gidx n, const lidx* rowlens, const std::vector<double>& weights, bool by_nnz);

// Host-side plan of one rank (no device memory; usable without a GPU).
struct RankPlan {
    int rank = 0, nranks = 1;
    gidx first_row = 0;
    lidx nrows = 0;
    std::vector<gidx> row_offset;       // nranks + 1
    std::vector<gidx> halo_cols;        // ascending global columns
    std::vector<int> halo_owner;
    std::vector<int> recv_owner;        // ascending owners
    std::vector<lidx> recv_count;
    std::vector<lidx> recv_offset;      // first halo row of each owner's block
    // what other ranks need from us: destination rank, our LOCAL (unpermuted) row indices
    std::vector<int> send_to;
    std::vector<std::vector<lidx>> send_local_rows;
    // host CRS split (rows of this rank)
    std::vector<gidx> lrowptr, rrowptr;
    std::vector<gidx> lcol, rcol;
    std::vector<unsigned char> lval, rval;
    std::vector<lidx> lens;             // combined row lengths
    Datatype dt = Datatype::r64;
};

// partition.hpp:136-220 for the rows [first_row, first_row + nrows) given as host CRS
// with global columns.
RankPlan plan_rank(Datatype dt, const gidx* rowptr, const gidx* col, const void* val, lidx nrows,
                   const std::vector<gidx>& row_offset, int rank);
// register the global columns rank `to` requests from this rank (send list)
void plan_set_sends(RankPlan& p, int to, const gidx* cols, lidx count);

// Device part of one rank.
struct RankPart {
    RankPlan plan;
    int device = 0;
    std::unique_ptr<SellMat> local;
    std::unique_ptr<SellMat> remote;  // rows with remote entries only (stored order)
    DeviceBuffer row_map;             // int32 [remote rows] -> stored row
    DeviceBuffer defer_mask;          // uint32 [ceil(nrows/32)]
    std::vector<DeviceBuffer> send_rows;  // int32 stored rows per send list
    cudaStream_t comm = nullptr;
    cudaEvent_t ev_x = nullptr, ev_halo = nullptr, ev_done = nullptr;
    mutable std::vector<lidx> perm_host;  // original local row -> stored row (cached)
    RankPart() = default;
    RankPart(const RankPart&) = delete;
    ~RankPart();
};

void rank_build_device(RankPart& part, lidx C, lidx sigma);

// Per-width scratch of a rank: halo block, packed send buffers, dot partials.
struct RankScratch {
    lidx width = 0;
    DeviceBuffer halo;     // n_halo x width (row-major)
    DeviceBuffer sendbuf;  // sum(send counts) x width
    DeviceBuffer dots;     // 3 * width
};

constexpr int kTraceEvents = 5;  // exchange start/end, local start/end, remote end

struct DistContext {
    Datatype dt = Datatype::r64;
    gidx n = 0, nnz = 0;
    lidx C = 1, sigma = 1;
    std::vector<gidx> row_offset;
    std::vector<std::unique_ptr<RankPart>> ranks;
    std::vector<RankScratch> scratch;
    bool record = false;
    std::uint64_t bytes = 0, msgs = 0;
    DeviceBuffer dots_all;      // k x 3w dot partials on rank 0's device
    bool trace = false;         // record a per-rank timeline of each dist_spmv
    std::vector<cudaEvent_t> tev;
    std::vector<double> timeline;  // k x kTraceEvents, ms after the call's start (-1: none)
    ~DistContext() {
        for (auto e : tev) cudaEventDestroy(e);
    }
    DistContext() = default;
    DistContext(const DistContext&) = delete;
    int ndev = 1;
    std::vector<char> peer_ok;  // [ndev x ndev]: peer access enabled from i to j
    // may rank memory on `dst` be written by kernels running on `src`?
    bool direct(int src, int dst) const {
        return src == dst || (src < ndev && dst < ndev && peer_ok[std::size_t(src) * ndev + dst]);
    }
};

struct DistVec {
    lidx width = 0;
    Order order = Order::row_major;
    std::vector<DenseMat> parts;
};

std::unique_ptr<DistContext> dist_context_create(const Crs& a, const std::vector<double>& weights, bool by_nnz,
                                                 lidx C, lidx sigma, bool record);
std::unique_ptr<DistVec> dist_vec_create(const DistContext& ctx, lidx width, Order order);
void dist_scatter(const DistContext& ctx, const DenseMat& global, DistVec& v);
void dist_gather(const DistContext& ctx, const DistVec& v, DenseMat& out);
// modes: 0 NO_OVERLAP, 1 NAIVE_OVERLAP, 2 TASK_OVERLAP (1 and 2 identical on the GPU)
void dist_spmv(DistVec& y, DistContext& ctx, const DistVec& x, const SpmvOptions& opts, int mode, DistVec* z,
               bool nocomm);

// ------------------------------------------ one process per GPU (NCCL or IPC)
enum class Transport : int { none = 0, nccl = 1, ipc = 2 };
struct RankContext;
RankContext* rankctx_create(const Crs& rows, const std::vector<gidx>& row_offset, int rank, lidx C, lidx sigma);
RankPlan& rankctx_plan(RankContext* rc);
void rankctx_finalize_sends(RankContext* rc);
void rankctx_connect(RankContext* rc, const void* nccl_id);
void rankctx_spmv(RankContext* rc, DenseMat& y, const DenseMat& x, const SpmvOptions& o, DenseMat* z, bool nocomm);
void rankctx_stats(RankContext* rc, std::uint64_t* bytes, std::uint64_t* msgs, lidx* n_halo, std::uint64_t* halo_rows,
                   gidx* local_nnz, gidx* remote_nnz);
const SellMat* rankctx_local(RankContext* rc);
void rankctx_destroy(RankContext* rc);
void nccl_unique_id(void* out128);
std::size_t rankctx_ipc_blob_bytes(RankContext* rc);
void rankctx_ipc_export(RankContext* rc, int max_width, void* blob);
void rankctx_ipc_connect(RankContext* rc, const void* blobs, std::size_t blob_bytes);
void rankctx_set_options(RankContext* rc, int graphs, int reserve_sms);
int rankctx_transport(RankContext* rc);

}  // namespace skb
