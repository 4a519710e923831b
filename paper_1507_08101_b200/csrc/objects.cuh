// Library objects behind the opaque C handles: CRS input, SELL-C-sigma matrix
// and dense block vectors.  All bulk data lives in device memory (HBM) of the
// device that was current when the object was created.
#pragma once

#include "core.cuh"

namespace skb {

// ---------------------------------------------------------------- CRS input --
// Mirrors CrsData (/root/reference/proj/src/sellcs.hpp:36-65): int64 rowptr[n+1],
// int64 col[nnz] (global, strictly increasing per row), val[nnz].  Stored on the
// device so construction runs there.
struct Crs {
    Datatype dt = Datatype::r64;
    gidx nrows = 0, ncols = 0, nnz = 0;
    int device = 0;
    DeviceBuffer rowptr;  // int64
    DeviceBuffer col;     // int64
    DeviceBuffer val;     // T
};

// Upload + validate (sellcs.hpp:49-64 checks, done by a device kernel).
std::unique_ptr<Crs> crs_from_host(Datatype dt, gidx nrows, gidx ncols, const gidx* rowptr,
                                   const gidx* col, const void* val);
std::unique_ptr<Crs> crs_from_device(Datatype dt, gidx nrows, gidx ncols, const gidx* rowptr,
                                     const gidx* col, const void* val);
void crs_validate(const Crs& a);
// host copies (for to-host export / the row-callback path)
void crs_download(const Crs& a, std::vector<gidx>& rowptr, std::vector<gidx>& col,
                  std::vector<unsigned char>& val);

// --------------------------------------------------------------- SELL-C-sigma --
// Mirrors SellMatrix (sellcs.hpp:96-123).  Layout: slot(c, i, j) =
// chunk_offset[c] + j*C + i; padding slots hold value 0 and column 0.
struct SellMat {
    Datatype dt = Datatype::r64;
    lidx nrows = 0, ncols = 0, nrows_padded = 0;
    lidx C = 1, sigma = 1;
    gidx nnz = 0, nchunks = 0, slots = 0;
    bool cols_permuted = false;
    double beta = 1.0;
    int device = 0;
    lidx max_chunk_len = 0;
    DeviceBuffer chunk_len;     // int32 [nchunks]
    DeviceBuffer chunk_offset;  // int64 [nchunks+1]
    DeviceBuffer val;           // T [slots]
    DeviceBuffer col;           // int32 [slots]
    DeviceBuffer row_perm;      // int32 [nrows]   original -> stored
    DeviceBuffer row_perm_inv;  // int32 [nrows]   stored -> original
    DeviceBuffer rowlen;        // int32 [nrows_padded]
    // optional sweep order of the row-contiguous kernel: blocks of sweep_block_rgs row
    // groups (32 stored rows each) visited in sweep_order[] (sellkit_ext_mat_set_sweep_order)
    DeviceBuffer sweep_order;   // int32 [sweep_blocks]
    int sweep_block_rgs = 0;
    gidx sweep_blocks = 0;
    // sweep policy: 0 = automatic locality order (spmv.cu), 1 = natural row order,
    // 2 = the caller's order above
    int sweep_policy = 0;
    // automatic order: coupling distance (median over row groups of the farthest
    // |column - row| in stored space; -1 = not yet measured, 0 = not applicable) and
    // the orders built so far, per slab size in blocks
    mutable gidx coupling = -1;
    struct AutoOrder {
        int slab_blocks = 0;
        gidx nblocks = 0;
        DeviceBuffer order;  // int32 [nblocks]; empty: natural order is as good
    };
    mutable std::vector<AutoOrder> auto_orders;
    // streamed host-buffer spmv: largest column index per row-group block (lazily computed)
    mutable std::vector<lidx> watermark;
    mutable int watermark_blocks = 0;
};

struct BuildOptions {
    bool permute_columns = true;        // sellcs.hpp:127
    const lidx* imposed_order = nullptr;  // device pointer, length nrows (sellcs.hpp:130)
};

// sellcs.hpp:143-246 on the device.
std::unique_ptr<SellMat> sell_build(const Crs& a, lidx C, lidx sigma, const BuildOptions& opt);
// sellcs.hpp:269-284
void sell_update_values(SellMat& m, const Crs& a);
// sellcs.hpp:288-311
std::unique_ptr<Crs> sell_to_crs(const SellMat& m);
// sellcs.hpp:313-324 bytes_total
std::uint64_t sell_bytes_total(const SellMat& m);

// ------------------------------------------------------------- dense blocks --
enum class Order : int { row_major = 0, col_major = 1 };
enum class ViewKind { owned, compact_view, scattered_view };

// Mirrors DenseMat (densemat.hpp:20-200).  Owned matrices are device
// allocations with rows padded to row_padding(); views alias their parent.
// view_plain over caller memory may name device memory (used in place) or host
// memory (staged through the device by every operation).
struct DenseMat {
    Datatype dt = Datatype::r64;
    lidx nrows = 0, ncols = 0;
    Order order = Order::row_major;
    lidx stride = 0;
    ViewKind kind = ViewKind::owned;
    MemKind mem = MemKind::device;
    int device = 0;
    std::shared_ptr<DeviceBuffer> owner;
    char* data = nullptr;          // element (row_offset, 0) base (compact: element (0,0))
    gidx row_offset = 0;           // scattered views only
    std::vector<gidx> col_map;     // scattered views only: storage column of logical column
    std::shared_ptr<DeviceBuffer> col_map_dev;

    bool scattered() const { return kind == ViewKind::scattered_view; }
    gidx row_stride() const { return order == Order::row_major ? gidx(stride) : 1; }
    gidx col_step() const { return order == Order::row_major ? 1 : gidx(stride); }
    std::size_t esize() const { return value_bytes(dt); }
    bool same_shape(const DenseMat& o) const { return nrows == o.nrows && ncols == o.ncols; }
    gidx map_col(lidx j) const { return scattered() ? col_map[std::size_t(j)] : gidx(j); }
};

// Element addressing handed to kernels (by value).
struct DAcc {
    char* base = nullptr;
    gidx rs = 0, cs = 1;  // strides in elements
    gidx row_offset = 0;
    const gidx* cmap = nullptr;  // device col map or null
};
DAcc dacc(DenseMat& m);  // uploads col_map on demand

DenseMat densemat_create(Datatype dt, lidx nrows, lidx ncols, Order order);
DenseMat densemat_view_plain(Datatype dt, void* buffer, std::size_t nelems, lidx nrows, lidx ncols,
                             lidx stride, Order order);
DenseMat densemat_view(const DenseMat& p, lidx row_begin, lidx row_end, const lidx* cols, lidx ncols);
DenseMat densemat_compact_clone(const DenseMat& m);
DenseMat densemat_convert_order(DenseMat& m, Order new_order, bool in_place);
void densemat_copy_in(DenseMat& m, const void* host, std::size_t nelems);
void densemat_copy_out(const DenseMat& m, void* host, std::size_t nelems);
// copy logical contents between two same-shaped matrices (any memory/kind)
void densemat_copy(DenseMat& dst, const DenseMat& src);

// Device-side working copy of a host-resident matrix (identity for device
// matrices).  write_back() copies the device contents back into the host view.
struct Staged {
    DenseMat* orig = nullptr;
    DenseMat dev;
    bool staged = false;
    // slot >= 0: stage into the device runtime's reusable staging buffer `slot` (0..2)
    // instead of a fresh allocation per call (host-resident spmv operands)
    Staged(DenseMat& m, bool load, int slot = -1);
    void write_back();
};

// BLAS-1 on block vectors (densemat.hpp:243-292)
void blas_axpby(DenseMat& y, const DenseMat& x, const void* alpha, const void* beta, bool per_column);
void blas_scal(DenseMat& x, const void* factor, bool per_column);
void blas_dot(const DenseMat& a, const DenseMat& b, void* out);

}  // namespace skb
