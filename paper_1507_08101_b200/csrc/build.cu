// CRS upload/validation and SELL-C-sigma construction on the device.
// Reference: /root/reference/proj/src/sellcs.hpp:28-324.  The result is
// bit-identical to the reference's layout: same sigma permutation (stable,
// descending row length per scope), chunk lengths, int64 chunk offsets,
// slot(c,i,j) = chunk_offset[c] + j*C + i, padding value 0 / column 0, and
// column indices mapped through row_perm when the matrix is square.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "objects.cuh"
#include "ops.cuh"

namespace skb {

namespace {

constexpr int kThreads = 256;
#ifndef SK_FILL_BATCH  // rows of <= 8 slots filled with all their loads in flight (fill 2.71 -> 2.28 ms, 400^3)
#define SK_FILL_BATCH 1
#endif

int blocks_for(gidx n, int threads = kThreads) {
    return int(std::max<gidx>(1, std::min<gidx>((n + threads - 1) / threads, gidx(1) << 30)));
}

enum : int {
    kErrRowptrStart = 1,
    kErrRowptrOrder = 2,
    kErrColRange = 4,
    kErrColOrder = 8,
    kErrPattern = 16,
};

// sellcs.hpp:49-64, one thread per row.
__global__ void crs_validate_kernel(const gidx* rowptr, const gidx* col, gidx nrows, gidx ncols,
                                    int check_sorted, int* err) {
    const gidx r = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (r == 0 && rowptr[0] != 0) atomicOr(err, kErrRowptrStart);
    if (r >= nrows) return;
    const gidx b = rowptr[r], e = rowptr[r + 1];
    if (b > e) {
        atomicOr(err, kErrRowptrOrder);
        return;
    }
    int bad = 0;
    for (gidx k = b; k < e; ++k) {
        const gidx c = col[k];
        if (c < 0 || c >= ncols) bad |= kErrColRange;
        if (check_sorted && k > b && c <= col[k - 1]) bad |= kErrColOrder;
    }
    if (bad) atomicOr(err, bad);
}

__global__ void row_lengths_kernel(const gidx* rowptr, lidx n, lidx* lens) {
    const gidx r = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (r < n) lens[r] = lidx(rowptr[r + 1] - rowptr[r]);
}

__global__ void iota_kernel(lidx* out, lidx n) {
    const gidx i = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = lidx(i);
}

// sigma_permutation (sellcs.hpp:80-91) for scopes that fit shared memory: one
// CTA per scope; the stable descending rank of element i is
// #{j : len_j > len_i} + #{j < i : len_j == len_i}.
// Scopes whose rows are all shorter than kSortLMax (stencils, lattices) count instead of
// comparing: a length histogram gives the first term, and for the second the elements are
// walked in index order, 256 at a time -- lanes of equal length within a warp rank by
// __match_any_sync, earlier warps of the chunk and earlier chunks by per-length counts.
// O(scope) instead of O(scope^2) work (400^3: 3.2 ms of the build).
constexpr int kSortLMax = 63;
constexpr int kSortThreads = 256;

__global__ void __launch_bounds__(kSortThreads) scope_sort_kernel(const gidx* __restrict__ rowptr, lidx n, lidx sigma,
                                                                  lidx* __restrict__ order) {
    extern __shared__ lidx sl[];
    __shared__ int hist[kSortLMax + 1];
    __shared__ int greater[kSortLMax + 1];
    __shared__ int run[kSortLMax + 1];
    __shared__ int wcnt[kSortThreads / 32][kSortLMax + 1];
    __shared__ int big;
    const gidx s0 = gidx(blockIdx.x) * sigma;
    const lidx cnt = lidx(std::min<gidx>(sigma, gidx(n) - s0));
    if (threadIdx.x <= kSortLMax) {
        hist[threadIdx.x] = 0;
        run[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) big = 0;
    __syncthreads();
    for (lidx i = threadIdx.x; i < cnt; i += blockDim.x) {
        const lidx l = lidx(rowptr[s0 + i + 1] - rowptr[s0 + i]);
        sl[i] = l;
        if (l > kSortLMax || l < 0) big = 1;
        else atomicAdd(&hist[l], 1);
    }
    __syncthreads();
    if (big) {  // long rows in this scope: the comparison rank
        for (lidx i = threadIdx.x; i < cnt; i += blockDim.x) {
            const lidx li = sl[i];
            lidx rank = 0;
            for (lidx j = 0; j < cnt; ++j) {
                const lidx lj = sl[j];
                rank += (lj > li) || (lj == li && j < i);
            }
            order[s0 + rank] = lidx(s0 + i);
        }
        return;
    }
    if (threadIdx.x <= kSortLMax) {
        int g = 0;
        for (int m = threadIdx.x + 1; m <= kSortLMax; ++m) g += hist[m];
        greater[threadIdx.x] = g;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    __syncthreads();
    for (lidx base = 0; base < cnt; base += kSortThreads) {
        const lidx i = base + lidx(threadIdx.x);
        const bool valid = i < cnt;
        const int l = valid ? int(sl[i]) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, l);
        const int in_warp = __popc(peers & lt);
        wcnt[warp][lane] = 0;
        wcnt[warp][lane + 32] = 0;
        __syncwarp();
        if (valid && in_warp == 0) wcnt[warp][l] = __popc(peers);
        __syncthreads();
        if (valid) {
            int before = 0;
            for (int w = 0; w < warp; ++w) before += wcnt[w][l];
            order[s0 + greater[l] + run[l] + before + in_warp] = lidx(s0 + i);
        }
        __syncthreads();
        if (threadIdx.x <= kSortLMax) {
            int t = 0;
            for (int w = 0; w < kSortThreads / 32; ++w) t += wcnt[w][threadIdx.x];
            run[threadIdx.x] += t;
        }
        __syncthreads();
    }
}

// Keys for the large-scope path: (scope, maxlen - len) as one integer; a
// stable LSD radix sort of (key, index) pairs reproduces the stable sort.
__global__ void scope_keys_kernel(const lidx* lens, lidx n, lidx sigma, lidx maxlen, int len_bits,
                                  unsigned long long* keys, lidx* idx) {
    const gidx i = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const unsigned long long scope = sigma >= n ? 0ull : (unsigned long long)(i / sigma);
    keys[i] = (scope << len_bits) | (unsigned long long)(maxlen - lens[i]);
    idx[i] = lidx(i);
}

__global__ void max_kernel(const lidx* v, gidx n, int* out) {
    __shared__ int red[kThreads];
    int m = 0;
    for (gidx i = blockIdx.x * gidx(blockDim.x) + threadIdx.x; i < n; i += gidx(gridDim.x) * blockDim.x)
        m = max(m, v[i]);
    red[threadIdx.x] = m;
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
        if (int(threadIdx.x) < w) red[threadIdx.x] = max(red[threadIdx.x], red[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) atomicMax(out, red[0]);
}

// row_perm[row_perm_inv[k]] = k ; rowlen[k] = len(row_perm_inv[k]) (sellcs.hpp:169-177).
// FUSED (C divides 32): a chunk is C consecutive lanes of one warp, so the chunk
// length (sellcs.hpp:179-186) is a segmented warp max and chunk_len_kernel is skipped.
template <bool FUSED>
__global__ void perm_kernel(const lidx* __restrict__ perm_inv, const gidx* __restrict__ rowptr, lidx n, lidx n_pad,
                            lidx C, lidx* __restrict__ perm, lidx* __restrict__ rowlen, lidx* __restrict__ chunk_len,
                            gidx* __restrict__ sizes, gidx nchunks, int* maxlen) {
    __shared__ int red[kThreads / 32];
    const int lane = threadIdx.x & 31;
    const gidx k = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    lidx len = 0;
    if (k < n) {
        const lidx o = perm_inv[k];
        perm[o] = lidx(k);
        len = lidx(rowptr[o + 1] - rowptr[o]);
    }
    if (k < n_pad) rowlen[k] = len;
    if constexpr (FUSED) {
        if (k == nchunks * C) sizes[nchunks] = 0;
        lidx lc = len;
        for (int d = 1; d < C; d <<= 1) lc = max(lc, __shfl_xor_sync(0xffffffffu, lc, d));
        if (k < n_pad && lane % C == 0) {
            const gidx c = k / C;
            chunk_len[c] = lc;
            sizes[c] = gidx(C) * lc;
        }
        for (int d = 16; d >= 1; d >>= 1) lc = max(lc, __shfl_xor_sync(0xffffffffu, lc, d));
        if (lane == 0) red[threadIdx.x >> 5] = lc;
        __syncthreads();
        if (threadIdx.x == 0) {
            int m = 0;
            for (int w = 0; w < kThreads / 32; ++w) m = max(m, red[w]);
            // one atomic per CTA, and only while it raises the maximum
            if (m > *reinterpret_cast<volatile int*>(maxlen)) atomicMax(maxlen, m);
        }
    }
}

// chunk_len[c] = max rowlen over the chunk; sizes[c] = C*chunk_len[c] (sellcs.hpp:179-186)
__global__ void chunk_len_kernel(const lidx* rowlen, gidx nchunks, lidx C, lidx* chunk_len, gidx* sizes,
                                 int* maxlen) {
    const gidx c = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (c > nchunks) return;
    if (c == nchunks) {
        sizes[c] = 0;
        return;
    }
    lidx lc = 0;
    for (lidx i = 0; i < C; ++i) lc = max(lc, rowlen[c * C + i]);
    chunk_len[c] = lc;
    sizes[c] = gidx(C) * lc;
    atomicMax(maxlen, lc);
}

// Chunk fill (sellcs.hpp:193-229), one thread per stored row: writes every
// slot j < chunk_len of its row, padding with value 0 / column 0.
template <class T>
__global__ void fill_kernel(const gidx* __restrict__ rowptr, const gidx* __restrict__ ccol, const T* __restrict__ cval,
                            const lidx* __restrict__ perm_inv, const lidx* __restrict__ perm,
                            const lidx* __restrict__ rowlen, const lidx* __restrict__ chunk_len,
                            const gidx* __restrict__ chunk_offset, lidx n, lidx n_pad, lidx C, gidx ncols, int permute,
                            T* __restrict__ val, lidx* __restrict__ col, int* err) {
    const gidx k = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (k >= n_pad) return;
    const gidx c = k / C;
    const lidx i = lidx(k - c * C);
    const lidx cl = chunk_len[c];
    const gidx off = chunk_offset[c];
    lidx len = 0;
    gidx src = 0;
    if (k < n) {
        len = rowlen[k];
        src = rowptr[perm_inv[k]];
    }
    int bad = 0;
#if SK_FILL_BATCH
    // rows of up to 8 slots (stencils, lattices): all loads of the row in flight at once
    if (cl <= 8) {
        gidx g[8];
        T v[8];
        lidx sc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < len) {
                g[j] = ccol[src + j];
                v[j] = cval[src + j];
            }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < len) {
                sc[j] = 0;
                if (g[j] < 0 || g[j] >= ncols) bad = 1;
                else sc[j] = permute ? perm[g[j]] : lidx(g[j]);
            }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < cl) {
                const gidx slot = off + gidx(j) * C + i;
                val[slot] = j < len ? v[j] : Ops<T>::zero();
                col[slot] = j < len ? sc[j] : 0;
            }
        if (bad) atomicOr(err, kErrColRange);
        return;
    }
#endif
#pragma unroll 4
    for (lidx j = 0; j < cl; ++j) {
        const gidx slot = off + gidx(j) * C + i;
        if (j < len) {
            const gidx g = ccol[src + j];
            lidx sc = 0;
            if (g < 0 || g >= ncols) bad = 1;
            else sc = permute ? perm[g] : lidx(g);
            val[slot] = cval[src + j];
            col[slot] = sc;
        } else {
            val[slot] = Ops<T>::zero();
            col[slot] = 0;
        }
    }
    if (bad) atomicOr(err, kErrColRange);
}

// update_values (sellcs.hpp:269-284), one thread per original row.
template <class T>
__global__ void update_values_kernel(const gidx* __restrict__ rowptr, const T* __restrict__ cval,
                                     const lidx* __restrict__ perm, const lidx* __restrict__ rowlen,
                                     const gidx* __restrict__ chunk_offset, lidx n, lidx C, T* __restrict__ val,
                                     int* err) {
    const gidx o = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (o >= n) return;
    const lidx stored = perm[o];
    const gidx b = rowptr[o];
    const lidx len = lidx(rowptr[o + 1] - b);
    if (len != rowlen[stored]) {
        atomicOr(err, kErrPattern);
        return;
    }
    const gidx c = stored / C;
    const lidx i = stored - lidx(c * C);
    const gidx base = chunk_offset[c];
#if SK_FILL_BATCH
    if (len <= 8) {
        T v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < len) v[j] = cval[b + j];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < len) val[base + gidx(j) * C + i] = v[j];
        return;
    }
#endif
#pragma unroll 4
    for (lidx j = 0; j < len; ++j) val[base + gidx(j) * C + i] = cval[b + j];
}

// to_crs (sellcs.hpp:288-311)
__global__ void to_crs_len_kernel(const lidx* perm, const lidx* rowlen, lidx n, gidx* lens64) {
    const gidx o = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (o < n) lens64[o] = rowlen[perm[o]];
    if (o == n) lens64[o] = 0;
}

template <class T>
__global__ void to_crs_fill_kernel(const lidx* perm, const lidx* perm_inv, const lidx* rowlen,
                                   const gidx* chunk_offset, const T* val, const lidx* col, lidx n, lidx C,
                                   int permuted, const gidx* rowptr, gidx* ocol, T* oval) {
    const gidx o = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (o >= n) return;
    const lidx stored = perm[o];
    const gidx c = stored / C;
    const lidx i = stored - lidx(c * C);
    const gidx base = chunk_offset[c];
    const gidx dst = rowptr[o];
    for (lidx j = 0; j < rowlen[stored]; ++j) {
        const lidx sc = col[base + gidx(j) * C + i];
        ocol[dst + j] = permuted ? gidx(perm_inv[sc]) : gidx(sc);
        oval[dst + j] = val[base + gidx(j) * C + i];
    }
}

int read_flag(DeviceBuffer& flag, DeviceRuntime& rt) {
    int h = 0;
    CK(cudaMemcpyAsync(&h, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, rt.stream));
    CK(cudaStreamSynchronize(rt.stream));
    return h;
}

}  // namespace

void exclusive_scan_i64(const gidx* in, gidx* out, gidx n, DeviceRuntime& rt) {
    std::size_t tmp_bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, in, out, n, rt.stream));
    DeviceBuffer tmp(std::max<std::size_t>(tmp_bytes, 1), rt.device);
    CK(cub::DeviceScan::ExclusiveSum(tmp.get(), tmp_bytes, in, out, n, rt.stream));
    CK(cudaStreamSynchronize(rt.stream));
}

// ------------------------------------------------------------------- CRS ---

void crs_validate_impl(const Crs& a, bool check_sorted) {
    auto& rt = runtime(a.device);
    int* flag = rt.flag();
    crs_validate_kernel<<<blocks_for(std::max<gidx>(a.nrows, 1)), kThreads, 0, rt.stream>>>(
        a.rowptr.as<gidx>(), a.col.as<gidx>(), a.nrows, a.ncols, check_sorted ? 1 : 0, flag);
    CK(cudaGetLastError());
    const int e = rt.read_flag();
    SK_REQUIRE(!(e & kErrRowptrStart), errc::invalid_arg, "rowptr must start at 0");
    SK_REQUIRE(!(e & kErrRowptrOrder), errc::invalid_arg, "rowptr must be non-decreasing");
    SK_REQUIRE(!(e & kErrColRange), errc::invalid_arg, "column index out of range");
    SK_REQUIRE(!(e & kErrColOrder), errc::invalid_arg, "columns must be strictly increasing per row");
}

void crs_validate(const Crs& a) { crs_validate_impl(a, true); }

static std::unique_ptr<Crs> crs_alloc(Datatype dt, gidx nrows, gidx ncols, gidx nnz) {
    auto a = std::make_unique<Crs>();
    a->dt = dt;
    a->nrows = nrows;
    a->ncols = ncols;
    a->nnz = nnz;
    a->device = current_device();
    a->rowptr = DeviceBuffer(std::size_t(nrows + 1) * sizeof(gidx), a->device);
    a->col = DeviceBuffer(std::max<std::size_t>(std::size_t(nnz) * sizeof(gidx), 8), a->device);
    a->val = DeviceBuffer(std::max<std::size_t>(std::size_t(nnz) * value_bytes(dt), 16), a->device);
    return a;
}

std::unique_ptr<Crs> crs_from_host(Datatype dt, gidx nrows, gidx ncols, const gidx* rowptr, const gidx* col,
                                   const void* val) {
    SK_REQUIRE(nrows >= 0 && ncols >= 0, errc::invalid_arg, "negative dimension");
    const gidx nnz = rowptr[nrows];
    SK_REQUIRE(nnz >= 0, errc::invalid_arg, "negative nonzero count");
    auto a = crs_alloc(dt, nrows, ncols, nnz);
    auto& rt = runtime(a->device);
    CK(cudaMemcpyAsync(a->rowptr.get(), rowptr, std::size_t(nrows + 1) * sizeof(gidx), cudaMemcpyHostToDevice,
                       rt.stream));
    if (nnz > 0) {
        CK(cudaMemcpyAsync(a->col.get(), col, std::size_t(nnz) * sizeof(gidx), cudaMemcpyHostToDevice, rt.stream));
        CK(cudaMemcpyAsync(a->val.get(), val, std::size_t(nnz) * value_bytes(dt), cudaMemcpyHostToDevice,
                           rt.stream));
    }
    crs_validate(*a);
    return a;
}

std::unique_ptr<Crs> crs_from_device(Datatype dt, gidx nrows, gidx ncols, const gidx* rowptr, const gidx* col,
                                     const void* val) {
    SK_REQUIRE(nrows >= 0 && ncols >= 0, errc::invalid_arg, "negative dimension");
    gidx nnz = 0;
    auto& rt0 = runtime(current_device());
    CK(cudaMemcpyAsync(&nnz, rowptr + nrows, sizeof(gidx), cudaMemcpyDeviceToHost, rt0.stream));
    CK(cudaStreamSynchronize(rt0.stream));
    SK_REQUIRE(nnz >= 0, errc::invalid_arg, "negative nonzero count");
    auto a = crs_alloc(dt, nrows, ncols, nnz);
    auto& rt = runtime(a->device);
    CK(cudaMemcpyAsync(a->rowptr.get(), rowptr, std::size_t(nrows + 1) * sizeof(gidx), cudaMemcpyDefault, rt.stream));
    if (nnz > 0) {
        CK(cudaMemcpyAsync(a->col.get(), col, std::size_t(nnz) * sizeof(gidx), cudaMemcpyDefault, rt.stream));
        CK(cudaMemcpyAsync(a->val.get(), val, std::size_t(nnz) * value_bytes(dt), cudaMemcpyDefault, rt.stream));
    }
    crs_validate(*a);
    return a;
}

void crs_download(const Crs& a, std::vector<gidx>& rowptr, std::vector<gidx>& col, std::vector<unsigned char>& val) {
    auto& rt = runtime(a.device);
    rowptr.resize(std::size_t(a.nrows + 1));
    col.resize(std::size_t(a.nnz));
    val.resize(std::size_t(a.nnz) * value_bytes(a.dt));
    CK(cudaMemcpyAsync(rowptr.data(), a.rowptr.get(), rowptr.size() * sizeof(gidx), cudaMemcpyDeviceToHost, rt.stream));
    if (a.nnz) {
        CK(cudaMemcpyAsync(col.data(), a.col.get(), col.size() * sizeof(gidx), cudaMemcpyDeviceToHost, rt.stream));
        CK(cudaMemcpyAsync(val.data(), a.val.get(), val.size(), cudaMemcpyDeviceToHost, rt.stream));
    }
    CK(cudaStreamSynchronize(rt.stream));
}

// ---------------------------------------------------------------- build ----

std::unique_ptr<SellMat> sell_build(const Crs& a, lidx C, lidx sigma, const BuildOptions& opt) {
    // sellcs.hpp:28-33
    SK_REQUIRE(C >= 1, errc::invalid_arg, "chunk height must be positive");
    SK_REQUIRE(sigma >= 1, errc::invalid_arg, "sigma must be positive");
    SK_REQUIRE(sigma == 1 || sigma % C == 0 || gidx(sigma) >= a.nrows, errc::invalid_arg,
               "sigma must be 1, a multiple of the chunk height, or cover all rows");
    const lidx n = narrow_index(a.nrows);
    const lidx nc = narrow_index(a.ncols);
    SK_REQUIRE(n > 0, errc::invalid_arg, "matrix must have at least one row");
    SK_REQUIRE(!opt.permute_columns || n == nc, errc::invalid_arg, "column permutation requires a square matrix");

    DeviceGuard g(a.device);
    auto& rt = runtime(a.device);
    auto m = std::make_unique<SellMat>();
    m->dt = a.dt;
    m->nrows = n;
    m->ncols = nc;
    m->C = C;
    m->sigma = sigma;
    m->cols_permuted = opt.permute_columns;
    m->device = a.device;
    m->nnz = a.nnz;


    m->row_perm_inv = DeviceBuffer::cached(std::size_t(n) * sizeof(lidx), a.device);
    lidx* pinv = m->row_perm_inv.as<lidx>();
    if (opt.imposed_order) {
        CK(cudaMemcpyAsync(pinv, opt.imposed_order, std::size_t(n) * sizeof(lidx), cudaMemcpyDefault, rt.stream));
    } else if (sigma <= 1) {
        iota_kernel<<<blocks_for(n), kThreads, 0, rt.stream>>>(pinv, n);
    } else {
        const lidx scope = lidx(std::min<gidx>(sigma, n));
        if (scope <= 4096) {
            const gidx nscopes = (gidx(n) + scope - 1) / scope;
            scope_sort_kernel<<<unsigned(nscopes), kSortThreads, std::size_t(scope) * sizeof(lidx), rt.stream>>>(
                a.rowptr.as<gidx>(), n, scope, pinv);
        } else {
            auto lens = DeviceBuffer::pooled(std::size_t(n) * sizeof(lidx), a.device);
            row_lengths_kernel<<<blocks_for(n), kThreads, 0, rt.stream>>>(a.rowptr.as<gidx>(), n, lens.as<lidx>());
            auto mx = DeviceBuffer::pooled(sizeof(int), a.device);
            CK(cudaMemsetAsync(mx.get(), 0, sizeof(int), rt.stream));
            max_kernel<<<std::min(blocks_for(n), rt.num_sms * 4), kThreads, 0, rt.stream>>>(lens.as<lidx>(), n,
                                                                                       mx.as<int>());
            const int maxlen = read_flag(mx, rt);
            int len_bits = 1;
            while ((gidx(1) << len_bits) <= maxlen) ++len_bits;
            const gidx nscopes = (gidx(n) + scope - 1) / scope;
            int scope_bits = 0;
            while ((gidx(1) << scope_bits) < nscopes) ++scope_bits;
            auto keys = DeviceBuffer::pooled(std::size_t(n) * 8, a.device);
            auto keys2 = DeviceBuffer::pooled(std::size_t(n) * 8, a.device);
            auto idx = DeviceBuffer::pooled(std::size_t(n) * 4, a.device);
            scope_keys_kernel<<<blocks_for(n), kThreads, 0, rt.stream>>>(lens.as<lidx>(), n, scope, maxlen, len_bits,
                                                                          keys.as<unsigned long long>(), idx.as<lidx>());
            std::size_t tmp_bytes = 0;
            const int end_bit = len_bits + scope_bits;
            CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.as<unsigned long long>(),
                                               keys2.as<unsigned long long>(), idx.as<lidx>(), pinv, n, 0, end_bit,
                                               rt.stream));
            auto tmp = DeviceBuffer::pooled(std::max<std::size_t>(tmp_bytes, 1), a.device);
            CK(cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, keys.as<unsigned long long>(),
                                               keys2.as<unsigned long long>(), idx.as<lidx>(), pinv, n, 0, end_bit,
                                               rt.stream));
            CK(cudaStreamSynchronize(rt.stream));
        }
    }
    CK(cudaGetLastError());

    const gidx nchunks = (gidx(n) + C - 1) / C;
    m->nchunks = nchunks;
    SK_REQUIRE(nchunks * C < (gidx(1) << 31), errc::overflow, "padded row count exceeds the 32-bit range");
    m->nrows_padded = lidx(nchunks * C);
    m->row_perm = DeviceBuffer::cached(std::size_t(n) * sizeof(lidx), a.device);
    m->rowlen = DeviceBuffer::cached(std::size_t(m->nrows_padded) * sizeof(lidx), a.device);
    m->chunk_len = DeviceBuffer::cached(std::size_t(nchunks) * sizeof(lidx), a.device);
    m->chunk_offset = DeviceBuffer::cached(std::size_t(nchunks + 1) * sizeof(gidx), a.device);
    {
        auto sizes = DeviceBuffer::pooled(std::size_t(nchunks + 1) * sizeof(gidx), a.device);
        auto out = DeviceBuffer::pooled(2 * sizeof(gidx), a.device);  // {max chunk length, slots}
        CK(cudaMemsetAsync(out.get(), 0, sizeof(gidx), rt.stream));
        const bool fused = 32 % C == 0;
        (fused ? perm_kernel<true> : perm_kernel<false>)<<<blocks_for(gidx(m->nrows_padded) + 1), kThreads, 0,
                                                           rt.stream>>>(
            pinv, a.rowptr.as<gidx>(), n, m->nrows_padded, C, m->row_perm.as<lidx>(), m->rowlen.as<lidx>(),
            m->chunk_len.as<lidx>(), sizes.as<gidx>(), nchunks, out.as<int>());
        CK(cudaGetLastError());
        if (!fused) {
            chunk_len_kernel<<<blocks_for(nchunks + 1), kThreads, 0, rt.stream>>>(
                m->rowlen.as<lidx>(), nchunks, C, m->chunk_len.as<lidx>(), sizes.as<gidx>(), out.as<int>());
            CK(cudaGetLastError());
        }
        std::size_t tmp_bytes = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, sizes.as<gidx>(), m->chunk_offset.as<gidx>(),
                                         nchunks + 1, rt.stream));
        auto tmp = DeviceBuffer::pooled(std::max<std::size_t>(tmp_bytes, 1), rt.device);
        CK(cub::DeviceScan::ExclusiveSum(tmp.get(), tmp_bytes, sizes.as<gidx>(), m->chunk_offset.as<gidx>(),
                                         nchunks + 1, rt.stream));
        CK(cudaMemcpyAsync(out.as<gidx>() + 1, m->chunk_offset.as<gidx>() + nchunks, sizeof(gidx),
                           cudaMemcpyDeviceToDevice, rt.stream));
        gidx h[2] = {0, 0};
        CK(cudaMemcpyAsync(h, out.get(), sizeof(h), cudaMemcpyDeviceToHost, rt.stream));
        CK(cudaStreamSynchronize(rt.stream));
        m->max_chunk_len = int(h[0] & 0xffffffff);
        m->slots = h[1];
    }
    m->beta = m->slots > 0 ? double(m->nnz) / double(m->slots) : 1.0;

    const std::size_t es = value_bytes(a.dt);
    m->val = DeviceBuffer::cached(std::max<std::size_t>(std::size_t(m->slots) * es, 16), a.device);
    m->col = DeviceBuffer::cached(std::max<std::size_t>(std::size_t(m->slots) * sizeof(lidx), 16), a.device);
    int* flag = rt.flag();
    visit_dt(a.dt, [&]<class T>() {
        fill_kernel<T><<<blocks_for(m->nrows_padded), kThreads, 0, rt.stream>>>(
            a.rowptr.as<gidx>(), a.col.as<gidx>(), a.val.as<T>(), pinv, m->row_perm.as<lidx>(), m->rowlen.as<lidx>(),
            m->chunk_len.as<lidx>(), m->chunk_offset.as<gidx>(), n, m->nrows_padded, C, a.ncols,
            m->cols_permuted ? 1 : 0, m->val.as<T>(), m->col.as<lidx>(), flag);
        return 0;
    });
    CK(cudaGetLastError());
    const int e = rt.read_flag();
    SK_REQUIRE(!(e & kErrColRange), errc::invalid_arg, "column index out of range");
    return m;
}

void sell_update_values(SellMat& m, const Crs& a) {
    SK_REQUIRE(a.nrows == m.nrows, errc::pattern_mismatch, "row count differs");
    SK_REQUIRE(a.nnz == m.nnz, errc::pattern_mismatch, "nonzero count differs");
    SK_REQUIRE(a.dt == m.dt, errc::invalid_arg, "datatype mismatch between matrix and CRS data");
    DeviceGuard g(m.device);
    auto& rt = runtime(m.device);
    int* flag = rt.flag();
    visit_dt(m.dt, [&]<class T>() {
        update_values_kernel<T><<<blocks_for(m.nrows), kThreads, 0, rt.stream>>>(
            a.rowptr.as<gidx>(), a.val.as<T>(), m.row_perm.as<lidx>(), m.rowlen.as<lidx>(), m.chunk_offset.as<gidx>(),
            m.nrows, m.C, m.val.as<T>(), flag);
        return 0;
    });
    CK(cudaGetLastError());
    const int e = rt.read_flag();
    SK_REQUIRE(!(e & kErrPattern), errc::pattern_mismatch, "row length differs from the stored pattern");
}

std::unique_ptr<Crs> sell_to_crs(const SellMat& m) {
    DeviceGuard g(m.device);
    auto& rt = runtime(m.device);
    auto out = crs_alloc(m.dt, m.nrows, m.ncols, m.nnz);
    DeviceBuffer lens64(std::size_t(m.nrows + 1) * sizeof(gidx), m.device);
    to_crs_len_kernel<<<blocks_for(gidx(m.nrows) + 1), kThreads, 0, rt.stream>>>(
        m.row_perm.as<lidx>(), m.rowlen.as<lidx>(), m.nrows, lens64.as<gidx>());
    CK(cudaGetLastError());
    exclusive_scan_i64(lens64.as<gidx>(), out->rowptr.as<gidx>(), gidx(m.nrows) + 1, rt);
    visit_dt(m.dt, [&]<class T>() {
        to_crs_fill_kernel<T><<<blocks_for(m.nrows), kThreads, 0, rt.stream>>>(
            m.row_perm.as<lidx>(), m.row_perm_inv.as<lidx>(), m.rowlen.as<lidx>(), m.chunk_offset.as<gidx>(),
            m.val.as<T>(), m.col.as<lidx>(), m.nrows, m.C, m.cols_permuted ? 1 : 0, out->rowptr.as<gidx>(),
            out->col.as<gidx>(), out->val.as<T>());
        return 0;
    });
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(rt.stream));
    return out;
}

std::uint64_t sell_bytes_total(const SellMat& m) {
    return std::uint64_t(m.slots) * (value_bytes(m.dt) + sizeof(lidx)) + std::uint64_t(m.nchunks) * sizeof(lidx) +
           std::uint64_t(m.nchunks + 1) * sizeof(gidx) +
           (std::uint64_t(m.nrows) * 2 + std::uint64_t(m.nrows_padded)) * sizeof(lidx);
}

}  // namespace skb
