// SELL-C-sigma SpMV/SpMMV kernels for sm_100a.
//
// Reference semantics: /root/reference/proj/src/spmv.hpp:68-92 (generic loop),
// kernels/spmv_cw.tpl.cpp:10-25 (unrolled C x W variants) and the fused row
// epilogue spmv_epilogue.hpp:12-36.  Per output element the accumulation order
// is the reference's (j ascending over the chunk, padding included), and every
// multiply/add is rounded separately, so y and z are bit-identical to the
// reference's CPU results.  Dots use a fixed-shape deterministic reduction
// (warp butterfly -> CTA -> ordered pass over CTAs), equal to the reference
// within 1e-12 relative (the reference's own dots depend on its worker count).
//
// Specialised kernel spmv_cw_kernel<T, C, W>: C in {4, 8, 32} (C divides 32),
// W in {1, 2, 4, 8, 16, 32, 64}, row-major x/y/z.  One warp owns 32 stored rows
// (32/C chunks) and a column slice of WS <= 256/sizeof(T) columns:
//   * lane l streams the value/column of its own row (coalesced 256 B + 128 B
//     per j for C = 32, L1::no_allocate + L2::evict_first so the RHS block keeps
//     the caches), and hands them to the TPR lanes that work on that row via
//     warp shuffles;
//   * each of the TPR lanes of a row gathers VEC contiguous RHS elements per
//     load (8/16-byte vector loads through the read-only path), so one warp
//     instruction reads 32/TPR complete RHS row segments of TPR*VEC*sizeof(T)
//     contiguous bytes -- the minimal number of L1 wavefronts for a row-major
//     block vector;
//   * accumulators: TPR passes x NV vectors x VEC = WS registers-worth per lane.
// The grid is persistent (occupancy x #SMs CTAs) and warps stride over row
// groups in ascending order, so all SMs sweep the matrix front-to-back together
// and the RHS window of a banded/stencil matrix stays L2-resident.
#include <algorithm>
#include <map>

#include "ops.cuh"
#include "spmv.cuh"

namespace skb {

template <class T>
struct KArgs {
    const gidx* __restrict__ chunk_offset;
    const lidx* __restrict__ chunk_len;
    const T* __restrict__ val;
    const lidx* __restrict__ col;
    lidx nrows;
    lidx nrows_padded;
    gidx nchunks;
    lidx C;
    T* y;
    gidx y_rs, y_cs;
    const T* x;
    gidx x_rs, x_cs;
    const T* xs;  // x of the output row (epilogue); == x except for remote sweeps
    gidx xs_rs, xs_cs;
    T* z;
    gidx z_rs, z_cs;
    lidx width;
    std::uint32_t flags;
    T alpha, beta, gamma, delta, eta;
    const T* gamma_list;
    T* partial;
    const std::uint32_t* defer_mask;
    const lidx* row_map;
};

namespace {

constexpr int kBlock = 256;
constexpr int kWarpsPerBlock = kBlock / 32;

// Work split of a block width over the lanes of a warp (see file comment).
template <class T, int W>
struct Plan {
    static constexpr int E = int(sizeof(T));
    static constexpr int WS_MAX = 256 / E;                       // 64 x 32-bit registers of accumulators
    static constexpr int WS = W < WS_MAX ? W : WS_MAX;           // columns per warp slice
    static constexpr int NSLICE = W / WS;
    static constexpr int VEC0 = 16 / E;
    static constexpr int VEC = WS < VEC0 ? WS : VEC0;            // elements per vector load
    static constexpr int TPR0 = WS / VEC;
    static constexpr int TPR = TPR0 < 8 ? TPR0 : 8;              // lanes per row
    static constexpr int NV = WS / (TPR * VEC);                  // vector loads per lane per row
    static constexpr int RP = 32 / TPR;                          // rows per pass
    static_assert(W % WS == 0, "width must be a multiple of the slice width");
    static_assert(kWarpsPerBlock % NSLICE == 0, "slices must tile the CTA");
};

template <class T>
__device__ __forceinline__ T apply_epilogue(const KArgs<T>& a, T t, T xv, T yv, lidx colidx) {
    using O = Ops<T>;
    if (a.flags & kFlagShift) t = O::sub(t, O::mul(a.gamma, xv));
    if (a.flags & kFlagVshift) t = O::sub(t, O::mul(a.gamma_list[colidx], xv));
    t = O::mul(t, a.alpha);
    if (a.flags & kFlagAxpby) t = O::add(t, O::mul(a.beta, yv));
    return t;
}

__device__ __forceinline__ bool deferred(const std::uint32_t* mask, gidx row) {
    return mask && ((mask[row >> 5] >> (row & 31)) & 1u);
}

template <class T, int C, int W, int U>
__global__ void __launch_bounds__(kBlock) spmv_cw_kernel(const KArgs<T> a) {
    using O = Ops<T>;
    using P = Plan<T, W>;
    constexpr int VEC = P::VEC, TPR = P::TPR, NV = P::NV, WS = P::WS, NSLICE = P::NSLICE, RP = P::RP;
    static_assert(32 % C == 0, "chunk height must divide the warp");

    __shared__ T red[kWarpsPerBlock][3][WS];

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const gidx gw = gidx(blockIdx.x) * kWarpsPerBlock + warp;
    const gidx tw = gidx(gridDim.x) * kWarpsPerBlock;
    const int slice = int(gw % NSLICE);
    const int sub = lane % TPR;
    const int rsub = lane / TPR;
    const int col_base = slice * WS;
    const gidx ngroups = (gidx(a.nrows_padded) + 31) / 32;
    const bool want_dots = (a.flags & kFlagDots) != 0;
    const bool need_x = (a.flags & (kFlagShift | kFlagVshift | kFlagDotXY | kFlagDotXX)) != 0;
    const unsigned long long pol = l2_evict_first_policy();

    T dsum[3][NV][VEC];
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
        for (int q = 0; q < NV; ++q)
#pragma unroll
            for (int e = 0; e < VEC; ++e) dsum[s][q][e] = O::zero();

    for (gidx rg = gw / NSLICE; rg < ngroups; rg += tw / NSLICE) {
        const gidx r_own = rg * 32 + lane;
        const gidx c_own = r_own / C;
        const lidx i_own = lidx(r_own - c_own * C);
        gidx off = 0;
        lidx len = 0;
        if (c_own < a.nchunks) {
            off = a.chunk_offset[c_own];
            len = a.chunk_len[c_own];
        }
        const lidx maxlen = (C == 32) ? len : lidx(__reduce_max_sync(0xffffffffu, unsigned(len)));
        const T* vptr = a.val + off + i_own;
        const lidx* cptr = a.col + off + i_own;

        T acc[TPR][NV][VEC];
#pragma unroll
        for (int p = 0; p < TPR; ++p)
#pragma unroll
            for (int q = 0; q < NV; ++q)
#pragma unroll
                for (int e = 0; e < VEC; ++e) acc[p][q][e] = O::zero();

        for (lidx j0 = 0; j0 < maxlen; j0 += U) {
            T vv[U];
            lidx cc[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const lidx j = j0 + u;
                if (j < len) {
                    vv[u] = ld_stream(vptr + gidx(j) * C, pol);
                    cc[u] = ld_stream(cptr + gidx(j) * C, pol);
                } else {
                    vv[u] = O::zero();
                    cc[u] = -1;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
#pragma unroll
                for (int p = 0; p < TPR; ++p) {
                    const int src = p * RP + rsub;
                    const T v = (TPR == 1) ? vv[u] : shfl(vv[u], src);
                    const lidx c = (TPR == 1) ? cc[u] : __shfl_sync(0xffffffffu, cc[u], src);
                    if (c >= 0) {
                        const T* xr = a.x + gidx(c) * a.x_rs + col_base + sub * VEC;
#pragma unroll
                        for (int q = 0; q < NV; ++q) {
                            const Vec<T, VEC> xv = ld_x<T, VEC>(xr + q * TPR * VEC);
#pragma unroll
                            for (int e = 0; e < VEC; ++e) acc[p][q][e] = O::add(acc[p][q][e], O::mul(v, xv.v[e]));
                        }
                    }
                }
            }
        }

        // fused epilogue (spmv_epilogue.hpp:12-36) for the TPR rows of this lane
#pragma unroll
        for (int p = 0; p < TPR; ++p) {
            const gidx row = rg * 32 + p * RP + rsub;
            if (row >= a.nrows) continue;
            const gidx orow = a.row_map ? gidx(a.row_map[row]) : row;
            const bool fin = !deferred(a.defer_mask, orow);
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const int cb = col_base + (q * TPR + sub) * VEC;
                T* yp = a.y + orow * a.y_rs + cb;
                Vec<T, VEC> xv, yv, out;
                if (need_x) xv = ld_x<T, VEC>(a.xs + orow * a.xs_rs + cb);
                if (a.flags & kFlagAxpby) yv = ld_vec<T, VEC>(yp);
#pragma unroll
                for (int e = 0; e < VEC; ++e)
                    out.v[e] = apply_epilogue(a, acc[p][q][e], need_x ? xv.v[e] : O::zero(),
                                              (a.flags & kFlagAxpby) ? yv.v[e] : O::zero(), cb + e);
                st_vec<T, VEC>(yp, out);
                if (!fin) continue;
                if (a.flags & kFlagChain) {
                    T* zp = a.z + orow * a.z_rs + cb;
                    Vec<T, VEC> zv = ld_vec<T, VEC>(zp);
#pragma unroll
                    for (int e = 0; e < VEC; ++e) zv.v[e] = O::add(O::mul(a.delta, zv.v[e]), O::mul(a.eta, out.v[e]));
                    st_vec<T, VEC>(zp, zv);
                }
                if (want_dots) {
#pragma unroll
                    for (int e = 0; e < VEC; ++e) {
                        if (a.flags & kFlagDotYY) dsum[0][q][e] = O::add(dsum[0][q][e], O::mul(O::conj(out.v[e]), out.v[e]));
                        if (a.flags & kFlagDotXY) dsum[1][q][e] = O::add(dsum[1][q][e], O::mul(O::conj(xv.v[e]), out.v[e]));
                        if (a.flags & kFlagDotXX) dsum[2][q][e] = O::add(dsum[2][q][e], O::mul(O::conj(xv.v[e]), xv.v[e]));
                    }
                }
            }
        }
    }

    if (!want_dots) return;  // uniform across the grid
    // lanes with equal `sub` hold partials of the same columns: butterfly over the row bits
#pragma unroll
    for (int m = TPR; m < 32; m <<= 1)
#pragma unroll
        for (int s = 0; s < 3; ++s)
#pragma unroll
            for (int q = 0; q < NV; ++q)
#pragma unroll
                for (int e = 0; e < VEC; ++e) dsum[s][q][e] = O::add(dsum[s][q][e], shfl_xor(dsum[s][q][e], m));
    if (lane < TPR) {
#pragma unroll
        for (int s = 0; s < 3; ++s)
#pragma unroll
            for (int q = 0; q < NV; ++q)
#pragma unroll
                for (int e = 0; e < VEC; ++e) red[warp][s][(q * TPR + lane) * VEC + e] = dsum[s][q][e];
    }
    __syncthreads();
    // CTA partial [3][W]: column c belongs to slice c / WS, summed over that slice's warps in order
    for (int t = threadIdx.x; t < 3 * W; t += kBlock) {
        const int s = t / W, c = t % W, sl = c / WS, cw = c % WS;
        T sum = O::zero();
        for (int w = sl; w < kWarpsPerBlock; w += NSLICE) sum = O::add(sum, red[w][s][cw]);
        a.partial[gidx(blockIdx.x) * 3 * W + t] = sum;
    }
}

// Generic fallback (spmv.hpp:68-92): any chunk height, any width, any strides.
// One thread per (stored row, block of GW columns).
constexpr int kGW = 8;

template <class T>
__global__ void __launch_bounds__(kBlock) spmv_generic_kernel(const KArgs<T> a) {
    using O = Ops<T>;
    __shared__ T red[3][kGW][kBlock / 32];
    const int cb0 = blockIdx.y * kGW;
    const int ncol = min(kGW, a.width - cb0);
    const bool want_dots = (a.flags & kFlagDots) != 0;
    const bool need_x = (a.flags & (kFlagShift | kFlagVshift | kFlagDotXY | kFlagDotXX)) != 0;
    T dsum[3][kGW];
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
        for (int e = 0; e < kGW; ++e) dsum[s][e] = O::zero();

    for (gidx r = blockIdx.x * gidx(blockDim.x) + threadIdx.x; r < a.nrows; r += gidx(gridDim.x) * blockDim.x) {
        const gidx c = r / a.C;
        const lidx i = lidx(r - c * a.C);
        const gidx off = a.chunk_offset[c];
        const lidx cl = a.chunk_len[c];
        T acc[kGW];
#pragma unroll
        for (int e = 0; e < kGW; ++e) acc[e] = O::zero();
        for (lidx j = 0; j < cl; ++j) {
            const gidx slot = off + gidx(j) * a.C + i;
            const T v = a.val[slot];
            const T* xr = a.x + gidx(a.col[slot]) * a.x_rs + gidx(cb0) * a.x_cs;
#pragma unroll
            for (int e = 0; e < kGW; ++e)
                if (e < ncol) acc[e] = O::add(acc[e], O::mul(v, xr[gidx(e) * a.x_cs]));
        }
        const gidx orow = a.row_map ? gidx(a.row_map[r]) : r;
        const bool fin = !deferred(a.defer_mask, orow);
#pragma unroll
        for (int e = 0; e < kGW; ++e) {
            if (e >= ncol) continue;
            const int cidx = cb0 + e;
            T* yp = a.y + orow * a.y_rs + gidx(cidx) * a.y_cs;
            const T xv = need_x ? a.xs[orow * a.xs_rs + gidx(cidx) * a.xs_cs] : O::zero();
            const T t = apply_epilogue(a, acc[e], xv, (a.flags & kFlagAxpby) ? *yp : O::zero(), cidx);
            *yp = t;
            if (!fin) continue;
            if (a.flags & kFlagChain) {
                T* zp = a.z + orow * a.z_rs + gidx(cidx) * a.z_cs;
                *zp = O::add(O::mul(a.delta, *zp), O::mul(a.eta, t));
            }
            if (a.flags & kFlagDotYY) dsum[0][e] = O::add(dsum[0][e], O::mul(O::conj(t), t));
            if (a.flags & kFlagDotXY) dsum[1][e] = O::add(dsum[1][e], O::mul(O::conj(xv), t));
            if (a.flags & kFlagDotXX) dsum[2][e] = O::add(dsum[2][e], O::mul(O::conj(xv), xv));
        }
    }
    if (!want_dots) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1)
#pragma unroll
        for (int s = 0; s < 3; ++s)
#pragma unroll
            for (int e = 0; e < kGW; ++e) dsum[s][e] = O::add(dsum[s][e], shfl_xor(dsum[s][e], m));
    if (lane == 0)
        for (int s = 0; s < 3; ++s)
            for (int e = 0; e < kGW; ++e) red[s][e][warp] = dsum[s][e];
    __syncthreads();
    if (threadIdx.x < 3 * kGW) {
        const int s = threadIdx.x / kGW, e = threadIdx.x % kGW;
        T sum = O::zero();
        for (int w = 0; w < kBlock / 32; ++w) sum = O::add(sum, red[s][e][w]);
        a.partial[(gidx(blockIdx.y) * gridDim.x + blockIdx.x) * 3 * kGW + threadIdx.x] = sum;
    }
}

// Ordered sum over CTA partials.  layout 0: partial[b][3][W]; layout 1:
// partial[cb][b][3][GW] (generic kernel).  accumulate: out += sum.
template <class T>
__global__ void dot_final_kernel(const T* partial, int nparts, int W, int layout, std::uint32_t flags, T* out,
                                 int accumulate) {
    using O = Ops<T>;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 3 * W) return;
    const int s = t / W, c = t % W;
    if (!(flags & (kFlagDotYY << s))) return;
    T sum = O::zero();
    for (int b = 0; b < nparts; ++b) {
        const gidx idx = layout == 0 ? gidx(b) * 3 * W + t
                                     : ((gidx(c / kGW) * nparts + b) * 3 + s) * kGW + (c % kGW);
        sum = O::add(sum, partial[idx]);
    }
    out[t] = accumulate ? O::add(out[t], sum) : sum;
}

// ------------------------------------------------------------------ dispatch

struct LaunchShape {
    int grid;
    int nparts;
    int layout;
};

template <class K>
int occupancy_blocks(K kernel) {
    static std::map<const void*, int> cache;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(reinterpret_cast<const void*>(kernel));
    if (it != cache.end()) return it->second;
    int nb = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kBlock, 0));
    nb = std::max(nb, 1);
    cache[reinterpret_cast<const void*>(kernel)] = nb;
    return nb;
}

template <class T, int C, int W>
LaunchShape launch_cw(const KArgs<T>& a, DeviceRuntime& rt, cudaStream_t st) {
    using P = Plan<T, W>;
    constexpr int U = (P::TPR * P::NV <= 2) ? 4 : (P::TPR * P::NV <= 4 ? 2 : 1);
    auto kern = spmv_cw_kernel<T, C, W, U>;
    const int per_sm = occupancy_blocks(kern);
    const gidx ngroups = (gidx(a.nrows_padded) + 31) / 32;
    const gidx items = ngroups * P::NSLICE;
    const gidx need = (items + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const int grid = int(std::max<gidx>(1, std::min<gidx>(need, gidx(per_sm) * rt.num_sms)));
    kern<<<grid, kBlock, 0, st>>>(a);
    return {grid, grid, 0};
}

template <class T>
LaunchShape launch_generic(const KArgs<T>& a, DeviceRuntime& rt, cudaStream_t st) {
    const int ncb = (a.width + kGW - 1) / kGW;
    const gidx need = (gidx(a.nrows) + kBlock - 1) / kBlock;
    const int gx = int(std::max<gidx>(1, std::min<gidx>(need, gidx(rt.num_sms) * 8)));
    spmv_generic_kernel<T><<<dim3(gx, ncb), kBlock, 0, st>>>(a);
    return {gx, gx, 1};
}

template <class T, int C>
bool try_launch_c(const KArgs<T>& a, DeviceRuntime& rt, cudaStream_t st, LaunchShape& ls) {
    switch (a.width) {
        case 1: ls = launch_cw<T, C, 1>(a, rt, st); return true;
        case 2: ls = launch_cw<T, C, 2>(a, rt, st); return true;
        case 4: ls = launch_cw<T, C, 4>(a, rt, st); return true;
        case 8: ls = launch_cw<T, C, 8>(a, rt, st); return true;
        case 16: ls = launch_cw<T, C, 16>(a, rt, st); return true;
        case 32: ls = launch_cw<T, C, 32>(a, rt, st); return true;
        case 64: ls = launch_cw<T, C, 64>(a, rt, st); return true;
        default: return false;
    }
}

template <class T>
LaunchShape launch_any(const KArgs<T>& a, bool specialised_ok, DeviceRuntime& rt, cudaStream_t st) {
    LaunchShape ls{};
    if (specialised_ok) {
        switch (a.C) {
            case 4:
                if (try_launch_c<T, 4>(a, rt, st, ls)) return ls;
                break;
            case 8:
                if (try_launch_c<T, 8>(a, rt, st, ls)) return ls;
                break;
            case 32:
                if (try_launch_c<T, 32>(a, rt, st, ls)) return ls;
                break;
            default: break;
        }
    }
    return launch_generic<T>(a, rt, st);
}

template <class T>
T scalar_of(const unsigned char* b) {
    T v;
    std::memcpy(&v, b, sizeof(T));
    return v;
}

// 16-B aligned view: every vector access of the specialised kernel is legal.
bool aligned_for_vectors(const DenseMat& m) {
    return (reinterpret_cast<std::uintptr_t>(m.data) % 16 == 0) &&
           ((std::size_t(m.stride) * m.esize()) % 16 == 0 || m.ncols * m.esize() < 16);
}

}  // namespace

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

        // scratch: [gamma_list W][final dots 3W][partials]
        const std::size_t max_parts = std::size_t(rt.num_sms) * 32 * std::size_t((W + kGW - 1) / kGW + 1);
        const std::size_t need = (std::size_t(W) + 3 * W + max_parts * 3 * std::max<int>(W, kGW)) * es + 256;
        auto* sc = static_cast<unsigned char*>(rt.scratch_bytes(need));
        T* gl = reinterpret_cast<T*>(sc);
        T* res = gl + W;
        a.partial = res + 3 * W;
        if (o.flags & kFlagVshift) {
            CK(cudaMemcpyAsync(gl, o.gamma_list, W * es, cudaMemcpyDefault, st));
            a.gamma_list = gl;
        }
        const LaunchShape ls = launch_any<T>(a, spec, rt, st);
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

// spmv.hpp:98-125 + 129-202
void spmv(DenseMat& y, const SellMat& A, const DenseMat& x_in, const SpmvOptions& o) {
    DenseMat x = x_in;
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

    DeviceGuard g(A.device);
    auto& rt = runtime(A.device);
    Staged xs(x, true);
    Staged ys(y, (f & kFlagAxpby) != 0);
    DenseMat zdummy;
    std::unique_ptr<Staged> zs;
    SpmvOptions run = o;
    if (f & kFlagChain) {
        zs = std::make_unique<Staged>(*o.z, true);
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
