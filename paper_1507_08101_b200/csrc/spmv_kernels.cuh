// SELL-C-sigma SpMV/SpMMV kernel templates for sm_100a (included by the per-type
// instantiation units spmv_r32.cu / spmv_r64.cu / spmv_c32.cu / spmv_c64.cu and by
// spmv.cu).  See the comment block below for the design.
#pragma once
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
#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>

#include "ops.cuh"
#include "spmv.cuh"
#include "tma.cuh"

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
    gidx rg0, rg1;  // row groups (32 stored rows each) [rg0, rg1) swept by this launch
    const int* sweep_order;  // full sweeps only: blocks of sweep_brg row groups in this order
    int sweep_brg;           // 0 = natural order
    int grid_sms;            // launch: SMs the grid may fill (0 = all; the rest stay free for a
                             // concurrent halo pack on the communication stream)
    int* tile_counter;       // rows kernels without dots: tiles handed out by an atomic counter
                             // (zeroed before the launch) instead of a static round robin
    int grp_end;             // rows kernel (set at launch): min(nrows_padded, 32 rg1)
#if SK_CHECK
    lidx xrows;              // checked build: rows of x (gather bound)
    gidx slots;              // checked build: stored slots of the matrix
#endif
};

// Checked build (make EXTRA_NVFLAGS=-DSK_CHECK=1, tools/check_build.sh): device-side bounds
// assertions on every gather index and matrix range -- the stand-in for compute-sanitizer's
// memcheck, which is closed on this pool.
#ifndef SK_CHECK
#define SK_CHECK 0
#endif
#if SK_CHECK
#define SK_DEVICE_CHECK(cond, what)                                                                    \
    do {                                                                                               \
        if (!(cond)) {                                                                                 \
            printf("[sellkit check] %s failed: %s (block %d thread %d)\n", what, #cond, int(blockIdx.x), \
                   int(threadIdx.x));                                                                  \
            __trap();                                                                                  \
        }                                                                                              \
    } while (0)
#else
#define SK_DEVICE_CHECK(cond, what) ((void)0)
#endif

namespace spmv_detail {

constexpr int kBlock = 256;
constexpr int kWarpsPerBlock = kBlock / 32;

// Work split of a block width over the lanes of a warp (see file comment).
template <class T, int W, int ACC_BYTES = 256, int VEC_BYTES = 16>
struct Plan {
    static constexpr int E = int(sizeof(T));
    static constexpr int WS_MAX = ACC_BYTES / E;                 // ACC_BYTES/4 32-bit registers of accumulators
    static constexpr int WS = W < WS_MAX ? W : WS_MAX;           // columns per warp slice
    static constexpr int NSLICE = W / WS;
    static constexpr int VEC0 = VEC_BYTES / E;
    static constexpr int VEC = WS < VEC0 ? WS : VEC0;            // elements per vector load
    static constexpr int TPR0 = WS / VEC;
    static constexpr int TPR = TPR0 < 8 ? TPR0 : 8;              // lanes per row
    static constexpr int NV = WS / (TPR * VEC);                  // vector loads per lane per row
    static constexpr int RP = 32 / TPR;                          // rows per pass
    static_assert(W % WS == 0, "width must be a multiple of the slice width");
    static_assert(kWarpsPerBlock % NSLICE == 0, "slices must tile the CTA");
};

// j-unroll: as many columns of the chunk in flight as fit ~32 registers of RHS data per lane
template <class T, class P, int BUDGET = 32>
constexpr int unroll_of() {
    constexpr int regs = P::TPR * P::NV * P::VEC * int(sizeof(T)) / 4;
    constexpr int u = BUDGET / (regs > 0 ? regs : 1);
    return u < 1 ? 1 : (u > 8 ? 8 : u);
}

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

// Producer look-ahead: after issuing tile it's copies, prefetch into L2 the chunk
// headers (chunk_offset / chunk_len) of the tile SK_HDR_PREFETCH tiles ahead, so the
// producer's dependent header loads for it hit L2; 0 = off.  Measured on B200 (same
// box, 3 rounds, gpurun_out/ab_hdrpf.log): C1 1000^2 w = 1 22.5 -> 20.5 us, 256^3 w = 1
// 260 -> 250 us, w = 4 374 -> 367 us, w >= 8 unchanged.  The row-contiguous kernels
// with an epilogue (AXPBY w = 8: 0.70 -> 0.715 ms, also with a runtime flag gate) got a
// worse schedule, so there it is compiled into the epilogue-free (PLAIN) and the dots
// kernels only (dots, gpurun_out/ab_hdrpf_dots.log: C3 C64 5.85 -> 5.71-5.81 ms row order,
// 5.03 -> 4.96 ms pencil order, 400^3 w = 1 with three dots 1.047 -> 1.016 ms).
#ifndef SK_HDR_PREFETCH
#define SK_HDR_PREFETCH 1
#endif
__device__ __forceinline__ void prefetch_headers(const gidx* chunk_offset, const lidx* chunk_len, gidx c0, int nc,
                                                 int lane) {
    // 16 offsets / 32 lengths per 128-B line
    if (lane * 16 <= nc) prefetch_l2(chunk_offset + c0 + lane * 16);
    if (lane * 32 < nc) prefetch_l2(chunk_len + c0 + lane * 32);
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
    const gidx ngroups = a.rg1;
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

    for (gidx rg = a.rg0 + gw / NSLICE; rg < ngroups; rg += tw / NSLICE) {
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
            // branch-free: gather all RHS vectors first (index -1 => row 0, result discarded)
            T vs[U][TPR];
            bool ok[U][TPR];
            Vec<T, VEC> xv[U][TPR][NV];
#pragma unroll
            for (int u = 0; u < U; ++u) {
#pragma unroll
                for (int p = 0; p < TPR; ++p) {
                    const int src = p * RP + rsub;
                    vs[u][p] = (TPR == 1) ? vv[u] : shfl(vv[u], src);
                    const lidx c = (TPR == 1) ? cc[u] : __shfl_sync(0xffffffffu, cc[u], src);
                    ok[u][p] = c >= 0;
                    const T* xr = a.x + gidx(c < 0 ? 0 : c) * a.x_rs + col_base + sub * VEC;
#pragma unroll
                    for (int q = 0; q < NV; ++q) xv[u][p][q] = ld_x<T, VEC>(xr + q * TPR * VEC);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int p = 0; p < TPR; ++p)
#pragma unroll
                    for (int q = 0; q < NV; ++q)
#pragma unroll
                        for (int e = 0; e < VEC; ++e) {
                            const T s = O::add(acc[p][q][e], O::mul(vs[u][p], xv[u][p][q].v[e]));
                            acc[p][q][e] = ok[u][p] ? s : acc[p][q][e];
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

// ---------------------------------------------------------------------------
// TMA-pipelined variant (the production path for C in {4, 8, 32}).
//
// CTA = kNCW consumer warps + 1 producer warp, persistent, tiles of `rgt` row
// groups (32 rows each) taken in ascending order (tile = blockIdx.x + k*grid).
// A tile's values and column indices are contiguous in the SELL arrays, so the
// producer streams each of them with ONE cp.async.bulk into a kStages-deep ring
// of shared-memory stages (mbarrier transaction counts signal arrival, an
// "empty" mbarrier per stage returns it).  The matrix stream therefore runs
// kStages-1 tiles ahead of the math without occupying registers, and the
// consumers read values/indices with broadcast LDS (no shuffles); only the RHS
// gathers use LDG (L1-cached, L2-resident window).
#ifndef SK_NCW
#define SK_NCW 8
#endif
#ifndef SK_STAGE_KB
#define SK_STAGE_KB 32
#endif
#ifndef SK_STAGES
#define SK_STAGES 3
#endif
#ifndef SK_MINB
#define SK_MINB 2
#endif
#ifndef SK_MINB_WIDE  // CTAs/SM of the column-slice kernel for complex-double RHS rows of 512 B and more
#define SK_MINB_WIDE 1  // (2 spills 176-520 B: cplx w = 32 / 64 plain 22.8 / 41.3 -> 19.3 / 32.1 ms, r2bd)
#endif
constexpr int kNCW = SK_NCW;
constexpr int kTmaThreads = (kNCW + 1) * 32;
constexpr int kStageBytes = SK_STAGE_KB * 1024;
constexpr int kStages = SK_STAGES;
constexpr int kMaxTileChunks = kNCW * 32 / 4;

struct StageHdr {
    int hoff[kMaxTileChunks + 1];  // slot offset of chunk q relative to the tile start
    int hlen[kMaxTileChunks];      // chunk lengths
    int overflow;                  // tile did not fit the stage: read from global
    int nchunks;
    long long off0;                // absolute slot offset of the tile
    int row0;                      // first stored row of the tile (rows kernel)
};

// Work split of the TMA kernel: every consumer warp owns one 32-B column slice of
// its 32 rows (lane = row, one LDG.256 per nonzero), so the RHS gathers of a warp
// hit 32 distinct rows and the accumulators stay at 8 registers; wider blocks are
// split into slices handled by different consumer warps that read the same
// shared-memory stage (the matrix is fetched from HBM once per tile either way).
// Measured on B200 (400^3 stencil, w = 8): 1 lane per row beats 2-4 lanes per row.
#ifndef SK_ACC
#define SK_ACC 32
#endif
#ifndef SK_UBUDGET
#define SK_UBUDGET 32
#endif
template <class T, int W>
using TPlan = Plan<T, W, (W * int(sizeof(T)) / 8 > SK_ACC ? W * int(sizeof(T)) / 8 : SK_ACC), 32>;

// Stage size: narrow blocks are matrix-stream bound and want deep stages; from
// 64-B RHS rows on, the RHS gathers dominate and profit from the L1 capacity that
// smaller stages leave free (measured: w=8 4.7 ms with 32 KB stages, 3.8 ms with 16 KB).
template <class T, int W>
struct TmaGeom {
    static constexpr int SB = (W * int(sizeof(T)) >= 64 ? 16 : kStageBytes / 1024) * 1024;
    static constexpr int SCAP = (SB / int(sizeof(T) + 4)) / 32 * 32;  // slots per stage
};

template <class T, int W>
constexpr std::size_t tma_smem_bytes() {
    return std::size_t(kStages) * TmaGeom<T, W>::SB + std::size_t(kStages) * sizeof(StageHdr) + 2 * kStages * 8 + 128;
}

template <class T, int C, int W, int U, bool SMEM>
__device__ __forceinline__ void tma_rowgroup(const KArgs<T>& a, const T* sval, const lidx* scol, const StageHdr& h,
                                             int rgi, gidx rg, int slice, int lane,
                                             T (&acc)[TPlan<T, W>::TPR][TPlan<T, W>::NV][TPlan<T, W>::VEC]) {
    using O = Ops<T>;
    using P = TPlan<T, W>;
    constexpr int VEC = P::VEC, TPR = P::TPR, NV = P::NV, WS = P::WS, RP = P::RP;
    const int sub = lane % TPR;
    const int rsub = lane / TPR;
    const int col_base = slice * WS;
    // slot of (pass p, j) relative to the stage (or, on overflow, to the tile start):
    // offp[p] + j*C.  C == 32: one chunk per row group, offp[p] = hoff + row.
    int offp[TPR];
    lidx lenp[TPR];
    lidx maxlen = 0;
#pragma unroll
    for (int p = 0; p < TPR; ++p) {
        const int rp = p * RP + rsub;
        const int cq = (rgi * 32 + rp) / C;
        const int ip = (rgi * 32 + rp) % C;
        lenp[p] = cq < h.nchunks ? h.hlen[cq] : 0;
        offp[p] = h.hoff[cq] + ip;
        maxlen = max(maxlen, lenp[p]);
    }
    if constexpr (C < 32) maxlen = lidx(__reduce_max_sync(0xffffffffu, unsigned(maxlen)));
    const T* vbase = SMEM ? sval : a.val + h.off0;
    const lidx* cbase = SMEM ? scol : a.col + h.off0;
#pragma unroll
    for (int p = 0; p < TPR; ++p)
#pragma unroll
        for (int q = 0; q < NV; ++q)
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[p][q][e] = O::zero();
    lidx minlen = maxlen;
#pragma unroll
    for (int p = 0; p < TPR; ++p) minlen = min(minlen, lenp[p]);
    if constexpr (C < 32) minlen = lidx(__reduce_min_sync(0xffffffffu, unsigned(minlen)));
    const T* xb = a.x + col_base + sub * VEC;
    const unsigned xrs = unsigned(a.x_rs);

    // Two-phase body: first every value/index/RHS load of U columns x TPR passes is
    // issued, then the products are accumulated.  In the main loop every (row, j)
    // is in range (j < min chunk length of the warp).  In the tail, out-of-range
    // slots read slot 0 (always present) and the accumulator is kept by a select,
    // so the result is exactly the reference's (no extra +0 terms).
    auto body = [&](lidx j0, auto tail) {
        constexpr bool TAIL = decltype(tail)::value;
        T vv[U][TPR];
        Vec<T, VEC> xv[U][TPR][NV];
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int p = 0; p < TPR; ++p) {
                const lidx j = j0 + u;
                const int slot = (!TAIL || j < lenp[p]) ? offp[p] + j * C : 0;
                vv[u][p] = vbase[slot];
                const unsigned c = unsigned(cbase[slot]);
                const T* xr = xb + std::size_t(c) * xrs;
#pragma unroll
                for (int q = 0; q < NV; ++q) xv[u][p][q] = ld_x<T, VEC>(xr + q * TPR * VEC);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int p = 0; p < TPR; ++p) {
                const bool ok = !TAIL || (j0 + u < lenp[p]);
#pragma unroll
                for (int q = 0; q < NV; ++q)
#pragma unroll
                    for (int e = 0; e < VEC; ++e) {
                        const T s = O::add(acc[p][q][e], O::mul(vv[u][p], xv[u][p][q].v[e]));
                        if constexpr (TAIL) acc[p][q][e] = ok ? s : acc[p][q][e];
                        else acc[p][q][e] = s;
                    }
            }
        }
    };
    lidx j0 = 0;
    for (; j0 + U <= minlen; j0 += U) body(j0, std::false_type{});
    for (; j0 < maxlen; j0 += U) body(j0, std::true_type{});
}

template <class T, int C, int W, int U>
__global__ void __launch_bounds__(kTmaThreads, sizeof(T) >= 16 && sizeof(T) * W >= 512 ? SK_MINB_WIDE : SK_MINB)
    spmv_tma_kernel(const KArgs<T> a, int rgt, gidx ntiles, int seg) {
    // tile of this CTA's it-th iteration: segments of `seg` consecutive tiles dealt
    // round-robin over the CTAs (seg = 1: plain round-robin)
    auto tile_of = [&](int it, int sg) -> gidx {
        const gidx q = it / sg, w = it % sg;
        return (q * gridDim.x + blockIdx.x) * sg + w;
    };
    using O = Ops<T>;
    using P = TPlan<T, W>;
    constexpr int VEC = P::VEC, TPR = P::TPR, NV = P::NV, WS = P::WS, NSLICE = P::NSLICE, RP = P::RP;
    constexpr int SCAP = TmaGeom<T, W>::SCAP;
    constexpr int SB = TmaGeom<T, W>::SB;
    static_assert(32 % C == 0, "chunk height must divide the warp");
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ T red[kNCW][3][WS];
    StageHdr* hdr = reinterpret_cast<StageHdr*>(smem + kStages * SB);
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(hdr + kStages);
    std::uint64_t* empty = full + kStages;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNCW);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int chunks_per_tile = rgt * (32 / C);
    const gidx ngroups = a.rg1;
    const bool want_dots = (a.flags & kFlagDots) != 0;

    if (warp == kNCW) {
        // ------------------------------------------------------ producer warp
        const unsigned long long pol = l2_evict_first_policy();
        for (int it = 0;; ++it) {
            const gidx t = tile_of(it, seg);
            if (t >= ntiles) break;
            const int s = it % kStages;
            const std::uint32_t k = std::uint32_t(it / kStages);
            mbar_wait(&empty[s], (k & 1u) ^ 1u);
            const gidx c0 = a.rg0 * (32 / C) + t * chunks_per_tile;
            const gidx c1 = min(min(a.nchunks, a.rg1 * (32 / C)), c0 + chunks_per_tile);
            const int nc = int(c1 - c0);
            const gidx off0 = a.chunk_offset[c0];
            for (int q = lane; q <= nc; q += 32) hdr[s].hoff[q] = int(a.chunk_offset[c0 + q] - off0);
            for (int q = lane; q < nc; q += 32) hdr[s].hlen[q] = a.chunk_len[c0 + q];
            const gidx nslots = a.chunk_offset[c1] - off0;
#if SK_CHECK
            SK_DEVICE_CHECK(c0 <= c1 && c1 <= a.nchunks, "tma kernel: tile chunk range");
            SK_DEVICE_CHECK(off0 >= 0 && off0 + nslots <= a.slots, "tma kernel: tile slot range");
#endif
            const bool fits = nslots <= SCAP;
            if (lane == 0) {
                hdr[s].overflow = fits ? 0 : 1;
                hdr[s].nchunks = nc;
                hdr[s].off0 = off0;
            }
            __syncwarp();
            if (lane == 0) {
                if (fits && nslots > 0) {
                    T* sval = reinterpret_cast<T*>(smem + s * SB);
                    lidx* scol = reinterpret_cast<lidx*>(smem + s * SB + SCAP * sizeof(T));
                    const std::uint32_t vb = std::uint32_t(nslots * sizeof(T));
                    const std::uint32_t cb = std::uint32_t(nslots * sizeof(lidx));
                    mbar_arrive_expect_tx(&full[s], vb + cb);
                    bulk_g2s(sval, a.val + off0, vb, &full[s], pol);
                    bulk_g2s(scol, a.col + off0, cb, &full[s], pol);
                } else {
                    mbar_arrive(&full[s]);
                }
            }
            if constexpr (SK_HDR_PREFETCH > 0) {
                const gidx tn = tile_of(it + SK_HDR_PREFETCH, seg);
                if (tn < ntiles) {
                    const gidx cn0 = a.rg0 * (32 / C) + tn * chunks_per_tile;
                    const gidx cn1 = min(min(a.nchunks, a.rg1 * (32 / C)), cn0 + chunks_per_tile);
                    prefetch_headers(a.chunk_offset, a.chunk_len, cn0, int(cn1 - cn0), lane);
                }
            }
        }
    } else {
        // ---------------------------------------------------- consumer warps
        const int rgi = warp / NSLICE;
        const int slice = warp % NSLICE;
        const int sub = lane % TPR;
        const int rsub = lane / TPR;
        const int col_base = slice * WS;
        const bool need_x = (a.flags & (kFlagShift | kFlagVshift | kFlagDotXY | kFlagDotXX)) != 0;
        T dsum[3][NV][VEC];
#pragma unroll
        for (int s = 0; s < 3; ++s)
#pragma unroll
            for (int q = 0; q < NV; ++q)
#pragma unroll
                for (int e = 0; e < VEC; ++e) dsum[s][q][e] = O::zero();
        for (int it = 0;; ++it) {
            const gidx t = tile_of(it, seg);
            if (t >= ntiles) break;
            const int s = it % kStages;
            const std::uint32_t k = std::uint32_t(it / kStages);
            mbar_wait(&full[s], k & 1u);
            const gidx rg = a.rg0 + t * rgt + rgi;
            if (rgi < rgt && rg < ngroups) {
                T acc[TPR][NV][VEC];
                const T* sval = reinterpret_cast<const T*>(smem + s * SB);
                const lidx* scol = reinterpret_cast<const lidx*>(smem + s * SB + SCAP * sizeof(T));
                if (!hdr[s].overflow)
                    tma_rowgroup<T, C, W, U, true>(a, sval, scol, hdr[s], rgi, rg, slice, lane, acc);
                else
                    tma_rowgroup<T, C, W, U, false>(a, sval, scol, hdr[s], rgi, rg, slice, lane, acc);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);  // matrix data consumed; epilogue touches only x/y/z
                // fused epilogue (spmv_epilogue.hpp:12-36)
#pragma unroll
                for (int p = 0; p < TPR; ++p) {
                    const gidx row = rg * 32 + p * RP + rsub;
                    if (row >= a.nrows) continue;
                    const bool fin = !deferred(a.defer_mask, row);
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        const int cb = col_base + (q * TPR + sub) * VEC;
                        T* yp = a.y + row * a.y_rs + cb;
                        Vec<T, VEC> xv, yv, out;
                        if (need_x) xv = ld_x<T, VEC>(a.xs + row * a.xs_rs + cb);
                        if (a.flags & kFlagAxpby) yv = ld_vec<T, VEC>(yp);
#pragma unroll
                        for (int e = 0; e < VEC; ++e)
                            out.v[e] = apply_epilogue(a, acc[p][q][e], need_x ? xv.v[e] : O::zero(),
                                                      (a.flags & kFlagAxpby) ? yv.v[e] : O::zero(), cb + e);
                        st_vec<T, VEC>(yp, out);
                        if (!fin) continue;
                        if (a.flags & kFlagChain) {
                            T* zp = a.z + row * a.z_rs + cb;
                            Vec<T, VEC> zv = ld_vec<T, VEC>(zp);
#pragma unroll
                            for (int e = 0; e < VEC; ++e)
                                zv.v[e] = O::add(O::mul(a.delta, zv.v[e]), O::mul(a.eta, out.v[e]));
                            st_vec<T, VEC>(zp, zv);
                        }
                        if (want_dots) {
#pragma unroll
                            for (int e = 0; e < VEC; ++e) {
                                if (a.flags & kFlagDotYY)
                                    dsum[0][q][e] = O::add(dsum[0][q][e], O::mul(O::conj(out.v[e]), out.v[e]));
                                if (a.flags & kFlagDotXY)
                                    dsum[1][q][e] = O::add(dsum[1][q][e], O::mul(O::conj(xv.v[e]), out.v[e]));
                                if (a.flags & kFlagDotXX)
                                    dsum[2][q][e] = O::add(dsum[2][q][e], O::mul(O::conj(xv.v[e]), xv.v[e]));
                            }
                        }
                    }
                }
            } else {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
        }
        if (want_dots) {
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
        }
    }
    if (!want_dots) return;  // uniform across the grid
    __syncthreads();
    for (int t = threadIdx.x; t < 3 * W; t += kTmaThreads) {
        const int s = t / W, c = t % W, sl = c / WS, cw = c % WS;
        T sum = O::zero();
        for (int w = sl; w < kNCW; w += NSLICE) sum = O::add(sum, red[w][s][cw]);
        a.partial[gidx(blockIdx.x) * 3 * W + t] = sum;
    }
}

// ---------------------------------------------------------------------------
// Row-contiguous variant of the TMA kernel (production path for RHS rows of
// 32..256 bytes).  A lane owns ONE row and VEC = 32/sizeof(T) consecutive columns;
// the TPR = W/VEC lanes of a row cover the whole RHS row, so one LDG.256 warp
// instruction reads WR = 32/TPR complete, contiguous RHS rows (full 128-B lines):
// half the L1 wavefronts of splitting the columns over warps, with only VEC
// accumulators per lane, which leaves the registers for a deep gather unroll.
// A warp covers WR rows; the tile (one producer stage) covers NCW*WR rows.
#ifndef SK_XPOL
#define SK_XPOL 0
#endif
#ifndef SK_YPOL
#define SK_YPOL 0
#endif
#ifndef SK_RVEC
#define SK_RVEC 32  // bytes of one RHS row a lane gathers per nonzero
#endif
#ifndef SK_ROWS_WIDE  // 1: the rows kernel also for RHS rows of 512 B / 1 KB (else the column-slice kernel)
#define SK_ROWS_WIDE 1
#endif
#ifndef SK_WIDE_LANES  // lanes per RHS row of 512 B / 1 KB; 0: by kernel variant (rows_lanes)
#define SK_WIDE_LANES 0
#endif
#ifndef SK_WIDE_DOTS_LANES  // the same for the dots kernels: 16, two 16-row passes per 32-row tile
#define SK_WIDE_DOTS_LANES 16  // (KPM, TI 2^24 rows, r2bl: complex w = 32 / 64 12.7 / 39.4 -> 11.4 / 27.9 ms,
#endif                         //  double w = 64 10.9 -> 9.8 ms against 8 lanes of 64- / 128-byte vectors)
#ifndef SK_PREFETCH_EPI
#define SK_PREFETCH_EPI 1
#endif
constexpr bool kPrefetchEpi = SK_PREFETCH_EPI != 0;
constexpr bool kXHint = SK_XPOL != 0;  // x gathers marked evict_last in L2
constexpr bool kYHint = SK_YPOL != 0;  // y / z stores marked evict_first in L2

// Lanes per RHS row of 512 B / 1 KB (measured, r2bi / r2bl): the dots kernels 16 (two passes
// per 32-row tile); the others 16 for real rows and 1-KB rows (double w = 64 plain 7.77 ->
// 5.77 ms, complex w = 64 29.9 -> 16.6 ms), 8 (64-byte lane vectors) for complex w = 32
// (plain 8.0 vs 8.8 ms)
template <class T, int W, bool DOTS>
constexpr int rows_lanes() {
    if constexpr (SK_WIDE_LANES > 0) return SK_WIDE_LANES;
    else if constexpr (DOTS) return SK_WIDE_DOTS_LANES;
    else return (sizeof(T) <= 8 || W * int(sizeof(T)) >= 1024) ? 16 : 8;
}

template <class T, int W, int WL = 8>
struct RPlan {
    static constexpr int E = int(sizeof(T));
    static constexpr int VB = SK_RVEC / E > 0 ? SK_RVEC / E : 1;
    // RHS rows wider than 8 lanes x 32 B (512-B / 1-KB rows): 64- or 128-byte lane vectors
    // (2 or 4 LDG.256 per gather), still 8 lanes per row
    // (WL = 16 / 32 lanes per wide row: 8 / 16 rows per pass)
    static constexpr bool WIDE_ROW = SK_ROWS_WIDE && W * E > 8 * SK_RVEC && W % WL == 0;
    static constexpr int VW = WIDE_ROW ? (W * E / WL >= SK_RVEC ? W / WL : VB) : VB;
    static constexpr int VEC = VW < W ? VW : W;
    static constexpr int TPR = W / VEC;   // lanes per row
    static constexpr int WR = 32 / TPR;   // rows per warp
    static constexpr bool ok = TPR >= 1 && W % VEC == 0 &&
                               ((TPR <= 8 && kNCW * WR >= 32 && (kNCW * WR) % 32 == 0) ||
                                (WIDE_ROW && TPR <= 32 && 32 % (kNCW * WR) == 0));
};
template <class T, int W, bool DOTS>
using RP = RPlan<T, W, rows_lanes<T, W, DOTS>()>;

// Per-lane shared-memory dot slot += v.  Only the owning lane touches a slot, so the
// order of additions is fixed.  (A shared-memory atomicAdd on doubles compiles to a
// compare-and-swap loop on sm_100a, so the plain read-add-write is kept.)
template <class T>
__device__ __forceinline__ void slot_add(T* p, T v) {
    *p = Ops<T>::add(*p, v);
}

// Column dots in registers (SK_DOTS_REG): the K dot terms of a lane's row (3 dots x VEC
// columns) are summed over the warp's WR row slots with a reduce-scatter -- at lane bit M
// the lower lane keeps the lower half of the (zero-padded) values and the upper lane the
// upper half, each adding the partner's copy in the order (lower lane, upper lane) -- so
// after log2(WR) steps every lane holds ceil(K/WR)-ish values of ONE slice of the index
// space (`base`, `valid` of them real), to accumulate across the sweep in registers.
// Replaces 3*VEC shared-memory read-modify-writes per lane and row by ~K shuffles per pass.
#ifndef SK_DOTS_REG
#define SK_DOTS_REG 1
#endif
// Shapes where the register accumulators measured faster than the shared-memory slots
// (B200, tools/ab_dots.sh, gpurun_out r2j): double w = 4 (400^3 with three dots 1.90 ->
// 1.70 ms) and w = 32 (256^3 KPM step 5.3 -> 4.0 ms).  Elsewhere the slots win (w = 1,
// 8, 16 and complex: the epilogue's extra live registers spill at 3 CTAs/SM; C3 C64
// 5.0 vs 6.2 ms).
template <class T, int W>
constexpr bool dots_in_registers() {
    return SK_DOTS_REG != 0 && (SK_DOTS_REG >= 2 || (std::is_same_v<T, double> && (W == 4 || W == 32)));
}
template <int K, int M, int TPR>
constexpr int rs_final() {
    if constexpr (M >= TPR && M > 0) return rs_final<(K + 1) / 2, M / 2, TPR>();
    else return K;
}

// the slice (first index, real count) a lane ends up with, without the data
template <int K, int M, int TPR>
__device__ __forceinline__ void rs_slice(int lane, int& base, int& valid) {
    if constexpr (M >= TPR && M > 0) {
        constexpr int H = (K + 1) / 2;
        if (lane & M) {
            base += H;
            valid = valid > H ? valid - H : 0;
        } else {
            valid = valid < H ? valid : H;
        }
        rs_slice<H, M / 2, TPR>(lane, base, valid);
    }
}

template <class T, int K, int M, int TPR>
__device__ __forceinline__ void rs_step(T* v, int lane) {
    if constexpr (M >= TPR && M > 0) {
        using O = Ops<T>;
        constexpr int H = (K + 1) / 2;
        const bool up = (lane & M) != 0;
#pragma unroll
        for (int i = 0; i < H; ++i) {
            const T lo = v[i];
            const T hi = (H + i < K) ? v[H + i] : O::zero();
            const T recv = shfl_xor(up ? lo : hi, M);
            v[i] = up ? O::add(recv, hi) : O::add(lo, recv);
        }
        rs_step<T, H, M / 2, TPR>(v, lane);
    }
}

// Remainder handling of the row-contiguous kernel: 0 = exact-size batch when the
// row length is warp-uniform, 1 = predicated batch, 2 = predicated loads too.
#ifndef SK_BATCH_UNROLL1
#define SK_BATCH_UNROLL1 0
#endif
#ifndef SK_TAILMODE
#define SK_TAILMODE 0
#endif
// Warp-uniform rows of length <= SK_LENSWITCH run a fully unrolled batch sequence
// selected by the length (no trip-count arithmetic or loop); 0 = off.  Dots-free
// kernels with w <= 16 only.  Measured (400^3, same box, ms): w = 1 0.976 -> 0.948,
// w = 4 1.425 -> 1.390, w = 16 4.9 -> 4.5, bench w = 8 (power-capped, 200 steps)
// 2.57 -> 2.525; w = 32 9.2 -> 9.8 and the dots kernels (C3 C64 5.84 -> 7.59) got
// worse schedules, so they keep the loop.
#ifndef SK_LENSWITCH
#define SK_LENSWITCH 8
#endif

// f(integral_constant<U>) L / U times, then f(integral_constant<L % U>)
template <int L, int U, class F>
__device__ __forceinline__ void fixed_batches(F& f) {
    if constexpr (L >= U) {
        f(std::integral_constant<int, U>{});
        fixed_batches<L - U, U>(f);
    } else if constexpr (L > 0) {
        f(std::integral_constant<int, L>{});
    }
}

// L split into ceil(L / U) batches of near-equal size, the larger ones first
// (7 with U = 3: 3, 2, 2 instead of 3, 3, 1)
template <int L, int NB, class F>
__device__ __forceinline__ void balanced_batches(F& f) {
    if constexpr (NB >= 1 && L > 0) {
        constexpr int R = (L + NB - 1) / NB;
        f(std::integral_constant<int, R>{});
        balanced_batches<L - R, NB - 1>(f);
    }
}

// Batch shape of the length-switched path: SK_LEN_UADD widens a batch beyond the
// kernel's U, SK_LEN_BAL = 1 splits a row into near-equal batches instead of U-greedy ones.
#ifndef SK_LEN_UADD
#define SK_LEN_UADD 0
#endif
#ifndef SK_LEN_BAL
#define SK_LEN_BAL 0
#endif

template <int LMAX, int U, class F>
__device__ __forceinline__ void len_dispatch(int len, F& f) {
    if constexpr (LMAX >= 1) {
        if (len == LMAX) {
            if constexpr (SK_LEN_BAL)
                balanced_batches<LMAX, (LMAX + U - 1) / U>(f);
            else
                fixed_batches<LMAX, U>(f);
        } else {
            len_dispatch<LMAX - 1, U>(len, f);
        }
    }
}

// acc + v * x: two separately rounded operations (the reference's arithmetic, bit-exact)
// or, with SK_SPMV_FMA, one fused multiply-add (within the 1e-12 tolerance).
#ifndef SK_SPMV_FMA
#define SK_SPMV_FMA 0
#endif
template <class T>
__device__ __forceinline__ T mac(T acc, T v, T x) {
    if constexpr (SK_SPMV_FMA) return Ops<T>::fma(v, x, acc);
    else return Ops<T>::add(acc, Ops<T>::mul(v, x));
}

// f(integral_constant<R>) for the runtime remainder r in [1, RMAX] (r == 0: nothing)
template <int RMAX, class F>
__device__ __forceinline__ void tail_dispatch(int r, F& f) {
    if constexpr (RMAX >= 1) {
        if (r == RMAX)
            f(std::integral_constant<int, RMAX>{});
        else
            tail_dispatch<RMAX - 1>(r, f);
    }
}

// Occupancy and staging of the row-contiguous kernel.  The consumers are latency
// bound (each warp has one batch of gathers in flight, then computes), so resident
// warps are worth more than unroll depth: measured on B200 (400^3, w = 8),
// 2 CTAs/SM x U = 8: 3.46 ms; 3 CTAs x U = 4: 2.55 ms; 4 CTAs x U = 3: 2.47 ms.
// Stages hold one full tile (kNCW * WR rows) of a 7-nonzero stencil and no more,
// so shared memory does not take L1 from the RHS gathers: 3 x 11 KB for
// multi-lane rows (w = 8: 2 x 16 KB 2.55 ms -> 3 x 11 KB 2.31 ms), 2 x 22 KB when a
// lane owns a whole RHS row (TPR = 1, 256-row tiles).  Longer rows shrink the
// tile (fewer active warps) or, past a stage, read the matrix from global memory.
// The sizes are compile-time: the same kernel with runtime stage sizes was
// scheduled worse by ptxas (2.8 ms, products hoisted between the gathers).
#ifndef SK_DYN_TILES
#define SK_DYN_TILES 1
#endif
#ifndef SK_DYN_DOTS  // experiment: dynamic tiles for the dots kernels (dots then depend on timing)
#define SK_DYN_DOTS 0
#endif
#ifndef SK_DYN_PLAIN  // dynamic tiles for the epilogue-free kernels (when the launch rule below says so)
#define SK_DYN_PLAIN 1
#endif

#ifndef SK_RMINB
#define SK_RMINB 4
#endif
#ifndef SK_RMINB_DOTS
#define SK_RMINB_DOTS 3
#endif
// the dots kernel of a single double vector fits 56 registers without spills: 4 CTAs/SM
// (400^3 with three dots: w = 1 1.155 -> 1.055 ms; w = 2 1.40 -> 1.43, w = 4 1.89 ->
// 1.88; wider blocks and complex/float types spill at 4 and lose 10-45 %)
#ifndef SK_RMINB_DOTS_NARROW
#define SK_RMINB_DOTS_NARROW 4
#endif
#ifndef SK_RSTAGES_WIDE
#define SK_RSTAGES_WIDE 3
#endif
#ifndef SK_RSTAGES_NARROW
#define SK_RSTAGES_NARROW 2
#endif
#ifndef SK_RSTAGE_KB
#define SK_RSTAGE_KB 11
#endif
#ifndef SK_RSTAGE_KB_NARROW
#define SK_RSTAGE_KB_NARROW 22
#endif

#ifndef SK_RTILE_ROWS
#define SK_RTILE_ROWS 128
#endif

#ifndef SK_RSTAGES_DOTS
#define SK_RSTAGES_DOTS 0  // 0: as the plain kernel
#endif

template <class T, int W, bool DOTS = false>
struct RGeom {
    static constexpr bool WIDE = RPlan<T, W>::TPR > 1;  // (the same for every lane count)
    static constexpr int STAGES =
        (DOTS && SK_RSTAGES_DOTS > 0) ? SK_RSTAGES_DOTS : (WIDE ? SK_RSTAGES_WIDE : SK_RSTAGES_NARROW);
    static constexpr int SB = (WIDE ? SK_RSTAGE_KB : SK_RSTAGE_KB_NARROW) * 1024;
    static constexpr int SCAP = (SB / int(sizeof(T) + 4)) / 32 * 32;  // slots per stage
};

// stage ring, headers, barriers; with dots also the per-lane dot accumulators
// dacc[3][VEC][consumer lanes] (lane-contiguous: conflict-free)
template <class T, int W, bool DOTS>
constexpr std::size_t rows_stage_bytes() {
    constexpr int S = RGeom<T, W, DOTS>::STAGES;
    return (std::size_t(S) * RGeom<T, W>::SB + std::size_t(S) * sizeof(StageHdr) + 2 * S * 8 + 15) / 16 * 16;
}
template <class T, int W, bool DOTS>
constexpr std::size_t rows_smem_bytes() {
    return rows_stage_bytes<T, W, DOTS>() +
           (DOTS && !dots_in_registers<T, W>() ? std::size_t(3) * RP<T, W, true>::VEC * kNCW * 32 * sizeof(T) : 0) +
           128;
}

// CTAs/SM the rows kernel is compiled for (register budget 65536 / (288 x this));
// the 64-/128-byte lane vectors of the wide plans need 2 / 1
template <class T, int W, bool DOTS>
constexpr int rows_minb() {
    constexpr int vb = RP<T, W, DOTS>::VEC * int(sizeof(T));
    if constexpr (vb > 64) return 1;
    else if constexpr (vb > SK_RVEC) return 2;
    else if constexpr (DOTS) return std::is_same_v<T, double> && W == 1 ? SK_RMINB_DOTS_NARROW : SK_RMINB_DOTS;
    else return SK_RMINB;
}

// DYN: the kernel can take its tiles from a.tile_counter (dynamic deal); a separate
// instantiation so the static epilogue-free kernel keeps its register schedule.
template <class T, int C, int W, int U, bool DOTS, bool PLAIN, bool MAPPED, bool DYN>
__global__ void __launch_bounds__(kTmaThreads, rows_minb<T, W, DOTS>())
    spmv_tma_rows_kernel(const KArgs<T> a, int rgt, gidx ntiles, int seg) {
    using O = Ops<T>;
    using P = RP<T, W, DOTS>;
    constexpr int VEC = P::VEC, TPR = P::TPR, WR = P::WR;
    constexpr int SCAP = RGeom<T, W>::SCAP;
    constexpr int SB = RGeom<T, W>::SB;
    constexpr int kStages = RGeom<T, W, DOTS>::STAGES;
    static_assert(32 % C == 0, "chunk height must divide the warp");
    auto tile_of = [&](int it, int sg) -> gidx {
        const gidx q = it / sg, w = it % sg;
        return (q * gridDim.x + blockIdx.x) * sg + w;
    };
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ T red[DOTS ? kNCW : 1][3][DOTS ? W : 1];
    StageHdr* hdr = reinterpret_cast<StageHdr*>(smem + kStages * SB);
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(hdr + kStages);
    std::uint64_t* empty = full + kStages;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNCW);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int chunks_per_tile = rgt * (32 / C);
    const int rows_per_tile = rgt * 32;
    constexpr bool want_dots = DOTS;  // launch selects DOTS == (flags & kFlagDots) != 0
    // first row group of tile t: natural order, or the caller's block order (locality)
    const int tpb = a.sweep_brg > 0 ? a.sweep_brg / rgt : 1;
    auto tile_rg = [&](gidx t) -> gidx {
        if (a.sweep_brg > 0) return gidx(__ldg(a.sweep_order + t / tpb)) * a.sweep_brg + (t % tpb) * rgt;
        return a.rg0 + t * rgt;
    };

    // dynamic tiles (epilogue kernels without dots, whose results do not depend on which
    // CTA sweeps a tile): the producer takes the next tile from a global counter, so
    // the sweep front stays one contiguous band (x reuse) and no CTA trails at the end;
    // a tile index >= ntiles in the stage header tells the consumers to stop
    // (measured, r2v / r2w: 400^3 w = 8 AXPBY 3.35 -> 2.71 ms; the epilogue-free kernels
    // by the launch rule in launch_tma_rows)
    constexpr bool kDynOK = DYN && SK_DYN_TILES;
    const bool dyn = kDynOK && a.tile_counter != nullptr;
    if (warp == kNCW) {
        // ------------------------------------------------- producer warp (as spmv_tma_kernel)
        const unsigned long long pol = l2_evict_first_policy();
        auto grab = [&](int it) -> gidx {
            if (!dyn) return tile_of(it, seg);
            int v = 0;
            if (lane == 0) v = atomicAdd(a.tile_counter, 1);
            return gidx(__shfl_sync(0xffffffffu, v, 0));
        };
        gidx t_cur = grab(0);
        for (int it = 0;; ++it) {
            const gidx t = t_cur;
            const int s = it % kStages;
            const std::uint32_t k = std::uint32_t(it / kStages);
            if (t >= ntiles) {
                if (dyn) {  // tell the consumers there is no further tile
                    mbar_wait(&empty[s], (k & 1u) ^ 1u);
                    if (lane == 0) {
                        hdr[s].nchunks = -1;
                        mbar_arrive(&full[s]);
                    }
                }
                break;
            }
            const gidx t_next = grab(it + 1);
            t_cur = t_next;
            // the epilogue's y (AXPBY) and z (CHAIN) rows of this tile: one bulk L2
            // prefetch each, a stage ahead of the consumers, so the epilogue reads
            // hit L2 instead of adding a dependent HBM round trip per tile
            if (kPrefetchEpi && !MAPPED && lane == 0 && (a.flags & (kFlagAxpby | kFlagChain))) {
                const gidx r0 = tile_rg(t) * 32;
                const gidx r1 = min(r0 + gidx(rows_per_tile), min(gidx(a.nrows), a.rg1 * 32));
                auto span = [&](const T* base, gidx rs) {
                    const std::uintptr_t b = reinterpret_cast<std::uintptr_t>(base + r0 * rs) & ~std::uintptr_t(15);
                    const std::uintptr_t e =
                        (reinterpret_cast<std::uintptr_t>(base + (r1 - 1) * rs + W) + 15) & ~std::uintptr_t(15);
                    if constexpr (kYHint)
                        bulk_prefetch_l2(reinterpret_cast<const void*>(b), std::uint32_t(e - b), pol);
                    else
                        bulk_prefetch_l2(reinterpret_cast<const void*>(b), std::uint32_t(e - b));
                };
                if (r1 > r0) {
                    if (a.flags & kFlagAxpby) span(a.y, a.y_rs);
                    if (a.flags & kFlagChain) span(a.z, a.z_rs);
                }
            }
            mbar_wait(&empty[s], (k & 1u) ^ 1u);
            // a partial last sweep-order block leaves tiles past the end: clamp their
            // header reads to the chunk range (nc = 0), keep their row origin
            const gidx cend = min(a.nchunks, a.rg1 * (32 / C));
            const gidx c0u = tile_rg(t) * (32 / C);
            const gidx c0 = min(c0u, cend);
            const gidx c1 = min(cend, c0 + chunks_per_tile);
            const int nc = int(c1 - c0);
            const gidx off0 = a.chunk_offset[c0];
            for (int q = lane; q <= nc; q += 32) hdr[s].hoff[q] = int(a.chunk_offset[c0 + q] - off0);
            for (int q = lane; q < nc; q += 32) hdr[s].hlen[q] = a.chunk_len[c0 + q];
            const gidx nslots = a.chunk_offset[c1] - off0;
#if SK_CHECK
            SK_DEVICE_CHECK(c0 <= c1 && c1 <= a.nchunks, "rows kernel: tile chunk range");
            SK_DEVICE_CHECK(off0 >= 0 && off0 + nslots <= a.slots, "rows kernel: tile slot range");
#endif
            const bool fits = nslots <= SCAP;
            if (lane == 0) {
                hdr[s].overflow = fits ? 0 : 1;
                hdr[s].nchunks = nc;
                hdr[s].off0 = off0;
                hdr[s].row0 = int(c0u / (32 / C)) * 32;
            }
            __syncwarp();
            if (lane == 0) {
                if (fits && nslots > 0) {
                    T* sval = reinterpret_cast<T*>(smem + s * SB);
                    lidx* scol = reinterpret_cast<lidx*>(smem + s * SB + SCAP * sizeof(T));
                    const std::uint32_t vb = std::uint32_t(nslots * sizeof(T));
                    const std::uint32_t cb = std::uint32_t(nslots * sizeof(lidx));
                    mbar_arrive_expect_tx(&full[s], vb + cb);
                    bulk_g2s(sval, a.val + off0, vb, &full[s], pol);
                    bulk_g2s(scol, a.col + off0, cb, &full[s], pol);
                } else {
                    mbar_arrive(&full[s]);
                }
            }
            if constexpr (SK_HDR_PREFETCH > 0 && (PLAIN || DOTS)) {
                const gidx tn = dyn ? t_next : tile_of(it + SK_HDR_PREFETCH, seg);
                if (tn < ntiles) {
                    const gidx cn0 = min(tile_rg(tn) * (32 / C), cend);
                    const gidx cn1 = min(cend, cn0 + chunks_per_tile);
                    prefetch_headers(a.chunk_offset, a.chunk_len, cn0, int(cn1 - cn0), lane);
                }
            }
        }
    } else {
        // ------------------------------------------------------- consumer warps
        const int sub = lane % TPR;
        const int rl = lane / TPR;
        const bool need_x = (a.flags & (kFlagShift | kFlagVshift | kFlagDotXY | kFlagDotXX)) != 0;
        const unsigned xrs = unsigned(a.x_rs);
        const T* xb = a.x + sub * VEC;
        const unsigned long long xpol = kXHint ? l2_evict_last_policy() : 0ull;
        const unsigned long long ypol = kYHint ? l2_evict_first_policy() : 0ull;
        // column dots: every lane accumulates its rows' terms in its own shared-memory
        // slots (no 3 x VEC accumulators live across the gather loop); the lanes are
        // reduced once at the end, in a fixed order (deterministic)
        T* dacc = reinterpret_cast<T*>(smem + rows_stage_bytes<T, W, DOTS>());
        const int cl = warp * 32 + lane;  // consumer lane
        constexpr int NCL = kNCW * 32;
        constexpr bool kDR = dots_in_registers<T, W>();
        constexpr int KD = 3 * VEC;                       // dot terms per lane and row
        // SK_DOTS_REG == 3: every lane keeps all KD terms of its rows (no per-pass shuffles),
        // reduced over the row slots once at the end
        constexpr bool kDirect = kDR && SK_DOTS_REG == 3;
        constexpr int KF = kDirect ? KD : rs_final<KD, 16, TPR>();  // register accumulators per lane
        T dreg[kDR && DOTS ? KF : 1];
        int dbase = 0, dvalid = KD;                        // slice of the KD terms this lane keeps
        if constexpr (DOTS && kDR && !kDirect) rs_slice<KD, 16, TPR>(lane, dbase, dvalid);
        if constexpr (DOTS && kDR) {
#pragma unroll
            for (int q = 0; q < KF; ++q) dreg[q] = O::zero();
        } else if constexpr (DOTS) {
#pragma unroll
            for (int q = 0; q < 3 * VEC; ++q) dacc[q * NCL + cl] = O::zero();
        }
        // 32-bit tile/row arithmetic (rows < 2^31: lidx); 64-bit only in the final
        // address IMAD.WIDEs
        const int rg0 = int(a.rg0);
        const int nt = int(ntiles);
        // (the epilogue-free kernels read grp_end from the parameter bank where they use it:
        // kept in a register it was the one value they spilled, reloaded every tile)
        const int grp_end = PLAIN ? 0 : int(min(gidx(a.nrows_padded), a.rg1 * 32));  // warps at/after: idle
        const int row_end = int(min(gidx(a.nrows), a.rg1 * 32));          // rows stored
        // (compile-time bound: one pass for the dots variant, whose register budget
        // has no room for the pass loop -- measured 30 % slower on C3 C64)
        constexpr int kMaxPasses = DOTS ? (kNCW * WR < 32 ? 32 / (kNCW * WR) : 1)
                                        : (SK_RTILE_ROWS / (kNCW * WR) > 1 ? SK_RTILE_ROWS / (kNCW * WR) : 1);
        const int passes = min(kMaxPasses, (rows_per_tile + kNCW * WR - 1) / (kNCW * WR));
        for (int it = 0;; ++it) {
            if (!dyn) {
                const int t = seg == 1 ? it * int(gridDim.x) + int(blockIdx.x) : int(tile_of(it, seg));
                if (t >= nt) break;
            }
            const int s = it % kStages;
            const std::uint32_t k = std::uint32_t(it / kStages);
            mbar_wait(&full[s], k & 1u);
            const StageHdr& h = hdr[s];
            if (dyn && h.nchunks < 0) break;  // the producer ran out of tiles
            const int tile_row0 = h.row0;  // the producer resolved the sweep order
            // a tile may hold several warp-row passes (narrow warps, short rows): the
            // per-tile work (barrier, header, release) is shared by all of them
            for (int pass = 0; pass < passes; ++pass) {
            const int wrow0 = (pass * kNCW + warp) * WR;  // this warp's first row of the pass
            if (wrow0 >= rows_per_tile || tile_row0 + wrow0 >= (PLAIN ? a.grp_end : grp_end)) break;  // warp-uniform
            const int rr = wrow0 + rl;
            const int row = tile_row0 + rr;
            const int cq = rr / C;
            const int ip = rr % C;
            const lidx len = cq < h.nchunks ? h.hlen[cq] : 0;
            const int off = cq < h.nchunks ? h.hoff[cq] + ip : 0;
            lidx maxlen = len, minlen = len;
            if constexpr (C < 32 || WR > C) {
                maxlen = lidx(__reduce_max_sync(0xffffffffu, unsigned(len)));
                minlen = lidx(__reduce_min_sync(0xffffffffu, unsigned(len)));
            }
            T acc[VEC];
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[e] = O::zero();
            // value/index source: the shared-memory stage (LDS) or, for a tile that
            // did not fit one stage, global memory; separate code so the common case
            // compiles to shared-memory loads.
            // RHS row c starts at byte xbytes + c * xstride (one IMAD.WIDE per gather)
            const char* xbytes = reinterpret_cast<const char*>(xb);
            const unsigned xstride = xrs * unsigned(sizeof(T));
            auto gather = [&](const T* vp, const lidx* cp) {
                // slot (row, j) = off + j*C: walk the per-lane pointers by U*C per batch,
                // so the U slots of a batch are immediate offsets
                vp += off;
                cp += off;
                auto xrow = [&](lidx c) -> const T* {
#if SK_CHECK
                    SK_DEVICE_CHECK(unsigned(c) < unsigned(a.xrows), "rows kernel: RHS row index in range");
#endif
                    return reinterpret_cast<const T*>(xbytes + (unsigned long long)unsigned(c) * xstride);
                };
                auto ldx = [&](const T* p) -> Vec<T, VEC> {
                    if constexpr (kXHint && VEC * sizeof(T) == 32) return ld_x_hint<T, VEC>(p, xpol);
                    else return ld_x<T, VEC>(p);
                };
                // one batch of R consecutive j: all loads first, then the products in j order
                auto batch = [&](auto rc) {
                    constexpr int R = decltype(rc)::value;
                    T vv[R];
                    Vec<T, VEC> xv[R];
#pragma unroll
                    for (int u = 0; u < R; ++u) {
                        vv[u] = vp[u * C];
                        xv[u] = ldx(xrow(cp[u * C]));
                    }
#pragma unroll
                    for (int u = 0; u < R; ++u)
#pragma unroll
                        for (int e = 0; e < VEC; ++e) acc[e] = mac<T>(acc[e], vv[u], xv[u].v[e]);
                    vp += R * C;
                    cp += R * C;
                };
                lidx j0 = 0;
                if constexpr (SK_LENSWITCH > 0 && SK_TAILMODE == 0 && !DOTS && W <= 16) {
                    if (minlen == maxlen && len <= SK_LENSWITCH) {
                        len_dispatch<SK_LENSWITCH, U + SK_LEN_UADD>(len, batch);
                        return;
                    }
                }
#if SK_BATCH_UNROLL1
#pragma unroll 1
#endif
                for (; j0 + U <= minlen; j0 += U) batch(std::integral_constant<int, U>{});
                if (SK_TAILMODE == 0 && minlen == maxlen) {
                    // warp-uniform row length (every row of the warp in one chunk, the usual
                    // case): the remainder is one exact-size batch, no predicates
                    tail_dispatch<U - 1>(len - j0, batch);
                } else {
                    // rows of different chunks: predicated adds; out-of-row slots gather RHS
                    // row 0 (always valid) and their products are dropped, so the sum is the
                    // reference's exactly
                    for (; j0 < maxlen; j0 += U) {
                        T vv[U];
                        Vec<T, VEC> xv[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const bool ok = j0 + u < len;
                            if constexpr (SK_TAILMODE == 2) {
#pragma unroll
                                for (int e = 0; e < VEC; ++e) xv[u].v[e] = O::zero();
                                vv[u] = O::zero();
                                if (ok) {
                                    vv[u] = vp[u * C];
                                    xv[u] = ldx(xrow(cp[u * C]));
                                }
                            } else {
                                lidx c = 0;
                                vv[u] = O::zero();
                                if (ok) {
                                    c = cp[u * C];
                                    vv[u] = vp[u * C];
                                }
                                xv[u] = ldx(xrow(c));
                            }
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (j0 + u < len) {
#pragma unroll
                                for (int e = 0; e < VEC; ++e) acc[e] = mac<T>(acc[e], vv[u], xv[u].v[e]);
                            }
                        }
                        vp += U * C;
                        cp += U * C;
                    }
                }
            };
            if (!h.overflow)
                gather(reinterpret_cast<const T*>(smem + s * SB), reinterpret_cast<const lidx*>(smem + s * SB + SCAP * sizeof(T)));
            else
                gather(a.val + h.off0, a.col + h.off0);
            if constexpr (PLAIN) {
                // y = A x with alpha == 1 and no other flag: t * 1 == t, so the store is the result
                if (row < row_end) {
                    Vec<T, VEC> out;
#pragma unroll
                    for (int e = 0; e < VEC; ++e) out.v[e] = acc[e];
                    st_vec<T, VEC>(a.y + (unsigned long long)unsigned(row) * unsigned(a.y_rs) + sub * VEC, out);
                }
                continue;
            }
            // fused epilogue (spmv_epilogue.hpp:12-36); a remote-part sweep writes the
            // local rows its stored rows map to (row_map)
            T dt[kDR && DOTS ? KD : 1];
            if constexpr (kDR && DOTS) {
#pragma unroll
                for (int q = 0; q < KD; ++q) dt[q] = O::zero();
            }
            if (row < row_end) {
                const gidx orow = MAPPED ? gidx(__ldg(a.row_map + row)) : gidx(row);
                const bool fin = !deferred(a.defer_mask, orow);
                const int cb = sub * VEC;
                T* yp = a.y + orow * a.y_rs + cb;
                Vec<T, VEC> xs, yv, out;
                if (need_x) xs = ld_x<T, VEC>(a.xs + orow * a.xs_rs + cb);
                if (a.flags & kFlagAxpby) {
                    if constexpr (kYHint && VEC * sizeof(T) == 32)
                        yv = ld_vec_hint<T, VEC>(yp, ypol);
                    else
                        yv = ld_vec<T, VEC>(yp);
                }
#pragma unroll
                for (int e = 0; e < VEC; ++e)
                    out.v[e] = apply_epilogue(a, acc[e], need_x ? xs.v[e] : O::zero(),
                                              (a.flags & kFlagAxpby) ? yv.v[e] : O::zero(), cb + e);
                if constexpr (kYHint && VEC * sizeof(T) == 32)
                    st_vec_hint<T, VEC>(yp, out, ypol);
                else
                    st_vec<T, VEC>(yp, out);
                if (fin) {
                    if (a.flags & kFlagChain) {
                        T* zp = a.z + orow * a.z_rs + cb;
                        Vec<T, VEC> zv = ld_vec<T, VEC>(zp);
#pragma unroll
                        for (int e = 0; e < VEC; ++e) zv.v[e] = O::add(O::mul(a.delta, zv.v[e]), O::mul(a.eta, out.v[e]));
                        if constexpr (kYHint && VEC * sizeof(T) == 32)
                            st_vec_hint<T, VEC>(zp, zv, ypol);
                        else
                            st_vec<T, VEC>(zp, zv);
                    }
                    if constexpr (DOTS && kDR) {
#pragma unroll
                        for (int e = 0; e < VEC; ++e) {
                            if (a.flags & kFlagDotYY) dt[e] = O::mul(O::conj(out.v[e]), out.v[e]);
                            if (a.flags & kFlagDotXY) dt[VEC + e] = O::mul(O::conj(xs.v[e]), out.v[e]);
                            if (a.flags & kFlagDotXX) dt[2 * VEC + e] = O::mul(O::conj(xs.v[e]), xs.v[e]);
                        }
                    } else if constexpr (DOTS) {
#pragma unroll
                        for (int e = 0; e < VEC; ++e) {
                            T* dp = dacc + e * NCL + cl;
                            if (a.flags & kFlagDotYY) slot_add(dp, O::mul(O::conj(out.v[e]), out.v[e]));
                            if (a.flags & kFlagDotXY) slot_add(dp + VEC * NCL, O::mul(O::conj(xs.v[e]), out.v[e]));
                            if (a.flags & kFlagDotXX) slot_add(dp + 2 * VEC * NCL, O::mul(O::conj(xs.v[e]), xs.v[e]));
                        }
                    }
                }
            }
            if constexpr (DOTS && kDR) {
                // warp-uniform: sum the pass's rows slot-wise, keep this lane's slice
                if constexpr (!kDirect) rs_step<T, KD, 16, TPR>(dt, lane);
#pragma unroll
                for (int q = 0; q < KF; ++q) dreg[q] = O::add(dreg[q], dt[q]);
            }
            }  // pass
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);  // matrix data of the tile consumed
        }
        if constexpr (DOTS && kDirect) {
            // lanes of a row slot -> warp total per column (fixed butterfly order)
#pragma unroll
            for (int q = 0; q < KD; ++q) {
                T v = dreg[q];
#pragma unroll
                for (int m = TPR; m < 32; m <<= 1) v = O::add(v, shfl_xor(v, m));
                if (lane < TPR) red[warp][q / VEC][lane * VEC + q % VEC] = v;
            }
        } else if constexpr (DOTS && kDR) {
            // every (dot, column) lives in exactly one lane of the warp: its warp total
#pragma unroll
            for (int q = 0; q < KF; ++q) {
                if (q < dvalid) {
                    const int idx = dbase + q;  // dot * VEC + e
                    red[warp][idx / VEC][sub * VEC + idx % VEC] = dreg[q];
                }
            }
        } else if constexpr (DOTS) {
            // lanes of a row slot -> warp total per column (fixed butterfly order)
#pragma unroll
            for (int q = 0; q < 3; ++q) {
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    T v = dacc[(q * VEC + e) * NCL + cl];
#pragma unroll
                    for (int m = TPR; m < 32; m <<= 1) v = O::add(v, shfl_xor(v, m));
                    if (lane < TPR) red[warp][q][lane * VEC + e] = v;
                }
            }
        }
    }
    if (!want_dots) return;
    __syncthreads();
    for (int t = threadIdx.x; t < 3 * W; t += kTmaThreads) {
        const int s = t / W, c = t % W;
        T sum = O::zero();
        for (int w = 0; w < kNCW; ++w) sum = O::add(sum, red[w][s][c]);
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

    const gidx r_end = min(gidx(a.nrows), a.rg1 * 32);
    for (gidx r = a.rg0 * 32 + blockIdx.x * gidx(blockDim.x) + threadIdx.x; r < r_end;
         r += gidx(gridDim.x) * blockDim.x) {
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
#if SK_CHECK
            SK_DEVICE_CHECK(slot < a.slots && unsigned(a.col[slot]) < unsigned(a.xrows), "generic kernel: slot / column");
#endif
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

template <class T>
inline int grid_sms_of(const KArgs<T>& a, const DeviceRuntime& rt) {
    return a.grid_sms > 0 ? std::min(a.grid_sms, rt.num_sms) : rt.num_sms;
}

struct LaunchShape {
    int grid;
    int nparts;
    int layout;
};

// The dynamic shared-memory limit set by cudaFuncSetAttribute applies to the current
// device only: set it once per (kernel, device), tracked in the caller's device mask.
template <class K>
void smem_attr_per_device(K kernel, std::size_t smem, int device, std::atomic<std::uint64_t>& devs) {
    const std::uint64_t bit = device < 64 ? (std::uint64_t(1) << device) : 0;
    if (bit && (devs.load(std::memory_order_acquire) & bit)) return;
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    if (bit) devs.fetch_or(bit, std::memory_order_acq_rel);
}

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

// Kernel choice for the specialised shapes: SELLKIT_SPMV_KERNEL = tma | ldg | auto (default auto = tma
// whenever a row group of the matrix fits one shared-memory stage).
inline int kernel_mode() {
    static int mode = [] {
        const char* e = std::getenv("SELLKIT_SPMV_KERNEL");
        if (e && std::string(e) == "ldg") return 1;
        if (e && std::string(e) == "tma") return 2;
        return 0;
    }();
    return mode;
}

template <class T, int C, int W>
LaunchShape launch_tma(const KArgs<T>& a, int rgt, DeviceRuntime& rt, cudaStream_t st) {
    using P = TPlan<T, W>;
    constexpr int U = unroll_of<T, P, SK_UBUDGET>();
    auto kern = spmv_tma_kernel<T, C, W, U>;
    static std::atomic<std::uint64_t> attr_devs{0};
    smem_attr_per_device(kern, tma_smem_bytes<T, W>(), rt.device, attr_devs);
    static int per_sm = [&] {
        int nb = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kTmaThreads, tma_smem_bytes<T, W>()));
        return std::max(nb, 1);
    }();
    const gidx ngroups = a.rg1 - a.rg0;
    const gidx ntiles = (ngroups + rgt - 1) / rgt;
    const int grid = int(std::max<gidx>(1, std::min<gidx>(ntiles, gidx(per_sm) * grid_sms_of(a, rt))));
    static const int seg = [] {
        const char* e = std::getenv("SELLKIT_TMA_SEG");
        return e ? std::max(1, std::atoi(e)) : 1;
    }();
    kern<<<grid, kTmaThreads, tma_smem_bytes<T, W>(), st>>>(a, rgt, ntiles, seg);
    return {grid, grid, 0};
}

#ifndef SK_RUBUDGET
#define SK_RUBUDGET 33
#endif
#ifndef SK_RUBUDGET_DOTS
#define SK_RUBUDGET_DOTS 44
#endif
// Row-contiguous TMA kernel: unroll so that the in-flight value/index/RHS registers
// of one gather batch stay within a register budget that fits the occupancy
// target (SK_RMINB CTAs/SM: 56 registers per thread at 4).
template <class T, int W, bool DOTS>
constexpr int rows_unroll() {
    constexpr int per = RP<T, W, DOTS>::VEC * int(sizeof(T)) / 4 + int(sizeof(T)) / 4 + 1;
    constexpr int budget = DOTS ? SK_RUBUDGET_DOTS : SK_RUBUDGET;
    constexpr int u = budget / per;
    return u < 1 ? 1 : (u > 8 ? 8 : u);
}

// SELLKIT_TMA_ROWS = 0 | 1 forces the column-slice / row-contiguous consumer mapping;
// default: row-contiguous from 32-B RHS rows on.
inline int rows_mode() {
    static int mode = [] {
        const char* e = std::getenv("SELLKIT_TMA_ROWS");
        return e ? std::atoi(e) : -1;
    }();
    return mode;
}

template <class T, int C, int W, bool DOTS, bool PLAIN, bool MAPPED = false,
          bool DYN = (!DOTS || SK_DYN_DOTS) && !PLAIN && SK_DYN_TILES>
LaunchShape launch_tma_rows(const KArgs<T>& a_in, int rgt, DeviceRuntime& rt, cudaStream_t st) {
    KArgs<T> a = a_in;
    if (!DYN) a.tile_counter = nullptr;
    a.grp_end = int(std::min<gidx>(gidx(a.nrows_padded), a.rg1 * 32));
    constexpr int U = rows_unroll<T, W, DOTS>();
    auto kern = spmv_tma_rows_kernel<T, C, W, U, DOTS, PLAIN, MAPPED, DYN>;
    constexpr std::size_t smem = rows_smem_bytes<T, W, DOTS>();
    static std::atomic<std::uint64_t> attr_devs{0};
    smem_attr_per_device(kern, smem, rt.device, attr_devs);
    static int per_sm = [&] {
        int nb = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kTmaThreads, smem));
        return std::max(nb, 1);
    }();
    const gidx ngroups = a.rg1 - a.rg0;
    // with a sweep order, tiles never straddle a block: blocks x (block / tile) tiles
    const gidx blocks = a.sweep_brg > 0 ? (ngroups + a.sweep_brg - 1) / a.sweep_brg : 0;
    const gidx ntiles = a.sweep_brg > 0 ? blocks * (a.sweep_brg / rgt) : (ngroups + rgt - 1) / rgt;
    const int grid = int(std::max<gidx>(1, std::min<gidx>(ntiles, gidx(per_sm) * grid_sms_of(a, rt))));
    static const int seg = [] {
        const char* e = std::getenv("SELLKIT_TMA_SEG");
        return e ? std::max(1, std::atoi(e)) : 1;
    }();
    // Epilogue-free sweeps deal tiles statically unless the static deal drifts: with many
    // tiles per CTA the CTAs' fronts spread apart and x falls out of L2 (400^3 w = 8: 10.51
    // vs 9.50 GB read, 2.29-2.32 -> 2.08-2.19 ms); smaller sweeps pay for the counter
    // instead (C1 21 -> 25 us, 256^3 w = 8 +2.6 %; wider RHS rows: within noise; r2ak, r2am)
    if constexpr (PLAIN && !DYN && SK_DYN_PLAIN && SK_DYN_TILES && std::is_same_v<T, double>) {
        if (a_in.tile_counter && ntiles >= 600 * gidx(grid))
            return launch_tma_rows<T, C, W, DOTS, PLAIN, MAPPED, true>(a_in, rgt, rt, st);
    }
    if (a.tile_counter) CK(cudaMemsetAsync(a.tile_counter, 0, sizeof(int), st));
    kern<<<grid, kTmaThreads, smem, st>>>(a, rgt, ntiles, seg);
    return {grid, grid, 0};
}

template <class T, int C, int W>
LaunchShape launch_cw(const KArgs<T>& a, DeviceRuntime& rt, cudaStream_t st, lidx max_chunk_len) {
    using P = Plan<T, W>;
    constexpr int U = unroll_of<T, P>();
    if constexpr (RP<T, W, false>::ok && RP<T, W, true>::ok) {
        const int rm = rows_mode();
        const bool rows = rm != 0;
        const bool stride_ok = gidx(a.x_rs) * gidx(sizeof(T)) < (gidx(1) << 31);  // 32-bit byte stride
        if (rows && stride_ok && kernel_mode() != 1) {
            // tiles of at least SK_RTILE_ROWS rows (several warp passes when a warp's
            // rows are few), as far as one stage holds them
            const int cap = RGeom<T, W>::SCAP / (32 * std::max<lidx>(1, max_chunk_len));
            const bool dots = (a.flags & kFlagDots) != 0;
            int rgt = std::min((dots ? std::max(kNCW * RP<T, W, true>::WR, 32)
                                     : std::max(kNCW * RP<T, W, false>::WR, SK_RTILE_ROWS)) / 32,
                               cap);
            while (a.sweep_brg > 0 && rgt > 1 && a.sweep_brg % rgt != 0) --rgt;  // tiles inside blocks
            if (rgt >= 1 && a.row_map != nullptr)  // remote-part sweep of a distributed matrix
                return dots ? launch_tma_rows<T, C, W, true, false, true>(a, rgt, rt, st)
                            : launch_tma_rows<T, C, W, false, false, true>(a, rgt, rt, st);
            if (rgt >= 1) {
                if (dots) return launch_tma_rows<T, C, W, true, false>(a, rgt, rt, st);
                // plain y = A x: no flag, alpha == 1, no deferred rows
                const T one = Ops<T>::one();
                static const bool no_plain = std::getenv("SELLKIT_SPMV_NOPLAIN") != nullptr;  // A/B switch
                const bool plain = !no_plain && a.flags == 0 && a.defer_mask == nullptr &&
                                   std::memcmp(&a.alpha, &one, sizeof(T)) == 0;
                return plain ? launch_tma_rows<T, C, W, false, true>(a, rgt, rt, st)
                             : launch_tma_rows<T, C, W, false, false>(a, rgt, rt, st);
            }
        }
    }
    if (kernel_mode() != 1 && a.row_map == nullptr) {
        // row groups per tile: as many as fit one stage, at most one per consumer warp (slice)
        const int cap = TmaGeom<T, W>::SCAP / (32 * std::max<lidx>(1, max_chunk_len));
        const int rgt = std::min(kNCW / TPlan<T, W>::NSLICE, cap);
        if (rgt >= 1) return launch_tma<T, C, W>(a, rgt, rt, st);
    }
    auto kern = spmv_cw_kernel<T, C, W, U>;
    const int per_sm = occupancy_blocks(kern);
    const gidx ngroups = a.rg1 - a.rg0;
    const gidx items = ngroups * P::NSLICE;
    const gidx need = (items + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const int grid = int(std::max<gidx>(1, std::min<gidx>(need, gidx(per_sm) * grid_sms_of(a, rt))));
    kern<<<grid, kBlock, 0, st>>>(a);
    return {grid, grid, 0};
}

template <class T>
LaunchShape launch_generic(const KArgs<T>& a, DeviceRuntime& rt, cudaStream_t st) {
    const int ncb = (a.width + kGW - 1) / kGW;
    const gidx need = ((a.rg1 - a.rg0) * 32 + kBlock - 1) / kBlock;
    const int gx = int(std::max<gidx>(1, std::min<gidx>(need, gidx(grid_sms_of(a, rt)) * 8)));
    spmv_generic_kernel<T><<<dim3(gx, ncb), kBlock, 0, st>>>(a);
    return {gx, gx, 1};
}

template <class T, int C>
bool try_launch_c(const KArgs<T>& a, DeviceRuntime& rt, cudaStream_t st, LaunchShape& ls, lidx mcl) {
    switch (a.width) {
        case 1: ls = launch_cw<T, C, 1>(a, rt, st, mcl); return true;
        case 2: ls = launch_cw<T, C, 2>(a, rt, st, mcl); return true;
        case 4: ls = launch_cw<T, C, 4>(a, rt, st, mcl); return true;
        case 8: ls = launch_cw<T, C, 8>(a, rt, st, mcl); return true;
        case 16: ls = launch_cw<T, C, 16>(a, rt, st, mcl); return true;
        case 32: ls = launch_cw<T, C, 32>(a, rt, st, mcl); return true;
        case 64: ls = launch_cw<T, C, 64>(a, rt, st, mcl); return true;
        default: return false;
    }
}

template <class T>
LaunchShape launch_any(const KArgs<T>& a, bool specialised_ok, DeviceRuntime& rt, cudaStream_t st, lidx mcl) {
    LaunchShape ls{};
    if (specialised_ok) {
        switch (a.C) {
            case 4:
                if (try_launch_c<T, 4>(a, rt, st, ls, mcl)) return ls;
                break;
            case 8:
                if (try_launch_c<T, 8>(a, rt, st, ls, mcl)) return ls;
                break;
            case 32:
                if (try_launch_c<T, 32>(a, rt, st, ls, mcl)) return ls;
                break;
            default: break;
        }
    }
    return launch_generic<T>(a, rt, st);
}

}  // namespace spmv_detail

// Launch the best kernel for this shape; explicit instantiations live in spmv_<type>.cu.
template <class T>
spmv_detail::LaunchShape launch_spmv(const KArgs<T>& a, bool specialised_ok, DeviceRuntime& rt, cudaStream_t st,
                                     lidx max_chunk_len);

}  // namespace skb
