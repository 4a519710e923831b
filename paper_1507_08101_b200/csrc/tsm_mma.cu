// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) kernels for the compute-heavy
// tall-skinny shapes (reference tsm.hpp:105-225).
//
// Measured on B200 (tools/micro/fp64_peak.cu): DFMA 36 TF/s, DMMA 37 TF/s.  The
// tensor-core path issues one instruction per 256 FMAs instead of 32, which
// leaves the issue slots to the shared-memory fragment loads and the copy
// pipeline.  Products are accumulated with fused multiply-adds, so these shapes
// agree with the reference to 1e-12 (like the FMA paths they replace); the
// bit-exact separate-rounding path stays for m*k <= 64.
//
// Both kernels stream row tiles of V (and W) through a 2-stage cp.async ring in
// shared memory.  Row pitch ps (doubles) is chosen with ps = 4 (mod 16), so the
// 4 rows x 4 consecutive columns one half-warp reads for a fragment fall in
// distinct banks.
//
//   TSMM     W = alpha V X + beta W: rows of W are the MMA M dimension, columns
//            of W the N dimension, m the reduction.  X lives in shared memory in
//            fragment order (one 8-byte load per lane per fragment).
//   TSMTTSM  X = alpha V^T W + beta X: rows of X (m) are M, columns (k) are N,
//            rows of V/W the reduction; one partial m x k block per CTA, the
//            ordered final pass of tsm.cu combines them (deterministic).
#include <algorithm>
#include <cstdint>

#include "ops.cuh"
#include "tma.cuh"
#include "tsm.cuh"

namespace skb {

namespace {

constexpr int kMT = 256;  // threads per CTA (8 warps)
// Tile heights: small enough that 2-3 CTAs fit an SM (the DMMA chains of 8 warps
// leave the tensor pipe idle on fixed-latency waits; measured N = 1e8, m = k = 64:
// TSMM 34.3 -> 30.5 ms, TSMTTSM 30.8 -> 28.1 ms).
#ifndef SK_MM_RM
#define SK_MM_RM 2
#endif
#ifndef SK_TT_RB
#define SK_TT_RB 32
#endif
#ifndef SK_MM_MINB
#define SK_MM_MINB 3
#endif
// V row tiles of the compute-bound TSMM shapes (k, m >= 32) staged by per-row bulk
// copies (one warp, mbarrier-completed) instead of 16-B cp.async from every thread:
// the staging address math left the DMMA pipe idle (m = k = 64, N = 1e8: 30.4 ->
// 27.3 ms).  The bandwidth-bound small shapes keep cp.async (short rows are
// slow bulk copies: m = k = 16 3.9 -> 5.5 ms).
#ifndef SK_MM_BULK
#define SK_MM_BULK 1
#endif
// The same staging for TSMTTSM (V and W rows, zeroed short tiles) is slower with its
// 32-row tiles (m = k = 64: 26.9 -> 31.8 ms; 32: 9.2 -> 12.6 ms): off
#ifndef SK_TT_BULK
#define SK_TT_BULK 0
#endif
#ifndef SK_TT_AM
#define SK_TT_AM 2
#endif
#ifndef SK_TT_MINB
#define SK_TT_MINB 2
#endif

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ std::uint32_t smem_addr(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async copy; bytes < 16 zero-fills the tail (rows past the end)
__device__ __forceinline__ void cp16(void* dst, const void* src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__host__ __device__ constexpr int pitch_of(int cols) { return cols <= 4 ? 4 : ((cols - 4 + 15) / 16) * 16 + 4; }

// Copy rows [r0, r0 + nr) of a compact row-major n x cols block into shared
// memory with row pitch ps (rows >= n are zero-filled).
__device__ __forceinline__ void stage_rows(double* dst, const double* src, gidx n, gidx r0, int nr, int cols, int ps) {
    const int per_row = cols / 2;
    for (int q = threadIdx.x; q < nr * per_row; q += kMT) {
        const int r = q / per_row, c = (q - r * per_row) * 2;
        const gidx gr = r0 + r;
        const bool in = gr < n;
        cp16(dst + r * ps + c, src + (in ? gr : 0) * cols + c, in ? 16 : 0);
    }
}

// ----------------------------------------------------------------- TSMM ----
// KB = k/8 column blocks; CN column blocks per warp, RM row blocks per warp.
template <int KB>
struct MmGeom {
    static constexpr int CN = KB < 4 ? KB : 4;
    static constexpr int WPR = KB / CN;           // warps per row set
    static constexpr int RSETS = 8 / WPR;         // row sets per CTA
    static constexpr int RM = KB >= 8 ? SK_MM_RM : 1;  // 8-row blocks per warp (1 for k <= 32: more CTAs)
    static constexpr int RB = RSETS * RM * 8;     // rows per tile
};

template <int KB, bool BULK>
__global__ void __launch_bounds__(kMT, KB >= 8 ? SK_MM_MINB : SK_MM_MINB + 1)
    tsmm_dmma_kernel(double* __restrict__ w, const double* __restrict__ v, const double* __restrict__ xcm, gidx n,
                     int m, double alpha, double beta, int beta_zero) {
    using G = MmGeom<KB>;
    constexpr int k = KB * 8;
    const int ps = pitch_of(m);
    extern __shared__ __align__(16) double sm[];
    double* xf = sm;                       // fragment-ordered X: [m/4][KB][32]
    double* vt = xf + (m / 4) * KB * 32;   // 2 stages x RB x ps
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // X (col-major m x k) -> fragment order: xf[(mb*KB + cb)*32 + l] = X[mb*4 + l%4][cb*8 + l/4]
    for (int q = threadIdx.x; q < m * k; q += kMT) {
        const int l = q & 31, blk = q >> 5, mb = blk / KB, cb = blk - mb * KB;
        xf[q] = xcm[gidx(cb * 8 + l / 4) * m + mb * 4 + (l & 3)];
    }
    const gidx ntiles = (n + G::RB - 1) / G::RB;
    const int rset = warp / G::WPR, cset = warp - rset * G::WPR;
    const int rbase = rset * G::RM * 8, cb0 = cset * G::CN;
    gidx t = blockIdx.x;
    __shared__ __align__(8) std::uint64_t full[2];
    const unsigned long long pol = l2_evict_first_policy();
    // BULK: rows past n are not copied; their (stale) products are never stored
    auto issue = [&](gidx tile, int s) {
        if constexpr (BULK) {
            if (warp != 0) return;
            const gidx rb = tile * G::RB;
            const int nr = int(min(gidx(G::RB), n - rb));
            if (lane == 0) mbar_arrive_expect_tx(&full[s], std::uint32_t(nr) * std::uint32_t(m) * 8u);
            __syncwarp();
            for (int r = lane; r < nr; r += 32)
                bulk_g2s(vt + (s * G::RB + r) * ps, v + (rb + r) * m, std::uint32_t(m) * 8u, &full[s], pol);
        } else {
            stage_rows(vt + s * G::RB * ps, v, n, tile * G::RB, G::RB, m, ps);
        }
    };
    if constexpr (BULK) {
        if (threadIdx.x == 0) {
            mbar_init(&full[0], 1);
            mbar_init(&full[1], 1);
            mbar_fence_init();
        }
        __syncthreads();
    }
    if (t < ntiles) issue(t, 0);
    if constexpr (!BULK) cp_commit();
    for (int it = 0; t < ntiles; ++it, t += gridDim.x) {
        const gidx tn = t + gridDim.x;
        if (tn < ntiles) issue(tn, (it + 1) & 1);
        if constexpr (BULK) {
            mbar_wait(&full[it & 1], std::uint32_t(it >> 1) & 1u);
        } else {
            cp_commit();
            cp_wait<1>();
            __syncthreads();
        }
        const double* vs = vt + (it & 1) * G::RB * ps;
        double acc[G::RM][G::CN][2];
#pragma unroll
        for (int i = 0; i < G::RM; ++i)
#pragma unroll
            for (int j = 0; j < G::CN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        const double* ap = vs + (rbase + (lane >> 2)) * ps + (lane & 3);
        const double* bp = xf + cb0 * 32 + lane;
#pragma unroll 2
        for (int mb = 0; mb < m / 4; ++mb) {
            double a[G::RM], b[G::CN];
#pragma unroll
            for (int i = 0; i < G::RM; ++i) a[i] = ap[i * 8 * ps + mb * 4];
#pragma unroll
            for (int j = 0; j < G::CN; ++j) b[j] = bp[(mb * KB + j) * 32];
#pragma unroll
            for (int i = 0; i < G::RM; ++i)
#pragma unroll
                for (int j = 0; j < G::CN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
        // epilogue: lane holds W[row][col], W[row][col + 1]
#pragma unroll
        for (int i = 0; i < G::RM; ++i) {
            const gidx row = t * G::RB + rbase + i * 8 + (lane >> 2);
            if (row >= n) continue;
#pragma unroll
            for (int j = 0; j < G::CN; ++j) {
                const int col = (cb0 + j) * 8 + 2 * (lane & 3);
                double2* wp = reinterpret_cast<double2*>(w + row * k + col);
                double2 o;
                if (beta_zero) {
                    o.x = __dmul_rn(alpha, acc[i][j][0]);
                    o.y = __dmul_rn(alpha, acc[i][j][1]);
                } else {
                    const double2 old = *wp;
                    o.x = __dadd_rn(__dmul_rn(alpha, acc[i][j][0]), __dmul_rn(beta, old.x));
                    o.y = __dadd_rn(__dmul_rn(alpha, acc[i][j][1]), __dmul_rn(beta, old.y));
                }
                *wp = o;
            }
        }
        __syncthreads();  // this stage is refilled two iterations on
    }
    if constexpr (!BULK) cp_wait<0>();
}

// --------------------------------------------------------------- TSMTTSM ----
template <int MB, int KB>
struct TtGeom {
    static constexpr int NBLK = MB * KB;
    static constexpr int BPW = NBLK >= 8 ? NBLK / 8 : 1;   // blocks per warp
    static constexpr int RS = NBLK >= 8 ? 1 : 8 / NBLK;    // row splits (warps sharing a block set)
    static constexpr int RB = SK_TT_RB;                     // rows per tile
    // a warp owns an AM x BN rectangle of blocks: per row quad it loads AM A- and BN
    // B-fragments for AM * BN DMMAs (2 x 4: 6 LDS per 8 DMMA instead of 9 for 1 x 8)
    static constexpr int AM = (SK_TT_AM > 1 && BPW >= 4 && MB % 2 == 0) ? 2 : 1;
    static constexpr int BN = BPW / AM;
    static_assert(KB % BN == 0 && MB % AM == 0, "block rectangle must tile the result");
};

template <int MB, int KB, bool BULK>
__global__ void __launch_bounds__(kMT, SK_TT_MINB)
    tsmttsm_dmma_kernel(const double* __restrict__ v, const double* __restrict__ w, gidx n, gidx rows_per_cta,
                        double* __restrict__ partial) {
    using G = TtGeom<MB, KB>;
    constexpr int m = MB * 8, k = KB * 8;
    constexpr int pv = pitch_of(m), pw = pitch_of(k);
    extern __shared__ __align__(16) double sm[];
    double* vt = sm;                        // 2 x RB x pv
    double* wt = vt + 2 * G::RB * pv;       // 2 x RB x pw
    double* red = wt + 2 * G::RB * pw;      // [RS][NBLK][64] (= 8 x BPW x 64)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rs = warp % G::RS, bg = warp / G::RS;
    constexpr int NCG = KB / G::BN;                        // column groups of blocks
    const int ab0 = (bg / NCG) * G::AM, bb0 = (bg % NCG) * G::BN;  // first a-block, b-block
    const gidx r0 = gidx(blockIdx.x) * rows_per_cta;
    const gidx r1 = min(n, r0 + rows_per_cta);
    const gidx ntiles = r1 > r0 ? (r1 - r0 + G::RB - 1) / G::RB : 0;
    double acc[G::AM][G::BN][2];
#pragma unroll
    for (int i = 0; i < G::AM; ++i)
#pragma unroll
        for (int j = 0; j < G::BN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    __shared__ __align__(8) std::uint64_t full[2];
    const unsigned long long pol = l2_evict_first_policy();
    auto stage = [&](gidx tile, int s) {
        const gidx rb = r0 + tile * G::RB;
        if constexpr (BULK) {
            // rows [nr, RB) of a short last tile are zeroed (they enter the row sum);
            // the trailing __syncthreads of the iteration publishes the zeros
            const int nr = int(min(gidx(G::RB), r1 - rb));
            if (nr < G::RB) {
                for (int q = threadIdx.x; q < (G::RB - nr) * pv; q += kMT) vt[(s * G::RB + nr) * pv + q] = 0.0;
                for (int q = threadIdx.x; q < (G::RB - nr) * pw; q += kMT) wt[(s * G::RB + nr) * pw + q] = 0.0;
            }
            if (warp != 0) return;
            if (lane == 0) mbar_arrive_expect_tx(&full[s], std::uint32_t(nr) * std::uint32_t(m + k) * 8u);
            __syncwarp();
            for (int r = lane; r < nr; r += 32) {
                bulk_g2s(vt + (s * G::RB + r) * pv, v + (rb + r) * m, m * 8u, &full[s], pol);
                bulk_g2s(wt + (s * G::RB + r) * pw, w + (rb + r) * k, k * 8u, &full[s], pol);
            }
        } else {
            // rows past r1 are zero-filled (n argument = r1)
            stage_rows(vt + s * G::RB * pv, v, r1, rb, G::RB, m, pv);
            stage_rows(wt + s * G::RB * pw, w, r1, rb, G::RB, k, pw);
        }
    };
    if constexpr (BULK) {
        if (threadIdx.x == 0) {
            mbar_init(&full[0], 1);
            mbar_init(&full[1], 1);
            mbar_fence_init();
        }
        __syncthreads();
    }
    if (ntiles > 0) stage(0, 0);
    if constexpr (BULK) {
        __syncthreads();  // zero rows of a one-tile range
    } else {
        cp_commit();
    }
    for (gidx t = 0; t < ntiles; ++t) {
        if (t + 1 < ntiles) stage(t + 1, int((t + 1) & 1));
        if constexpr (BULK) {
            mbar_wait(&full[t & 1], std::uint32_t(t >> 1) & 1u);
        } else {
            cp_commit();
            cp_wait<1>();
            __syncthreads();
        }
        const double* vs = vt + (t & 1) * G::RB * pv;
        const double* ws = wt + (t & 1) * G::RB * pw;
        // A (8 a x 4 rows): lane -> V[row + l%4][a + l/4]; B (4 rows x 8 b): W[row + l%4][b + l/4]
        const double* ap = vs + (lane & 3) * pv + ab0 * 8 + (lane >> 2);
        const double* bp = ws + (lane & 3) * pw + bb0 * 8 + (lane >> 2);
#pragma unroll 4
        for (int r4 = rs; r4 < G::RB / 4; r4 += G::RS) {
            double a[G::AM], b[G::BN];
#pragma unroll
            for (int i = 0; i < G::AM; ++i) a[i] = ap[r4 * 4 * pv + i * 8];
#pragma unroll
            for (int j = 0; j < G::BN; ++j) b[j] = bp[r4 * 4 * pw + j * 8];
#pragma unroll
            for (int i = 0; i < G::AM; ++i)
#pragma unroll
                for (int j = 0; j < G::BN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
        __syncthreads();
    }
    if constexpr (!BULK) cp_wait<0>();
    // warp partials -> shared memory, then the row splits of each block are summed
    // in a fixed order and written col-major (cell = b*m + a, as tsm.hpp:145)
#pragma unroll
    for (int i = 0; i < G::AM; ++i)
#pragma unroll
        for (int j = 0; j < G::BN; ++j) {
            const int blk = (ab0 + i) * KB + bb0 + j;
            red[(rs * G::NBLK + blk) * 64 + lane * 2] = acc[i][j][0];
            red[(rs * G::NBLK + blk) * 64 + lane * 2 + 1] = acc[i][j][1];
        }
    __syncthreads();
    for (int c = threadIdx.x; c < m * k; c += kMT) {
        const int a = c % m, b = c / m;
        const int blk = (a / 8) * KB + b / 8;
        // fragment position of (a % 8, b % 8): lane = (a%8)*4 + (b%8)/2, element (b%8)%2
        const int idx = ((a & 7) * 4 + ((b & 7) >> 1)) * 2 + (b & 1);
        double s = 0.0;
        for (int q = 0; q < G::RS; ++q) s = __dadd_rn(s, red[(q * G::NBLK + blk) * 64 + idx]);
        partial[gidx(blockIdx.x) * m * k + c] = s;
    }
}

template <class F>
bool dispatch_blocks(int nb, F&& f) {
    switch (nb) {
        case 1: f(std::integral_constant<int, 1>{}); return true;
        case 2: f(std::integral_constant<int, 2>{}); return true;
        case 4: f(std::integral_constant<int, 4>{}); return true;
        case 8: f(std::integral_constant<int, 8>{}); return true;
        default: return false;
    }
}

}  // namespace

bool tsmm_dmma(double* w, const double* v, const double* xcm, gidx n, int m, int k, double alpha, double beta,
               bool beta_zero, DeviceRuntime& rt) {
    if (m % 4 != 0 || m < 4 || m > 64 || k % 8 != 0 || k < 8 || k > 64 || n <= 0) return false;
    bool ok = false;
    dispatch_blocks(k / 8, [&](auto kb) {
        constexpr int KB = decltype(kb)::value;
        using G = MmGeom<KB>;
        const std::size_t smem = (std::size_t(m) * KB * 8 + 2 * std::size_t(G::RB) * pitch_of(m)) * sizeof(double);
        if (smem > 220 * 1024) return;
        const bool bulk = SK_MM_BULK && KB >= 4 && m >= 32;
        auto kern = bulk ? tsmm_dmma_kernel<KB, true> : tsmm_dmma_kernel<KB, false>;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        const gidx ntiles = (n + G::RB - 1) / G::RB;
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMT, smem));
        const int grid = int(std::max<gidx>(1, std::min<gidx>(ntiles, gidx(std::max(per_sm, 1)) * rt.num_sms)));
        kern<<<grid, kMT, smem, rt.stream>>>(w, v, xcm, n, m, alpha, beta, beta_zero ? 1 : 0);
        CK(cudaGetLastError());
        ok = true;
    });
    return ok;
}

int tsmttsm_dmma_partials(const double* v, const double* w, gidx n, int m, int k, double* part, int max_parts,
                          DeviceRuntime& rt) {
    if (m % 8 != 0 || k % 8 != 0 || m < 8 || k < 8 || m > 64 || k > 64 || n <= 0) return 0;
    int nparts = 0;
    dispatch_blocks(m / 8, [&](auto mbc) {
        dispatch_blocks(k / 8, [&](auto kbc) {
            constexpr int MB = decltype(mbc)::value, KB = decltype(kbc)::value;
            using G = TtGeom<MB, KB>;
            const std::size_t smem =
                (2 * std::size_t(G::RB) * (pitch_of(MB * 8) + pitch_of(KB * 8)) + 8 * std::size_t(G::BPW) * 64) *
                sizeof(double);
            const bool bulk = SK_TT_BULK && MB >= 4 && KB >= 4;
            auto kern = bulk ? tsmttsm_dmma_kernel<MB, KB, true> : tsmttsm_dmma_kernel<MB, KB, false>;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            int per_sm = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMT, smem));
            const int slots = std::max(per_sm, 1) * rt.num_sms;
            nparts = int(std::max<gidx>(1, std::min<gidx>(std::min(slots, max_parts), (n + G::RB - 1) / G::RB)));
            const gidx rows_per = (n + nparts - 1) / nparts;
            kern<<<nparts, kMT, smem, rt.stream>>>(v, w, n, rows_per, part);
            CK(cudaGetLastError());
        });
    });
    return nparts;
}

}  // namespace skb
