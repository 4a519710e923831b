// Tall-skinny dense kernels on the device.
// Reference: /root/reference/proj/src/tsm.hpp:37-305.
//
// TSMM      W = alpha*V*X + beta*W : one thread per output element, X (m x k)
//           staged once per CTA in shared memory, V rows read through L1 (all
//           lanes of a row share the row's bytes), tmp accumulated over m in the
//           reference's order.  For m*k <= 64 (HBM-bound shapes) every product
//           and sum is rounded separately => bit-identical to the reference;
//           larger shapes are FP64-issue-bound and use FMA (within 1e-12).
//           beta == 0 => W is not read (BLAS convention; the reference forms
//           beta*W, which differs only for non-finite W).
// TSMTTSM   X = alpha*V^H*W + beta*X : each CTA reduces a contiguous row range
//           (rows staged in shared memory, 32 at a time) into per-thread cell
//           accumulators, writes its partial m x k block, and an ordered pass
//           combines CTA partials (Kahan-Babuska-Neumaier on request, like
//           CompensatedSum tsm.hpp:73-87) and applies alpha/beta.
// Fast paths for compact row-major real operands (measured, N = 1e8, B200):
//   m, k <= 8      one row per thread, whole rows moved with vector accesses
//                  (tsmm_row_kernel keeps the reference's rounding): 80-94 % of HBM
//   m, k >= 8      FP64 tensor cores, tsm_mma.cu: m = k = 64 at 24-27 TF/s
//   otherwise      the generic kernels above.
#include <algorithm>

#include "ops.cuh"
#include "tsm.cuh"

namespace skb {

namespace {

constexpr int kT = 256;
constexpr int kCellsPerThread = 16;
constexpr int kRowTile = 32;

__device__ __forceinline__ char* eptr(const DAcc& a, gidx i, gidx j, std::size_t es) {
    const gidx c = a.cmap ? a.cmap[j] : j;
    return a.base + ((a.row_offset + i) * a.rs + c * a.cs) * gidx(es);
}
template <class T>
__device__ __forceinline__ T& el(const DAcc& a, gidx i, gidx j) {
    return *reinterpret_cast<T*>(eptr(a, i, j, sizeof(T)));
}

template <class T, bool EXACT>
__device__ __forceinline__ T madd(T acc, T a, T b) {
    using O = Ops<T>;
    if constexpr (EXACT) return O::add(acc, O::mul(a, b));
    else return O::fma(a, b, acc);
}

// X copied to a dense col-major device array (tsm.hpp:93-98 normalize_small_colmajor)
template <class T>
__global__ void x_colmajor_kernel(DAcc x, lidx m, lidx k, T* out) {
    const gidx t = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (t >= gidx(m) * k) return;
    const lidx kk = lidx(t / m), mm = lidx(t % m);
    out[t] = el<T>(x, mm, kk);
}

template <class T, bool EXACT>
__global__ void __launch_bounds__(kT) tsmm_kernel(DAcc w, DAcc v, const T* __restrict__ xcm, gidx n, lidx m, lidx k,
                                                  T alpha, T beta, int beta_zero, int x_in_smem) {
    using O = Ops<T>;
    extern __shared__ unsigned char smem_raw[];
    T* xs = reinterpret_cast<T*>(smem_raw);
    const T* X = xcm;
    if (x_in_smem) {
        for (int t = threadIdx.x; t < m * k; t += blockDim.x) xs[t] = xcm[t];
        __syncthreads();
        X = xs;
    }
    const gidx total = n * k;
    for (gidx e = blockIdx.x * gidx(blockDim.x) + threadIdx.x; e < total; e += gidx(gridDim.x) * blockDim.x) {
        const gidx i = e / k;
        const lidx kk = lidx(e - i * k);
        T tmp = O::zero();
        for (lidx mm = 0; mm < m; ++mm) tmp = madd<T, EXACT>(tmp, el<T>(v, i, mm), X[gidx(kk) * m + mm]);
        T& wr = el<T>(w, i, kk);
        wr = beta_zero ? O::mul(alpha, tmp) : O::add(O::mul(alpha, tmp), O::mul(beta, wr));
    }
}

// In place: each CTA owns `rows` rows; all outputs are computed into registers
// before any of them is written back (tsm.hpp:230-249 row-local temp).
template <class T, bool EXACT>
__global__ void __launch_bounds__(kT) tsmm_inplace_kernel(DAcc v, const T* __restrict__ xcm, gidx n, lidx m,
                                                          lidx rows, T alpha, T beta) {
    using O = Ops<T>;
    const gidx r0 = gidx(blockIdx.x) * rows;
    const gidx cnt = min(gidx(rows), n - r0) * m;
    T out[kCellsPerThread];
#pragma unroll
    for (int q = 0; q < kCellsPerThread; ++q) {
        const gidx e = threadIdx.x + gidx(q) * kT;
        out[q] = O::zero();
        if (e < cnt) {
            const gidx i = r0 + e / m;
            const lidx kk = lidx(e % m);
            T s = O::zero();
            for (lidx mm = 0; mm < m; ++mm) s = madd<T, EXACT>(s, el<T>(v, i, mm), xcm[gidx(kk) * m + mm]);
            out[q] = s;
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kCellsPerThread; ++q) {
        const gidx e = threadIdx.x + gidx(q) * kT;
        if (e < cnt) {
            const gidx i = r0 + e / m;
            const lidx kk = lidx(e % m);
            T& vr = el<T>(v, i, kk);
            vr = O::add(O::mul(alpha, out[q]), O::mul(beta, vr));
        }
    }
}

// Kahan-Babuska-Neumaier step (tsm.hpp:78-85)
template <class T>
__device__ __forceinline__ void kbn_add(T& sum, T& comp, T x) {
    using O = Ops<T>;
    const T t = O::add(sum, x);
    if (O::abs2(sum) >= O::abs2(x))
        comp = O::add(comp, O::add(O::sub(sum, t), x));
    else
        comp = O::add(comp, O::add(O::sub(x, t), sum));
    sum = t;
}

template <class T, bool KAHAN>
__global__ void __launch_bounds__(kT) tsmttsm_partial_kernel(DAcc v, DAcc w, gidx n, lidx m, lidx k, gidx rows_per_cta,
                                                             T* partial, T* pcomp) {
    using O = Ops<T>;
    extern __shared__ unsigned char smem_raw[];
    T* vs = reinterpret_cast<T*>(smem_raw);      // [kRowTile][m]
    T* ws = vs + kRowTile * m;                   // [kRowTile][k]
    const gidx cells = gidx(m) * k;
    const gidx cell0 = gidx(blockIdx.y) * kT * kCellsPerThread;
    T acc[kCellsPerThread], cmp[kCellsPerThread];
    lidx cm[kCellsPerThread], ck[kCellsPerThread];
#pragma unroll
    for (int q = 0; q < kCellsPerThread; ++q) {
        acc[q] = O::zero();
        cmp[q] = O::zero();
        const gidx c = cell0 + threadIdx.x + gidx(q) * kT;
        cm[q] = lidx(c % m);  // X accumulators are col-major: cell = kk*m + mm
        ck[q] = lidx(c / m);
    }
    const gidx r_begin = gidx(blockIdx.x) * rows_per_cta;
    const gidx r_end = min(n, r_begin + rows_per_cta);
    for (gidx r0 = r_begin; r0 < r_end; r0 += kRowTile) {
        const int nr = int(min(gidx(kRowTile), r_end - r0));
        __syncthreads();
        for (int t = threadIdx.x; t < nr * m; t += kT) vs[t] = O::conj(el<T>(v, r0 + t / m, t % m));
        for (int t = threadIdx.x; t < nr * k; t += kT) ws[t] = el<T>(w, r0 + t / k, t % k);
        __syncthreads();
        for (int r = 0; r < nr; ++r) {
#pragma unroll
            for (int q = 0; q < kCellsPerThread; ++q) {
                if (cell0 + threadIdx.x + gidx(q) * kT < cells) {
                    const T p = O::mul(vs[r * m + cm[q]], ws[r * k + ck[q]]);
                    if constexpr (KAHAN) kbn_add(acc[q], cmp[q], p);
                    else acc[q] = O::add(acc[q], p);
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < kCellsPerThread; ++q) {
        const gidx c = cell0 + threadIdx.x + gidx(q) * kT;
        if (c < cells) {
            partial[gidx(blockIdx.x) * cells + c] = acc[q];
            if constexpr (KAHAN) pcomp[gidx(blockIdx.x) * cells + c] = cmp[q];
        }
    }
}

template <class T, bool KAHAN>
__global__ void tsmttsm_final_kernel(const T* partial, const T* pcomp, int nparts, lidx m, lidx k, DAcc x, T alpha,
                                     T beta) {
    using O = Ops<T>;
    const gidx c = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    const gidx cells = gidx(m) * k;
    if (c >= cells) return;
    T s = O::zero();
    if constexpr (KAHAN) {
        T cs = O::zero();
        for (int b = 0; b < nparts; ++b) {
            kbn_add(s, cs, partial[gidx(b) * cells + c]);
            kbn_add(s, cs, pcomp[gidx(b) * cells + c]);
        }
        s = O::add(s, cs);
    } else {
        for (int b = 0; b < nparts; ++b) s = O::add(s, partial[gidx(b) * cells + c]);
    }
    const lidx mm = lidx(c % m), kk = lidx(c / m);
    T& xr = el<T>(x, mm, kk);
    xr = O::add(O::mul(alpha, s), O::mul(beta, xr));
}

template <class T>
__global__ void gemm_naive_kernel(DAcc c, DAcc a, DAcc b, lidx n, lidx kc, lidx inner, int ta, int tb, T alpha,
                                  T beta) {
    using O = Ops<T>;
    const gidx t = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (t >= gidx(n) * kc) return;
    const lidx i = lidx(t / kc), j = lidx(t % kc);
    T s = O::zero();
    for (lidx l = 0; l < inner; ++l) {
        T av = ta == 0 ? el<T>(a, i, l) : el<T>(a, l, i);
        if (ta == 2) av = O::conj(av);
        T bv = tb == 0 ? el<T>(b, l, j) : el<T>(b, j, l);
        if (tb == 2) bv = O::conj(bv);
        s = O::add(s, O::mul(av, bv));
    }
    T& cr = el<T>(c, i, j);
    cr = O::add(O::mul(alpha, s), O::mul(beta, cr));
}

// ---------------------------------------------------------------- fast paths
// Row-major, compact V/W (column step 1, no column map), real element types.

// A whole compact row of N elements in as few vector accesses as its size allows
// (32-byte LDG/STG pieces, else 16/8 bytes); p must be aligned to the row size
// (rows of a compact row-major block with N in {1,2,4,8} are).
template <class T, int N>
__device__ __forceinline__ void load_row(const T* p, T (&r)[N]) {
    constexpr int B = N * int(sizeof(T));
    if constexpr (B >= 32 && B % 32 == 0) {
        constexpr int P = 32 / int(sizeof(T));
#pragma unroll
        for (int q = 0; q < N / P; ++q) {
            const Vec<T, P> x = ld_x<T, P>(p + q * P);
#pragma unroll
            for (int e = 0; e < P; ++e) r[q * P + e] = x.v[e];
        }
    } else {
        const Vec<T, N> x = ld_x<T, N>(p);
#pragma unroll
        for (int e = 0; e < N; ++e) r[e] = x.v[e];
    }
}
template <class T, int N>
__device__ __forceinline__ void store_row(T* p, const T (&r)[N]) {
    constexpr int B = N * int(sizeof(T));
    if constexpr (B >= 32 && B % 32 == 0) {
        constexpr int P = 32 / int(sizeof(T));
#pragma unroll
        for (int q = 0; q < N / P; ++q) {
            Vec<T, P> x;
#pragma unroll
            for (int e = 0; e < P; ++e) x.v[e] = r[q * P + e];
            st_vec<T, P>(p + q * P, x);
        }
    } else {
        Vec<T, N> x;
#pragma unroll
        for (int e = 0; e < N; ++e) x.v[e] = r[e];
        st_vec<T, N>(p, x);
    }
}

// TSMTTSM shapes with at least this many cells (and m, k multiples of 8) use DMMA
// (m = k = 8 through DMMA measured 2.40 -> 2.37 ms at N = 1e8, within the spread: kept
// on the register kernel)
#ifndef SK_TT_DMMA_MIN_CELLS
#define SK_TT_DMMA_MIN_CELLS 65
#endif
// partials (CTAs) per SM of the register TSMTTSM for m * k <= 4 (measured m = k = 1,
// N = 1e8: 2 / 3 / 4 / 8 / 16 per SM -> 0.45 / 0.35 / 0.31 / 0.34 / 0.41 ms)
#ifndef SK_TT_PARTS_SMALL
#define SK_TT_PARTS_SMALL 4
#endif
#ifndef SK_TT_UR_MAX
#define SK_TT_UR_MAX 8
#endif
#ifndef SK_TT_CHUNK_UR  // 32-byte chunks in flight per thread in the chunked TSMTTSM path
#define SK_TT_CHUNK_UR 2
#endif
#ifndef SK_TSM_CHUNK    // 1: chunked paths for the 8- and 16-byte-row shapes (1x1, 2x2)
#define SK_TSM_CHUNK 1
#endif
#ifndef SK_TSM_PAIR8    // 1: TSMTTSM 8 x 8 with a lane pair per row (32 accumulators per lane)
#define SK_TSM_PAIR8 1
#endif
#ifndef SK_TT_PAIR_UR
#define SK_TT_PAIR_UR 2
#endif
#ifndef SK_TT_SPLIT_LPR  // lanes per row of the 8 x 8 split kernel
#define SK_TT_SPLIT_LPR 2
#endif

// TSMTTSM, m <= MM, k <= KK (MM, KK in {1,2,4,8}): each thread keeps the whole
// m x k block in registers and walks its rows of the CTA's contiguous range;
// warp butterfly + ordered CTA sum -> one partial per CTA (deterministic).
// Compact operands with m == MM, k == KK load whole rows with vector accesses.
// R > 1 (compact m == MM, k == KK, MM * R * sizeof(T) == 32): a thread loads R consecutive
// rows of V and of W with one 32-byte access each (1 x 1: four rows per LDG.256), UR2
// chunks in flight -- the 8- and 16-byte rows otherwise leave too few bytes in flight.
template <class T, int MM, int KK, bool KAHAN, int R = 1>
__global__ void __launch_bounds__(kT) tsmttsm_reg_kernel(const T* __restrict__ v, gidx vs, const T* __restrict__ w,
                                                         gidx ws, gidx n, int m, int k, gidx rows_per_cta, T* partial,
                                                         T* pcomp) {
    using O = Ops<T>;
    __shared__ T red[kT / 32][MM * KK];
    __shared__ T redc[KAHAN ? kT / 32 : 1][MM * KK];
    T acc[MM][KK], cmp[MM][KK];
#pragma unroll
    for (int a = 0; a < MM; ++a)
#pragma unroll
        for (int b = 0; b < KK; ++b) acc[a][b] = cmp[a][b] = O::zero();
    const gidx r0 = gidx(blockIdx.x) * rows_per_cta;
    const gidx r1 = min(n, r0 + rows_per_cta);
    // (the scalar loop is as fast for 1 x 1 and keeps its loads batched)
    const bool vec = MM * KK > 1 && m == MM && k == KK && vs == MM && ws == KK;
    auto load = [&](gidx i, T (&vr)[MM], T (&wr)[KK]) {
        if (vec) {
            load_row<T, MM>(v + i * MM, vr);
            load_row<T, KK>(w + i * KK, wr);
#pragma unroll
            for (int a = 0; a < MM; ++a) vr[a] = O::conj(vr[a]);
        } else {
#pragma unroll
            for (int a = 0; a < MM; ++a) vr[a] = a < m ? O::conj(__ldg(v + i * vs + a)) : O::zero();
#pragma unroll
            for (int b = 0; b < KK; ++b) wr[b] = b < k ? __ldg(w + i * ws + b) : O::zero();
        }
    };
    auto accum = [&](const T (&vr)[MM], const T (&wr)[KK]) {
#pragma unroll
        for (int a = 0; a < MM; ++a)
#pragma unroll
            for (int b = 0; b < KK; ++b) {
                if constexpr (KAHAN) kbn_add(acc[a][b], cmp[a][b], O::mul(vr[a], wr[b]));
                else acc[a][b] = O::fma(vr[a], wr[b], acc[a][b]);
            }
    };
    // UR rows of this thread per batch, all loads first (bytes in flight: the small
    // shapes are HBM-bound); the rows are still accumulated in row order
    // (measured per shape, N = 1e8, ms with UR = 4 vs 1: 4x4 0.98 / 1.14, 2x4 0.93 / 1.04,
    // 8x2 1.31 / 1.39, 8x1 1.07 / 1.13; slower with 4 or 2 for 4x2, 2x8, 4x8, 8x4, 1x1, 2x2)
    constexpr bool kUnroll = (MM == 4 && KK == 4) || (MM == 2 && KK == 4) || (MM == 8 && KK == 2) || (MM == 8 && KK == 1);
    constexpr int UR0 = !KAHAN && kUnroll ? 4 : 1;
    constexpr int UR = UR0 < SK_TT_UR_MAX ? UR0 : SK_TT_UR_MAX;
    gidx i = r0 + threadIdx.x;
    if constexpr (R > 1) {
        // chunks of R rows (the CTA range starts on a chunk; only the last CTA's end may not)
        constexpr int UR2 = SK_TT_CHUNK_UR;
        i = r0 + gidx(threadIdx.x) * R;
        for (; i + gidx(UR2 - 1) * kT * R + R <= r1; i += gidx(UR2) * kT * R) {
            T vr[UR2][R * MM], wr[UR2][R * KK];
#pragma unroll
            for (int u = 0; u < UR2; ++u) {
                load_row<T, R * MM>(v + (i + gidx(u) * kT * R) * MM, vr[u]);
                load_row<T, R * KK>(w + (i + gidx(u) * kT * R) * KK, wr[u]);
            }
#pragma unroll
            for (int u = 0; u < UR2; ++u)
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int a = 0; a < MM; ++a)
#pragma unroll
                        for (int b = 0; b < KK; ++b)
                            acc[a][b] = O::fma(O::conj(vr[u][r * MM + a]), wr[u][r * KK + b], acc[a][b]);
        }
        for (; i < r1; i += gidx(kT) * R) {  // remaining chunks one at a time, the last one by rows
            if (i + R <= r1) {
                T vr[R * MM], wr[R * KK];
                load_row<T, R * MM>(v + i * MM, vr);
                load_row<T, R * KK>(w + i * KK, wr);
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int a = 0; a < MM; ++a)
#pragma unroll
                        for (int b = 0; b < KK; ++b)
                            acc[a][b] = O::fma(O::conj(vr[r * MM + a]), wr[r * KK + b], acc[a][b]);
            } else {
                for (gidx j = i; j < r1; ++j) {
                    T vr[MM], wr[KK];
                    load(j, vr, wr);
                    accum(vr, wr);
                }
            }
        }
        i = r1;  // nothing left for the row loops below
    }
    if constexpr (UR > 1) {
        for (; i + gidx(UR - 1) * kT < r1; i += gidx(UR) * kT) {
            T vr[UR][MM], wr[UR][KK];
#pragma unroll
            for (int u = 0; u < UR; ++u) load(i + gidx(u) * kT, vr[u], wr[u]);
#pragma unroll
            for (int u = 0; u < UR; ++u) accum(vr[u], wr[u]);
        }
    }
    for (; i < r1; i += kT) {
        T vr[MM], wr[KK];
        load(i, vr, wr);
        accum(vr, wr);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int a = 0; a < MM; ++a)
#pragma unroll
        for (int b = 0; b < KK; ++b)
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) {
                if constexpr (KAHAN) {
                    // combine (sum, comp) pairs of two lanes compensatedly
                    const T os = shfl_xor(acc[a][b], s), oc = shfl_xor(cmp[a][b], s);
                    T ss = acc[a][b], cc = cmp[a][b];
                    kbn_add(ss, cc, os);
                    kbn_add(ss, cc, oc);
                    acc[a][b] = ss;
                    cmp[a][b] = cc;
                } else {
                    acc[a][b] = O::add(acc[a][b], shfl_xor(acc[a][b], s));
                }
            }
    if (lane == 0) {
#pragma unroll
        for (int a = 0; a < MM; ++a)
#pragma unroll
            for (int b = 0; b < KK; ++b) {
                red[warp][b * MM + a] = acc[a][b];
                if constexpr (KAHAN) redc[warp][b * MM + a] = cmp[a][b];
            }
    }
    __syncthreads();
    if (int(threadIdx.x) < MM * KK) {
        const int a = threadIdx.x % MM, b = threadIdx.x / MM;
        if (a < m && b < k) {
            T s = O::zero(), c = O::zero();
            for (int q = 0; q < kT / 32; ++q) {
                if constexpr (KAHAN) {
                    kbn_add(s, c, red[q][threadIdx.x]);
                    kbn_add(s, c, redc[q][threadIdx.x]);
                } else {
                    s = O::add(s, red[q][threadIdx.x]);
                }
            }
            const gidx cell = gidx(b) * m + a;  // col-major m x k like tsm.hpp:145
            partial[gidx(blockIdx.x) * m * k + cell] = s;
            if constexpr (KAHAN) pcomp[gidx(blockIdx.x) * m * k + cell] = c;
        }
    }
}

// TSMTTSM 8 x 8 (double, compact rows; measured 2.40 -> 2.35 ms at N = 1e8 with LPR = 2,
// UR = 2; LPR = 4 / 8 and UR = 4 no better, profiles r2ac): LPR lanes share a row -- lane q of the group
// keeps the (8/LPR) x 8 slice of the cell block for V columns q*8/LPR.., loads its slice of
// the V row and the whole W row (the group's identical W addresses merge into one
// request), so a lane holds 8*8/LPR accumulators instead of 64 (more lanes resident, more
// rows in flight); UR rows per lane per batch.
template <int LPR, int UR>
__global__ void __launch_bounds__(kT) tsmttsm_split8_kernel(const double* __restrict__ v, const double* __restrict__ w,
                                                            gidx n, gidx rows_per_cta, double* partial) {
    constexpr int MA = 8 / LPR;  // V columns (cell rows) per lane
    __shared__ double red[kT / 32][64];
    double acc[MA][8];
#pragma unroll
    for (int a = 0; a < MA; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
    const int q = threadIdx.x % LPR;
    const gidx r0 = gidx(blockIdx.x) * rows_per_cta;
    const gidx r1 = min(n, r0 + rows_per_cta);
    constexpr int kRowsPerPass = kT / LPR;
    gidx i = r0 + threadIdx.x / LPR;
    for (; i + gidx(UR - 1) * kRowsPerPass < r1; i += gidx(UR) * kRowsPerPass) {
        double vr[UR][MA], wr[UR][8];
#pragma unroll
        for (int u = 0; u < UR; ++u) {
            load_row<double, MA>(v + (i + gidx(u) * kRowsPerPass) * 8 + MA * q, vr[u]);
            load_row<double, 8>(w + (i + gidx(u) * kRowsPerPass) * 8, wr[u]);
        }
#pragma unroll
        for (int u = 0; u < UR; ++u)
#pragma unroll
            for (int a = 0; a < MA; ++a)
#pragma unroll
                for (int b = 0; b < 8; ++b) acc[a][b] = fma(vr[u][a], wr[u][b], acc[a][b]);
    }
    for (; i < r1; i += kRowsPerPass) {
        double vr[MA], wr[8];
        load_row<double, MA>(v + i * 8 + MA * q, vr);
        load_row<double, 8>(w + i * 8, wr);
#pragma unroll
        for (int a = 0; a < MA; ++a)
#pragma unroll
            for (int b = 0; b < 8; ++b) acc[a][b] = fma(vr[a], wr[b], acc[a][b]);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int a = 0; a < MA; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b)
#pragma unroll
            for (int s = 16; s >= LPR; s >>= 1) acc[a][b] += __shfl_xor_sync(0xffffffffu, acc[a][b], s);
    if (lane < LPR) {
#pragma unroll
        for (int a = 0; a < MA; ++a)
#pragma unroll
            for (int b = 0; b < 8; ++b) red[warp][b * 8 + MA * q + a] = acc[a][b];  // col-major 8 x 8
    }
    __syncthreads();
    if (threadIdx.x < 64) {
        double s = 0.0;
        for (int t = 0; t < kT / 32; ++t) s += red[t][threadIdx.x];
        partial[gidx(blockIdx.x) * 64 + threadIdx.x] = s;
    }
}

// TSMTTSM, general sizes: rows staged in shared memory 64 at a time (coalesced,
// contiguous copy when V/W are compact), each thread owns a TM x TK tile of cells.
template <class T, int TM, int TK, bool KAHAN>
__global__ void __launch_bounds__(kT) tsmttsm_tile_kernel(const T* __restrict__ v, gidx vs, const T* __restrict__ w,
                                                          gidx ws, gidx n, int m, int k, gidx rows_per_cta, T* partial,
                                                          T* pcomp) {
    using O = Ops<T>;
    constexpr int RT = 64;
    extern __shared__ unsigned char smem_raw[];
    T* vsm = reinterpret_cast<T*>(smem_raw);  // [RT][m]
    T* wsm = vsm + RT * m;                     // [RT][k]
    const int tm = (m + TM - 1) / TM, tk = (k + TK - 1) / TK;
    const int tid = threadIdx.x + blockIdx.y * kT;  // cell tile index
    const bool active = tid < tm * tk;
    const int a0 = (tid % tm) * TM, b0 = (tid / tm) * TK;
    T acc[TM][TK], cmp[TM][TK];
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TK; ++b) acc[a][b] = cmp[a][b] = O::zero();
    const gidx r0 = gidx(blockIdx.x) * rows_per_cta;
    const gidx r1 = min(n, r0 + rows_per_cta);
    for (gidx rb = r0; rb < r1; rb += RT) {
        const int nr = int(min(gidx(RT), r1 - rb));
        __syncthreads();
        for (int t = threadIdx.x; t < nr * m; t += kT) vsm[t] = O::conj(v[(rb + t / m) * vs + t % m]);
        for (int t = threadIdx.x; t < nr * k; t += kT) wsm[t] = w[(rb + t / k) * ws + t % k];
        __syncthreads();
        if (!active) continue;
        for (int r = 0; r < nr; ++r) {
            T va[TM], wb[TK];
#pragma unroll
            for (int a = 0; a < TM; ++a) va[a] = a0 + a < m ? vsm[r * m + a0 + a] : O::zero();
#pragma unroll
            for (int b = 0; b < TK; ++b) wb[b] = b0 + b < k ? wsm[r * k + b0 + b] : O::zero();
#pragma unroll
            for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TK; ++b) {
                    if constexpr (KAHAN) kbn_add(acc[a][b], cmp[a][b], O::mul(va[a], wb[b]));
                    else acc[a][b] = O::fma(va[a], wb[b], acc[a][b]);
                }
        }
    }
    if (!active) return;
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TK; ++b)
            if (a0 + a < m && b0 + b < k) {
                const gidx cell = gidx(b0 + b) * m + a0 + a;
                partial[gidx(blockIdx.x) * m * k + cell] = acc[a][b];
                if constexpr (KAHAN) pcomp[gidx(blockIdx.x) * m * k + cell] = cmp[a][b];
            }
}

// TSMM, row-major V/W: a thread computes RT rows x KT columns of W; X (m x k,
// row-major) lives in shared memory.  EXACT keeps the reference's rounding
// (separate mul/add, m ascending) for the bandwidth-bound shapes.
template <class T, int RT, int KT, bool EXACT>
__global__ void __launch_bounds__(kT) tsmm_tile_kernel(T* __restrict__ w, gidx ws, const T* __restrict__ v, gidx vs,
                                                       const T* __restrict__ xcm, gidx n, int m, int k, T alpha, T beta,
                                                       int beta_zero) {
    using O = Ops<T>;
    extern __shared__ unsigned char smem_raw[];
    T* xs = reinterpret_cast<T*>(smem_raw);  // row-major [m][k]
    for (int t = threadIdx.x; t < m * k; t += kT) xs[t] = xcm[gidx(t % k) * m + t / k];
    __syncthreads();
    const int nkb = (k + KT - 1) / KT;
    const gidx nrb = (n + RT - 1) / RT;
    const gidx items = nrb * nkb;
    for (gidx it = blockIdx.x * gidx(kT) + threadIdx.x; it < items; it += gidx(gridDim.x) * kT) {
        const gidx rb = it / nkb;
        const int kb = int(it - rb * nkb);
        const gidx i0 = rb * RT;
        const int c0 = kb * KT;
        T tmp[RT][KT];
#pragma unroll
        for (int r = 0; r < RT; ++r)
#pragma unroll
            for (int e = 0; e < KT; ++e) tmp[r][e] = O::zero();
        for (int mm = 0; mm < m; ++mm) {
            T vr[RT], xk[KT];
#pragma unroll
            for (int r = 0; r < RT; ++r) vr[r] = i0 + r < n ? __ldg(v + (i0 + r) * vs + mm) : O::zero();
#pragma unroll
            for (int e = 0; e < KT; ++e) xk[e] = c0 + e < k ? xs[mm * k + c0 + e] : O::zero();
#pragma unroll
            for (int r = 0; r < RT; ++r)
#pragma unroll
                for (int e = 0; e < KT; ++e) tmp[r][e] = madd<T, EXACT>(tmp[r][e], vr[r], xk[e]);
        }
#pragma unroll
        for (int r = 0; r < RT; ++r) {
            if (i0 + r >= n) break;
#pragma unroll
            for (int e = 0; e < KT; ++e) {
                if (c0 + e >= k) break;
                T* wp = w + (i0 + r) * ws + c0 + e;
                *wp = beta_zero ? O::mul(alpha, tmp[r][e]) : O::add(O::mul(alpha, tmp[r][e]), O::mul(beta, *wp));
            }
        }
    }
}

// TSMM with the reference's rounding (m*k <= 64, HBM-bound): one thread per
// row, the V row and the W row moved with vector accesses, X broadcast from
// shared memory; tmp[e] = sum over m ascending of V[i,m]*X[m,e], each product and
// sum rounded separately (tsm.hpp:51-68).
// R > 1: a thread computes R consecutive rows, moving their V and W rows with one vector
// access each (1 x 1: four rows per LDG.256 / STG.256); same arithmetic per row.
template <class T, int M, int K, int R>
__device__ __forceinline__ void tsmm_rows_chunk(T* __restrict__ w, const T* __restrict__ v, const T* xs, gidx i,
                                                T alpha, T beta, int beta_zero) {
    using O = Ops<T>;
    T vr[R * M], out[R * K];
    load_row<T, R * M>(v + i * M, vr);
    T old[R * K];
    if (!beta_zero) load_row<T, R * K>(w + i * K, old);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        T tmp[K];
#pragma unroll
        for (int e = 0; e < K; ++e) tmp[e] = O::zero();
#pragma unroll
        for (int mm = 0; mm < M; ++mm)
#pragma unroll
            for (int e = 0; e < K; ++e) tmp[e] = O::add(tmp[e], O::mul(vr[r * M + mm], xs[mm * K + e]));
#pragma unroll
        for (int e = 0; e < K; ++e)
            out[r * K + e] = beta_zero ? O::mul(alpha, tmp[e]) : O::add(O::mul(alpha, tmp[e]), O::mul(beta, old[r * K + e]));
    }
    store_row<T, R * K>(w + i * K, out);
}

template <class T, int M, int K, int R>
__global__ void __launch_bounds__(kT) tsmm_chunk_kernel(T* __restrict__ w, const T* __restrict__ v,
                                                        const T* __restrict__ xcm, gidx n, T alpha, T beta,
                                                        int beta_zero) {
    __shared__ T xs[M * K];  // row-major
    for (int t = threadIdx.x; t < M * K; t += kT) xs[t] = xcm[(t % K) * M + t / K];
    __syncthreads();
    const gidx nch = n / R;
    for (gidx c = blockIdx.x * gidx(kT) + threadIdx.x; c < nch; c += gidx(gridDim.x) * kT)
        tsmm_rows_chunk<T, M, K, R>(w, v, xs, c * R, alpha, beta, beta_zero);
    if (blockIdx.x == 0 && threadIdx.x < n - nch * R)  // the last n % R rows one by one
        tsmm_rows_chunk<T, M, K, 1>(w, v, xs, nch * R + threadIdx.x, alpha, beta, beta_zero);
}

template <class T, int M, int K>
__global__ void __launch_bounds__(kT) tsmm_row_kernel(T* __restrict__ w, const T* __restrict__ v,
                                                      const T* __restrict__ xcm, gidx n, T alpha, T beta,
                                                      int beta_zero) {
    using O = Ops<T>;
    __shared__ T xs[M * K];  // row-major
    for (int t = threadIdx.x; t < M * K; t += kT) xs[t] = xcm[(t % K) * M + t / K];
    __syncthreads();
    for (gidx i = blockIdx.x * gidx(kT) + threadIdx.x; i < n; i += gidx(gridDim.x) * kT) {
        T vr[M], tmp[K], out[K];
        load_row<T, M>(v + i * M, vr);
#pragma unroll
        for (int e = 0; e < K; ++e) tmp[e] = O::zero();
#pragma unroll
        for (int mm = 0; mm < M; ++mm)
#pragma unroll
            for (int e = 0; e < K; ++e) tmp[e] = O::add(tmp[e], O::mul(vr[mm], xs[mm * K + e]));
        if (beta_zero) {
#pragma unroll
            for (int e = 0; e < K; ++e) out[e] = O::mul(alpha, tmp[e]);
        } else {
            T old[K];
            load_row<T, K>(w + i * K, old);
#pragma unroll
            for (int e = 0; e < K; ++e) out[e] = O::add(O::mul(alpha, tmp[e]), O::mul(beta, old[e]));
        }
        store_row<T, K>(w + i * K, out);
    }
}

bool compact_rows(const DenseMat& m) { return !m.scattered() && m.order == Order::row_major; }

template <class T>
T scalar_or(const void* p, T dflt) {
    if (!p) return dflt;
    T v;
    std::memcpy(&v, p, sizeof(T));
    return v;
}

template <class T>
bool is_zero(const T& v) {
    unsigned char z[sizeof(T)] = {};
    T zero;
    std::memcpy(&zero, z, sizeof(T));
    // exact +0 or -0 in every component
    if constexpr (scalar_traits<T>::is_complex) return v.re == 0 && v.im == 0;
    else return v == 0;
}

int grid_cap(gidx work, const DeviceRuntime& rt, int per_sm = 8) {
    return int(std::max<gidx>(1, std::min<gidx>((work + kT - 1) / kT, gidx(rt.num_sms) * per_sm)));
}

void check_same_device(const DenseMat& a, const DenseMat& b) {
    SK_REQUIRE(a.device == b.device, errc::invalid_arg, "operands must live on the same device");
}

}  // namespace

void tsmttsm(DenseMat& x, const DenseMat& v_in, const DenseMat& w_in, const void* alpha, const void* beta, bool kahan) {
    SK_REQUIRE(v_in.nrows == w_in.nrows, errc::shape_mismatch, "V and W must have equal row counts");
    SK_REQUIRE(x.nrows == v_in.ncols && x.ncols == w_in.ncols, errc::shape_mismatch, "X must be (V cols) x (W cols)");
    SK_REQUIRE(x.dt == v_in.dt && x.dt == w_in.dt, errc::invalid_arg, "datatype mismatch between x and v");
    DenseMat v = v_in, w = w_in;
    Staged xs(x, true), vs(v, true), wsg(w, true);
    check_same_device(xs.dev, vs.dev);
    check_same_device(xs.dev, wsg.dev);
    const int dev = xs.dev.device;
    DeviceGuard g(dev);
    auto& rt = runtime(dev);
    const lidx m = x.nrows, k = x.ncols;
    const gidx n = v.nrows;
    const gidx cells = gidx(m) * k;
    const std::size_t es = x.esize();
    if (!is_complex(x.dt) && compact_rows(vs.dev) && compact_rows(wsg.dev) && n > 0) {
        const int nparts = int(std::max<gidx>(1, std::min<gidx>(gidx(rt.num_sms) * (cells <= 4 ? SK_TT_PARTS_SMALL : 4), (n + 255) / 256)));
        const gidx rows_per = (n + nparts - 1) / nparts;
        auto* part = static_cast<unsigned char*>(rt.scratch_bytes(std::size_t(nparts) * cells * es * 2 + 256));
        DAcc xa = dacc(xs.dev);
        auto p2 = [](int q) { return q <= 1 ? 1 : q <= 2 ? 2 : q <= 4 ? 4 : 8; };
        visit_dt(x.dt, [&]<class T>() {
            if constexpr (!scalar_traits<T>::is_complex) {
                T* p = reinterpret_cast<T*>(part);
                T* pc = p + std::size_t(nparts) * cells;
                const T a = scalar_or<T>(alpha, Ops<T>::one()), b = scalar_or<T>(beta, Ops<T>::zero());
                const T* vp = reinterpret_cast<const T*>(vs.dev.data);
                const T* wp = reinterpret_cast<const T*>(wsg.dev.data);
                const gidx vst = vs.dev.stride, wst = wsg.dev.stride;
                int used = 0;
                if constexpr (std::is_same_v<T, double>) {
                    if (!kahan && cells >= SK_TT_DMMA_MIN_CELLS && vst == m && wst == k)
                        used = tsmttsm_dmma_partials(vp, wp, n, m, k, p, nparts, rt);
                }
                if (used > 0) {
                    tsmttsm_final_kernel<T, false><<<int((cells + 127) / 128), 128, 0, rt.stream>>>(p, pc, used, m, k, xa, a, b);
                    return 0;
                }
                // chunked path: 1 x 1 and 2 x 2 (double) with compact, 32-byte aligned rows
                const bool chunk = SK_TSM_CHUNK && std::is_same_v<T, double> && !kahan && m == k && (m == 1 || m == 2) &&
                                   vst == m && wst == k && reinterpret_cast<std::uintptr_t>(vp) % 32 == 0 &&
                                   reinterpret_cast<std::uintptr_t>(wp) % 32 == 0;
                if (chunk) {
                    auto goc = [&]<int MK>() {
                        constexpr int R = 32 / (MK * int(sizeof(T)));
                        const gidx rp = (rows_per + R - 1) / R * R;  // CTA ranges start on a chunk
                        const int np = int((n + rp - 1) / rp);
                        tsmttsm_reg_kernel<T, MK, MK, false, R><<<np, kT, 0, rt.stream>>>(vp, vst, wp, wst, n, m, k, rp, p,
                                                                                         pc);
                        CK(cudaGetLastError());
                        tsmttsm_final_kernel<T, false><<<int((cells + 127) / 128), 128, 0, rt.stream>>>(p, pc, np, m, k, xa,
                                                                                                        a, b);
                    };
                    if (m == 1) goc.template operator()<1>();
                    else goc.template operator()<2>();
                    return 0;
                }
                if (SK_TSM_PAIR8 && std::is_same_v<T, double> && !kahan && m == 8 && k == 8 && vst == 8 && wst == 8 &&
                    reinterpret_cast<std::uintptr_t>(vp) % 32 == 0 && reinterpret_cast<std::uintptr_t>(wp) % 32 == 0) {
                    if constexpr (std::is_same_v<T, double>) {
                        tsmttsm_split8_kernel<SK_TT_SPLIT_LPR, SK_TT_PAIR_UR><<<nparts, kT, 0, rt.stream>>>(vp, wp, n, rows_per, p);
                        CK(cudaGetLastError());
                        tsmttsm_final_kernel<T, false><<<int((cells + 127) / 128), 128, 0, rt.stream>>>(p, pc, nparts, m,
                                                                                                        k, xa, a, b);
                    }
                    return 0;
                }
                // the Kahan register kernel keeps sum + compensation of every cell: an 8 x 8
                // block would not fit the register file (1.1 KB of spills), so it takes the
                // shared-memory tile kernel below
                const bool kahan_regs_ok = !kahan || p2(m) * p2(k) <= 32;
                if (m <= 8 && k <= 8 && kahan_regs_ok) {
                    auto go = [&]<int MM, int KK>() {
                        if constexpr (MM * KK <= 32) {
                            if (kahan) {
                                tsmttsm_reg_kernel<T, MM, KK, true><<<nparts, kT, 0, rt.stream>>>(vp, vst, wp, wst, n, m, k,
                                                                                                 rows_per, p, pc);
                                return;
                            }
                        }
                        tsmttsm_reg_kernel<T, MM, KK, false><<<nparts, kT, 0, rt.stream>>>(vp, vst, wp, wst, n, m, k, rows_per, p, pc);
                    };
                    auto gok = [&]<int MM>() {
                        switch (p2(k)) {
                            case 1: go.template operator()<MM, 1>(); break;
                            case 2: go.template operator()<MM, 2>(); break;
                            case 4: go.template operator()<MM, 4>(); break;
                            default: go.template operator()<MM, 8>(); break;
                        }
                    };
                    switch (p2(m)) {
                        case 1: gok.template operator()<1>(); break;
                        case 2: gok.template operator()<2>(); break;
                        case 4: gok.template operator()<4>(); break;
                        default: gok.template operator()<8>(); break;
                    }
                } else {
                    const std::size_t smem = 64 * std::size_t(m + k) * es;
                    SK_REQUIRE(smem <= 200 * 1024, errc::unsupported, "tsmttsm: V/W rows too wide");
                    auto go = [&]<int TM, int TK>() {
                        const int tiles = ((m + TM - 1) / TM) * ((k + TK - 1) / TK);
                        const dim3 grid(nparts, (tiles + kT - 1) / kT);
                        if (kahan) {
                            auto kern = tsmttsm_tile_kernel<T, TM, TK, true>;
                            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
                            kern<<<grid, kT, smem, rt.stream>>>(vp, vst, wp, wst, n, m, k, rows_per, p, pc);
                        } else {
                            auto kern = tsmttsm_tile_kernel<T, TM, TK, false>;
                            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
                            kern<<<grid, kT, smem, rt.stream>>>(vp, vst, wp, wst, n, m, k, rows_per, p, pc);
                        }
                    };
                    if (cells <= 256) go.template operator()<1, 1>();
                    else if (cells <= 1024) go.template operator()<2, 2>();
                    else go.template operator()<4, 4>();
                }
                CK(cudaGetLastError());
                if (kahan)
                    tsmttsm_final_kernel<T, true><<<int((cells + 127) / 128), 128, 0, rt.stream>>>(p, pc, nparts, m, k, xa, a, b);
                else
                    tsmttsm_final_kernel<T, false><<<int((cells + 127) / 128), 128, 0, rt.stream>>>(p, pc, nparts, m, k, xa, a, b);
            }
            return 0;
        });
        CK(cudaGetLastError());
        xs.write_back();
        finish(rt);
        return;
    }
    const int cell_tiles = int((cells + kT * kCellsPerThread - 1) / (kT * kCellsPerThread));
    // CTAs over rows: enough to fill the machine, rows per CTA a multiple of the tile
    const int want = std::max(1, rt.num_sms * 2 / cell_tiles);
    gidx rows_per = std::max<gidx>(kRowTile, (n + want - 1) / want);
    rows_per = (rows_per + kRowTile - 1) / kRowTile * kRowTile;
    const int nparts = int(std::max<gidx>(1, (n + rows_per - 1) / rows_per));
    const std::size_t smem = std::size_t(kRowTile) * (m + k) * es;
    SK_REQUIRE(smem <= 200 * 1024, errc::unsupported, "tsmttsm: V/W rows too wide for the staged kernel");
    auto* part = static_cast<unsigned char*>(rt.scratch_bytes(std::size_t(nparts) * cells * es * 2 + 256));
    DAcc va = dacc(vs.dev), wa = dacc(wsg.dev), xa = dacc(xs.dev);
    visit_dt(x.dt, [&]<class T>() {
        T* p = reinterpret_cast<T*>(part);
        T* pc = p + std::size_t(nparts) * cells;
        const T a = scalar_or<T>(alpha, Ops<T>::one()), b = scalar_or<T>(beta, Ops<T>::zero());
        auto launch = [&](auto kern, auto fin) {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            if (n > 0) kern<<<dim3(nparts, cell_tiles), kT, smem, rt.stream>>>(va, wa, n, m, k, rows_per, p, pc);
            else CK(cudaMemsetAsync(p, 0, std::size_t(nparts) * cells * es * 2, rt.stream));
            fin<<<int((cells + 127) / 128), 128, 0, rt.stream>>>(p, pc, nparts, m, k, xa, a, b);
        };
        if (kahan) launch(tsmttsm_partial_kernel<T, true>, tsmttsm_final_kernel<T, true>);
        else launch(tsmttsm_partial_kernel<T, false>, tsmttsm_final_kernel<T, false>);
        return 0;
    });
    CK(cudaGetLastError());
    xs.write_back();
    finish(rt);
}

void tsmm(DenseMat& w, const DenseMat& v_in, const DenseMat& x_in, const void* alpha, const void* beta) {
    SK_REQUIRE(w.nrows == v_in.nrows, errc::shape_mismatch, "V and W must have equal row counts");
    SK_REQUIRE(x_in.nrows == v_in.ncols && x_in.ncols == w.ncols, errc::shape_mismatch, "X must be (V cols) x (W cols)");
    SK_REQUIRE(w.data != v_in.data, errc::invalid_arg, "V and W must be distinct");
    SK_REQUIRE(w.dt == v_in.dt && w.dt == x_in.dt, errc::invalid_arg, "datatype mismatch between w and v");
    DenseMat v = v_in, x = x_in;
    const lidx m = x.nrows, k = x.ncols;
    const gidx n = v.nrows;
    bool beta_zero = false;
    visit_dt(w.dt, [&]<class T>() {
        beta_zero = is_zero(scalar_or<T>(beta, Ops<T>::zero()));
        return 0;
    });
    Staged wsg(w, !beta_zero), vs(v, true), xs(x, true);
    check_same_device(wsg.dev, vs.dev);
    check_same_device(wsg.dev, xs.dev);
    const int dev = wsg.dev.device;
    DeviceGuard g(dev);
    auto& rt = runtime(dev);
    const std::size_t es = w.esize();
    auto* xcm = static_cast<unsigned char*>(rt.scratch_bytes(std::size_t(m) * k * es + 256));
    DAcc wa = dacc(wsg.dev), va = dacc(vs.dev), xa = dacc(xs.dev);
    const std::size_t xbytes = std::size_t(m) * k * es;
    const int x_in_smem = xbytes <= 96 * 1024 ? 1 : 0;
    const bool exact = gidx(m) * k <= 64;
    const bool fast = !is_complex(w.dt) && compact_rows(vs.dev) && compact_rows(wsg.dev) && x_in_smem && n > 0;
    visit_dt(w.dt, [&]<class T>() {
        T* xc = reinterpret_cast<T*>(xcm);
        x_colmajor_kernel<T><<<int((gidx(m) * k + 255) / 256), 256, 0, rt.stream>>>(xa, m, k, xc);
        const T a = scalar_or<T>(alpha, Ops<T>::one()), b = scalar_or<T>(beta, Ops<T>::zero());
        if constexpr (!scalar_traits<T>::is_complex) {
            if (fast) {
                T* wp = reinterpret_cast<T*>(wsg.dev.data);
                const T* vp = reinterpret_cast<const T*>(vs.dev.data);
                const gidx wst = wsg.dev.stride, vst = vs.dev.stride;
                if constexpr (std::is_same_v<T, double>) {
                    if (!exact && vst == m && wst == k && tsmm_dmma(wp, vp, xc, n, m, k, a, b, beta_zero, rt)) return 0;
                }
                auto pow2 = [](lidx q) { return q == 1 || q == 2 || q == 4 || q == 8; };
                // 1 x 1 and 2 x 2 (double, 32-byte aligned): R rows per thread and vector access
                if (SK_TSM_CHUNK && std::is_same_v<T, double> && m == k && (m == 1 || m == 2) && vst == m &&
                    wst == k && reinterpret_cast<std::uintptr_t>(vp) % 32 == 0 &&
                    reinterpret_cast<std::uintptr_t>(wp) % 32 == 0) {
                    auto chunked = [&]<int MK>() {
                        constexpr int R = 32 / (MK * int(sizeof(T)));
                        const gidx nch = std::max<gidx>(1, n / R);
                        const int grid = int(std::max<gidx>(1, std::min<gidx>((nch + kT - 1) / kT, gidx(rt.num_sms) * 8)));
                        tsmm_chunk_kernel<T, MK, MK, R><<<grid, kT, 0, rt.stream>>>(wp, vp, xc, n, a, b,
                                                                                  beta_zero ? 1 : 0);
                    };
                    if (m == 1) chunked.template operator()<1>();
                    else chunked.template operator()<2>();
                    return 0;
                }
                if (exact && pow2(m) && pow2(k) && vst == m && wst == k) {
                    const int grid = int(std::max<gidx>(1, std::min<gidx>((n + kT - 1) / kT, gidx(rt.num_sms) * 8)));
                    auto row = [&]<int M, int K>() {
                        tsmm_row_kernel<T, M, K><<<grid, kT, 0, rt.stream>>>(wp, vp, xc, n, a, b, beta_zero ? 1 : 0);
                    };
                    auto rowk = [&]<int M>() {
                        switch (k) {
                            case 1: row.template operator()<M, 1>(); break;
                            case 2: row.template operator()<M, 2>(); break;
                            case 4: row.template operator()<M, 4>(); break;
                            default: row.template operator()<M, 8>(); break;
                        }
                    };
                    switch (m) {
                        case 1: rowk.template operator()<1>(); break;
                        case 2: rowk.template operator()<2>(); break;
                        case 4: rowk.template operator()<4>(); break;
                        default: rowk.template operator()<8>(); break;
                    }
                    return 0;
                }
                auto go = [&]<int RT, int KT, bool EX>() {
                    auto kern = tsmm_tile_kernel<T, RT, KT, EX>;
                    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(xbytes)));
                    const gidx items = ((n + RT - 1) / RT) * ((k + KT - 1) / KT);
                    const int grid = int(std::max<gidx>(1, std::min<gidx>((items + kT - 1) / kT, gidx(rt.num_sms) * 8)));
                    kern<<<grid, kT, xbytes, rt.stream>>>(wp, wst, vp, vst, xc, n, m, k, a, b, beta_zero ? 1 : 0);
                };
                if (exact) {  // m*k <= 64: one thread per row, all k columns, reference rounding
                    if (k <= 1) go.template operator()<1, 1, true>();
                    else if (k <= 2) go.template operator()<1, 2, true>();
                    else if (k <= 4) go.template operator()<1, 4, true>();
                    else go.template operator()<1, 8, true>();
                } else if (k <= 4) {
                    go.template operator()<4, 4, false>();
                } else {
                    go.template operator()<4, 8, false>();
                }
                return 0;
            }
        }
        auto launch = [&](auto kern) {
            const std::size_t smem = x_in_smem ? xbytes : 0;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(std::max<std::size_t>(smem, 1))));
            if (n > 0) kern<<<grid_cap(n * k, rt), kT, smem, rt.stream>>>(wa, va, xc, n, m, k, a, b, beta_zero ? 1 : 0, x_in_smem);
        };
        if (exact) launch(tsmm_kernel<T, true>);
        else launch(tsmm_kernel<T, false>);
        return 0;
    });
    CK(cudaGetLastError());
    wsg.write_back();
    finish(rt);
}

void tsmm_inplace(DenseMat& v, const DenseMat& x_in, const void* alpha, const void* beta) {
    SK_REQUIRE(x_in.nrows == x_in.ncols, errc::shape_mismatch, "in-place tsmm requires a square X");
    SK_REQUIRE(x_in.nrows == v.ncols, errc::shape_mismatch, "X must be (V cols) x (V cols)");
    SK_REQUIRE(v.dt == x_in.dt, errc::invalid_arg, "datatype mismatch between v and x");
    const lidx m = x_in.nrows;
    SK_REQUIRE(m <= kT * kCellsPerThread, errc::unsupported, "tsmm_inplace: X wider than 4096 columns");
    DenseMat x = x_in;
    Staged vs(v, true), xs(x, true);
    check_same_device(vs.dev, xs.dev);
    const int dev = vs.dev.device;
    DeviceGuard g(dev);
    auto& rt = runtime(dev);
    const std::size_t es = v.esize();
    const gidx n = v.nrows;
    auto* xcm = static_cast<unsigned char*>(rt.scratch_bytes(std::size_t(m) * m * es + 256));
    DAcc va = dacc(vs.dev), xa = dacc(xs.dev);
    const lidx rows = std::max<lidx>(1, (kT * kCellsPerThread) / m);
    const bool exact = gidx(m) * m <= 64;
    visit_dt(v.dt, [&]<class T>() {
        T* xc = reinterpret_cast<T*>(xcm);
        x_colmajor_kernel<T><<<int((gidx(m) * m + 255) / 256), 256, 0, rt.stream>>>(xa, m, m, xc);
        const T a = scalar_or<T>(alpha, Ops<T>::one()), b = scalar_or<T>(beta, Ops<T>::zero());
        const int grid = int((n + rows - 1) / rows);
        if (grid > 0) {
            if (exact) tsmm_inplace_kernel<T, true><<<grid, kT, 0, rt.stream>>>(va, xc, n, m, rows, a, b);
            else tsmm_inplace_kernel<T, false><<<grid, kT, 0, rt.stream>>>(va, xc, n, m, rows, a, b);
        }
        return 0;
    });
    CK(cudaGetLastError());
    vs.write_back();
    finish(rt);
}

// tsm.hpp:281-305
void gemm(DenseMat& c, const DenseMat& a_in, const DenseMat& b_in, const void* alpha, const void* beta, Trans ta,
          Trans tb) {
    constexpr lidx small = 64;  // small_dim_bound tsm.hpp:13
    const lidx a_rows = ta == Trans::none ? a_in.nrows : a_in.ncols;
    const lidx a_cols = ta == Trans::none ? a_in.ncols : a_in.nrows;
    const lidx b_rows = tb == Trans::none ? b_in.nrows : b_in.ncols;
    const lidx b_cols = tb == Trans::none ? b_in.ncols : b_in.nrows;
    SK_REQUIRE(a_cols == b_rows, errc::shape_mismatch, "inner dimensions must agree");
    SK_REQUIRE(c.nrows == a_rows && c.ncols == b_cols, errc::shape_mismatch, "output shape mismatch");
    SK_REQUIRE(c.dt == a_in.dt && c.dt == b_in.dt, errc::invalid_arg, "datatype mismatch between c and a");
    const bool a_tall = a_in.nrows > small && a_in.ncols <= small;
    const bool conj_ok = !is_complex(c.dt) || ta == Trans::conj_transpose;
    if (a_tall && ta != Trans::none && conj_ok && tb == Trans::none && b_in.nrows == a_in.nrows && b_in.ncols <= small) {
        tsmttsm(c, a_in, b_in, alpha, beta, false);
        return;
    }
    if (a_tall && ta == Trans::none && tb == Trans::none && b_in.nrows <= small && b_in.ncols <= small) {
        tsmm(c, a_in, b_in, alpha, beta);
        return;
    }
    DenseMat a = a_in, b = b_in;
    Staged cs(c, true), as(a, true), bs(b, true);
    const int dev = cs.dev.device;
    DeviceGuard g(dev);
    auto& rt = runtime(dev);
    DAcc ca = dacc(cs.dev), aa = dacc(as.dev), ba = dacc(bs.dev);
    visit_dt(c.dt, [&]<class T>() {
        const T al = scalar_or<T>(alpha, Ops<T>::one()), be = scalar_or<T>(beta, Ops<T>::zero());
        const gidx tot = gidx(c.nrows) * c.ncols;
        gemm_naive_kernel<T><<<int((tot + 255) / 256), 256, 0, rt.stream>>>(ca, aa, ba, c.nrows, c.ncols, a_cols,
                                                                             int(ta), int(tb), al, be);
        return 0;
    });
    CK(cudaGetLastError());
    cs.write_back();
    finish(rt);
}

}  // namespace skb
