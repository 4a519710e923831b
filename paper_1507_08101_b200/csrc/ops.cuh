// Device arithmetic with explicit rounding.  Every multiply and add is issued
// as its own IEEE round-to-nearest operation (__dmul_rn/__dadd_rn, never a
// contracted FMA) so the SpMV/BLAS-1 results are bit-identical to the
// reference's Release build, which has no FMA (x86-64 baseline; SURVEY §7
// "FMA vs reference rounding").  The sweeps are HBM-bound, so the second FP64
// instruction per nonzero costs nothing measurable.
//
// Complex products follow the naive formula of libstdc++ / __muldc3 for finite
// operands: (ac - bd) + i(ad + bc), each term rounded separately.
#pragma once

#include "core.cuh"

namespace skb {

template <class T>
struct Ops;

template <>
struct Ops<double> {
    using T = double;
    static __host__ __device__ __forceinline__ T zero() { return 0.0; }
    static __host__ __device__ __forceinline__ T one() { return 1.0; }
#ifdef __CUDA_ARCH__
    static __device__ __forceinline__ T mul(T a, T b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ T add(T a, T b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ T sub(T a, T b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ T fma(T a, T b, T c) { return __fma_rn(a, b, c); }
#else
    static T mul(T a, T b) { return a * b; }
    static T add(T a, T b) { return a + b; }
    static T sub(T a, T b) { return a - b; }
    static T fma(T a, T b, T c) { return a * b + c; }
#endif
    static __host__ __device__ __forceinline__ T conj(T a) { return a; }
    static __host__ __device__ __forceinline__ double abs2(T a) { return a * a; }
};

template <>
struct Ops<float> {
    using T = float;
    static __host__ __device__ __forceinline__ T zero() { return 0.0f; }
    static __host__ __device__ __forceinline__ T one() { return 1.0f; }
#ifdef __CUDA_ARCH__
    static __device__ __forceinline__ T mul(T a, T b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ T add(T a, T b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ T sub(T a, T b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ T fma(T a, T b, T c) { return __fmaf_rn(a, b, c); }
#else
    static T mul(T a, T b) { return a * b; }
    static T add(T a, T b) { return a + b; }
    static T sub(T a, T b) { return a - b; }
    static T fma(T a, T b, T c) { return a * b + c; }
#endif
    static __host__ __device__ __forceinline__ T conj(T a) { return a; }
    static __host__ __device__ __forceinline__ double abs2(T a) { return double(a) * a; }
};

template <class R>
struct Ops<cplx<R>> {
    using T = cplx<R>;
    using RO = Ops<R>;
    static __host__ __device__ __forceinline__ T zero() { return T{R(0), R(0)}; }
    static __host__ __device__ __forceinline__ T one() { return T{R(1), R(0)}; }
    static __device__ __forceinline__ T mul(T a, T b) {
        return T{RO::sub(RO::mul(a.re, b.re), RO::mul(a.im, b.im)),
                 RO::add(RO::mul(a.re, b.im), RO::mul(a.im, b.re))};
    }
    static __device__ __forceinline__ T add(T a, T b) { return T{RO::add(a.re, b.re), RO::add(a.im, b.im)}; }
    static __device__ __forceinline__ T sub(T a, T b) { return T{RO::sub(a.re, b.re), RO::sub(a.im, b.im)}; }
    // complex fused multiply-add (used only by the compute-bound TSM kernels)
    static __device__ __forceinline__ T fma(T a, T b, T c) {
        return T{RO::fma(-a.im, b.im, RO::fma(a.re, b.re, c.re)), RO::fma(a.im, b.re, RO::fma(a.re, b.im, c.im))};
    }
    static __host__ __device__ __forceinline__ T conj(T a) { return T{a.re, -a.im}; }
    static __host__ __device__ __forceinline__ double abs2(T a) {
        return double(a.re) * a.re + double(a.im) * a.im;
    }
};

// ----------------------------------------------------------- memory access --

// Streaming read of matrix data (values / column indices): read once, keep it
// out of L1 (L1::no_allocate) and mark it evict-first in L2 through an L2 cache
// policy, so the RHS block keeps the caches.
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double ld_stream(const double* p, unsigned long long pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_stream(const float* p, unsigned long long pol) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int ld_stream(const int* p, unsigned long long pol) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ cdouble ld_stream(const cdouble* p, unsigned long long pol) {
    cdouble v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.re), "=d"(v.im)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ cfloat ld_stream(const cfloat* p, unsigned long long pol) {
    cfloat v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
                 : "=f"(v.re), "=f"(v.im)
                 : "l"(p), "l"(pol));
    return v;
}

// Vector of N elements of T loaded/stored as one access when the byte size
// allows (8, 16 or 32 bytes; 32-byte accesses are sm_100 LDG.256/STG.256).
template <class T, int N>
struct Vec {
    T v[N];
};

template <int BYTES>
struct RawVec;
template <>
struct RawVec<4> {
    using type = unsigned int;
};
template <>
struct RawVec<8> {
    using type = uint2;
};
template <>
struct RawVec<16> {
    using type = uint4;
};

// x gathers: cached (L1 + L2 normal) read-only loads.  RHS rows are reused by
// neighbouring rows of the sweep, so they should stay in L1/L2.
template <class T, int N>
__device__ __forceinline__ Vec<T, N> ld_x(const T* p) {
    Vec<T, N> r;
    constexpr int B = int(sizeof(T)) * N;
    if constexpr (B == 32) {
        unsigned long long a, b, c, d;
        asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
        unsigned long long tmp[4] = {a, b, c, d};
        memcpy(&r, tmp, 32);
    } else if constexpr (B == 4 || B == 8 || B == 16) {
        using R = typename RawVec<B>::type;
        R raw = __ldg(reinterpret_cast<const R*>(p));
        memcpy(&r, &raw, B);
    } else if constexpr (B % 32 == 0) {  // 64-/128-byte lane vectors: consecutive 32-byte loads
        constexpr int M = 32 / int(sizeof(T));
#pragma unroll
        for (int q = 0; q < N / M; ++q) {
            const Vec<T, M> h = ld_x<T, M>(p + q * M);
#pragma unroll
            for (int i = 0; i < M; ++i) r.v[q * M + i] = h.v[i];
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) r.v[i] = p[i];
    }
    return r;
}

// Plain (coherent) vector load/store for y/z, which the kernel may also write.
template <class T, int N>
__device__ __forceinline__ Vec<T, N> ld_vec(const T* p) {
    Vec<T, N> r;
    constexpr int B = int(sizeof(T)) * N;
    if constexpr (B == 32) {
        unsigned long long t[4];
        asm volatile("ld.global.v4.u64 {%0, %1, %2, %3}, [%4];"
                     : "=l"(t[0]), "=l"(t[1]), "=l"(t[2]), "=l"(t[3])
                     : "l"(p));
        memcpy(&r, t, 32);
    } else if constexpr (B == 4 || B == 8 || B == 16) {
        using R = typename RawVec<B>::type;
        R raw = *reinterpret_cast<const R*>(p);
        memcpy(&r, &raw, B);
    } else if constexpr (B % 32 == 0) {
        constexpr int M = 32 / int(sizeof(T));
#pragma unroll
        for (int q = 0; q < N / M; ++q) {
            const Vec<T, M> h = ld_vec<T, M>(p + q * M);
#pragma unroll
            for (int i = 0; i < M; ++i) r.v[q * M + i] = h.v[i];
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) r.v[i] = p[i];
    }
    return r;
}

template <class T, int N>
__device__ __forceinline__ void st_vec(T* p, const Vec<T, N>& v) {
    constexpr int B = int(sizeof(T)) * N;
    if constexpr (B == 32) {
        unsigned long long t[4];
        memcpy(t, &v, 32);
        asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(t[0]), "l"(t[1]), "l"(t[2]), "l"(t[3])
                     : "memory");
    } else if constexpr (B == 4 || B == 8 || B == 16) {
        using R = typename RawVec<B>::type;
        R raw;
        memcpy(&raw, &v, B);
        *reinterpret_cast<R*>(p) = raw;
    } else if constexpr (B % 32 == 0) {
        constexpr int M = 32 / int(sizeof(T));
#pragma unroll
        for (int q = 0; q < N / M; ++q) {
            Vec<T, M> h;
#pragma unroll
            for (int i = 0; i < M; ++i) h.v[i] = v.v[q * M + i];
            st_vec<T, M>(p + q * M, h);
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) p[i] = v.v[i];
    }
}

__device__ __forceinline__ unsigned long long l2_evict_last_policy() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// 32-byte RHS gather with an L2 eviction-priority hint (x rows are re-read by the
// neighbouring rows of the sweep; the matrix and y stream past them).
template <class T, int N>
__device__ __forceinline__ Vec<T, N> ld_x_hint(const T* p, unsigned long long pol) {
    static_assert(int(sizeof(T)) * N == 32, "32-byte gathers only");
    Vec<T, N> r;
    unsigned long long t[4];
    asm("ld.global.nc.L2::cache_hint.v4.u64 {%0, %1, %2, %3}, [%4], %5;"
        : "=l"(t[0]), "=l"(t[1]), "=l"(t[2]), "=l"(t[3])
        : "l"(p), "l"(pol));
    memcpy(&r, t, 32);
    return r;
}

template <class T, int N>
__device__ __forceinline__ Vec<T, N> ld_vec_hint(const T* p, unsigned long long pol) {
    static_assert(int(sizeof(T)) * N == 32, "32-byte loads only");
    Vec<T, N> r;
    unsigned long long t[4];
    asm volatile("ld.global.L2::cache_hint.v4.u64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=l"(t[0]), "=l"(t[1]), "=l"(t[2]), "=l"(t[3])
                 : "l"(p), "l"(pol));
    memcpy(&r, t, 32);
    return r;
}

template <class T, int N>
__device__ __forceinline__ void st_vec_hint(T* p, const Vec<T, N>& v, unsigned long long pol) {
    static_assert(int(sizeof(T)) * N == 32, "32-byte stores only");
    unsigned long long t[4];
    memcpy(t, &v, 32);
    asm volatile("st.global.L2::cache_hint.v4.u64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "l"(t[0]), "l"(t[1]), "l"(t[2]),
                 "l"(t[3]), "l"(pol)
                 : "memory");
}

template <class T>
__device__ __forceinline__ T shfl(T v, int src) {
    if constexpr (sizeof(T) == 4) {
        return __shfl_sync(0xffffffffu, v, src);
    } else if constexpr (sizeof(T) == 8) {
        unsigned long long u;
        memcpy(&u, &v, 8);
        u = __shfl_sync(0xffffffffu, u, src);
        T r;
        memcpy(&r, &u, 8);
        return r;
    } else {
        static_assert(sizeof(T) == 16, "unsupported shuffle width");
        unsigned long long u[2];
        memcpy(u, &v, 16);
        u[0] = __shfl_sync(0xffffffffu, u[0], src);
        u[1] = __shfl_sync(0xffffffffu, u[1], src);
        T r;
        memcpy(&r, u, 16);
        return r;
    }
}

template <class T>
__device__ __forceinline__ T shfl_xor(T v, int mask) {
    if constexpr (sizeof(T) == 4) {
        return __shfl_xor_sync(0xffffffffu, v, mask);
    } else if constexpr (sizeof(T) == 8) {
        unsigned long long u;
        memcpy(&u, &v, 8);
        u = __shfl_xor_sync(0xffffffffu, u, mask);
        T r;
        memcpy(&r, &u, 8);
        return r;
    } else {
        unsigned long long u[2];
        memcpy(u, &v, 16);
        u[0] = __shfl_xor_sync(0xffffffffu, u[0], mask);
        u[1] = __shfl_xor_sync(0xffffffffu, u[1], mask);
        T r;
        memcpy(&r, u, 16);
        return r;
    }
}

}  // namespace skb
