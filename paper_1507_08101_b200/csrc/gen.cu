// Synthetic inputs generated on the device: Laplacian stencils
// and counter-hash block vectors.  Used by the benchmark and the tests; the
// CPU oracle regenerates identical values from the same formulas.
#include <algorithm>

#include "objects.cuh"
#include "ops.cuh"

namespace skb {

void exclusive_scan_i64(const gidx* in, gidx* out, gidx n, DeviceRuntime& rt);

namespace {

__device__ __forceinline__ int stencil_neighbours(int points, gidx n, gidx r, gidx* cols) {
    int cnt = 0;
    if (points == 5) {
        const gidx x = r % n, y = r / n;
        if (y > 0) cols[cnt++] = r - n;
        if (x > 0) cols[cnt++] = r - 1;
        cols[cnt++] = r;
        if (x + 1 < n) cols[cnt++] = r + 1;
        if (y + 1 < n) cols[cnt++] = r + n;
    } else {
        const gidx n2 = n * n;
        const gidx x = r % n, y = (r / n) % n, z = r / n2;
        if (z > 0) cols[cnt++] = r - n2;
        if (y > 0) cols[cnt++] = r - n;
        if (x > 0) cols[cnt++] = r - 1;
        cols[cnt++] = r;
        if (x + 1 < n) cols[cnt++] = r + 1;
        if (y + 1 < n) cols[cnt++] = r + n;
        if (z + 1 < n) cols[cnt++] = r + n2;
    }
    return cnt;
}

__global__ void stencil_len_kernel(int points, gidx n, gidx rb, gidx nrows, gidx* lens) {
    const gidx t = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (t > nrows) return;
    if (t == nrows) {
        lens[t] = 0;
        return;
    }
    gidx cols[7];
    lens[t] = stencil_neighbours(points, n, rb + t, cols);
}

template <class T>
__global__ void stencil_fill_kernel(int points, gidx n, gidx rb, gidx nrows, const gidx* rowptr, gidx* col, T* val) {
    const gidx t = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (t >= nrows) return;
    gidx cols[7];
    const gidx r = rb + t;
    const int cnt = stencil_neighbours(points, n, r, cols);
    const gidx b = rowptr[t];
    const double diag = points == 5 ? 4.0 : 6.0;
    for (int k = 0; k < cnt; ++k) {
        col[b + k] = cols[k];
        const double v = cols[k] == r ? diag : -1.0;
        if constexpr (scalar_traits<T>::is_complex) val[b + k] = T{typename scalar_traits<T>::real(v), 0};
        else val[b + k] = T(v);
    }
}

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double hash_u11(unsigned long long seed, unsigned long long idx) {
    const unsigned long long h = splitmix64(seed ^ idx);
    return double(h >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

template <class T>
__global__ void fill_hash_kernel(DAcc a, lidx nrows, lidx ncols, unsigned long long seed) {
    const gidx total = gidx(nrows) * ncols;
    for (gidx t = blockIdx.x * gidx(blockDim.x) + threadIdx.x; t < total; t += gidx(gridDim.x) * blockDim.x) {
        const gidx i = t / ncols;
        const lidx j = lidx(t - i * ncols);
        const gidx c = a.cmap ? a.cmap[j] : gidx(j);
        T* p = reinterpret_cast<T*>(a.base + ((a.row_offset + i) * a.rs + c * a.cs) * gidx(sizeof(T)));
        if constexpr (scalar_traits<T>::is_complex) {
            using R = typename scalar_traits<T>::real;
            *p = T{R(hash_u11(seed, t)), R(hash_u11(seed + 1, t))};
        } else {
            *p = T(hash_u11(seed, t));
        }
    }
}

}  // namespace

std::unique_ptr<Crs> crs_stencil(Datatype dt, int points, gidx n, gidx rb, gidx re) {
    SK_REQUIRE(points == 5 || points == 7, errc::invalid_arg, "stencil points must be 5 or 7");
    SK_REQUIRE(n >= 1, errc::invalid_arg, "grid size must be positive");
    const gidx N = points == 5 ? n * n : n * n * n;
    SK_REQUIRE(rb >= 0 && rb <= re && re <= N, errc::invalid_arg, "row range out of bounds");
    const gidx nrows = re - rb;
    auto a = std::make_unique<Crs>();
    a->dt = dt;
    a->nrows = nrows;
    a->ncols = N;
    a->device = current_device();
    auto& rt = runtime(a->device);
    a->rowptr = DeviceBuffer(std::size_t(nrows + 1) * sizeof(gidx), a->device);
    {
        DeviceBuffer lens(std::size_t(nrows + 1) * sizeof(gidx), a->device);
        stencil_len_kernel<<<int((nrows + 256) / 256), 256, 0, rt.stream>>>(points, n, rb, nrows, lens.as<gidx>());
        CK(cudaGetLastError());
        exclusive_scan_i64(lens.as<gidx>(), a->rowptr.as<gidx>(), nrows + 1, rt);
    }
    CK(cudaMemcpyAsync(&a->nnz, a->rowptr.as<gidx>() + nrows, sizeof(gidx), cudaMemcpyDeviceToHost, rt.stream));
    CK(cudaStreamSynchronize(rt.stream));
    a->col = DeviceBuffer(std::max<std::size_t>(std::size_t(a->nnz) * sizeof(gidx), 8), a->device);
    a->val = DeviceBuffer(std::max<std::size_t>(std::size_t(a->nnz) * value_bytes(dt), 16), a->device);
    visit_dt(dt, [&]<class T>() {
        if (nrows > 0)
            stencil_fill_kernel<T><<<int((nrows + 255) / 256), 256, 0, rt.stream>>>(
                points, n, rb, nrows, a->rowptr.as<gidx>(), a->col.as<gidx>(), a->val.as<T>());
        return 0;
    });
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(rt.stream));
    return a;
}

void densemat_fill_hash(DenseMat& m, unsigned long long seed) {
    Staged s(m, false);
    DeviceGuard g(s.dev.device);
    auto& rt = runtime(s.dev.device);
    DAcc a = dacc(s.dev);
    visit_dt(m.dt, [&]<class T>() {
        const gidx total = gidx(m.nrows) * m.ncols;
        const int grid = int(std::max<gidx>(1, std::min<gidx>((total + 255) / 256, gidx(rt.num_sms) * 16)));
        fill_hash_kernel<T><<<grid, 256, 0, rt.stream>>>(a, m.nrows, m.ncols, seed);
        return 0;
    });
    CK(cudaGetLastError());
    s.write_back();
    finish(rt);
}

}  // namespace skb
