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

// Synthetic topological-insulator Hamiltonian (the KPM benchmark
// of Kreutzer et al. 2015): 4 orbitals per site of an Lx x Ly x Lz periodic lattice,
// row = site * 4 + orbital, site = (z * Ly + y) * Lx + x.
//   on-site  : 2 G1 + V_site G0        (G0 = I4, G1 = tau_z (x) I2: diagonal)
//   hopping  : to the +/- neighbour along axis a in {x, y, z}: (G1 -/+ i G_{a+2}) / 2
//              with G2 = tau_x (x) sigma_x, G3 = tau_x (x) sigma_y, G4 = tau_x (x) sigma_z,
//              so every hopping block has 2 nonzeros per row -> 13 nonzeros per row.
// V_site in [-disorder/2, disorder/2) from the counter hash of the site index.
__device__ __forceinline__ void ti_entries(gidx r, gidx Lx, gidx Ly, gidx Lz, double disorder, gidx* cols, double* re,
                                           double* im, int& cnt) {
    const gidx site = r >> 2;
    const int o = int(r & 3);
    const gidx x = site % Lx, y = (site / Lx) % Ly, z = site / (Lx * Ly);
    const double g1 = (o < 2) ? 1.0 : -1.0;  // tau_z
    cnt = 0;
    auto push = [&](gidx c, double vr, double vi) {
        // insertion sort by column (at most 13 entries)
        int p = cnt++;
        while (p > 0 && cols[p - 1] > c) {
            cols[p] = cols[p - 1];
            re[p] = re[p - 1];
            im[p] = im[p - 1];
            --p;
        }
        cols[p] = c;
        re[p] = vr;
        im[p] = vi;
    };
    {
        const unsigned long long h = splitmix64(0x51ull ^ (unsigned long long)site);
        const double u = double(h >> 11) * 0x1.0p-53 - 0.5;
        push(r, 2.0 * g1 + disorder * u, 0.0);
    }
    // partner orbital of G_{a+2} = tau_x (x) sigma_{x,y,z}: flips tau, sigma per axis
    for (int a = 0; a < 3; ++a) {
        for (int s = -1; s <= 1; s += 2) {
            gidx nx = x, ny = y, nz = z;
            if (a == 0) nx = (x + s + Lx) % Lx;
            if (a == 1) ny = (y + s + Ly) % Ly;
            if (a == 2) nz = (z + s + Lz) % Lz;
            const gidx ns = (nz * Ly + ny) * Lx + nx;
            // G1 / 2 diagonal part
            push(ns * 4 + o, 0.5 * g1, 0.0);
            // -/+ i G_{a+2} / 2: tau_x maps orbital block 0<->1 (o ^ 2); sigma acts on o & 1
            const int to = o ^ 2, so = o & 1;
            double mr = 0.0, mi = 0.0;  // matrix element <o| tau_x (x) sigma_a |o'>
            int op;
            if (a == 0) { op = to ^ 1; mr = 1.0; }                               // sigma_x
            else if (a == 1) { op = to ^ 1; mi = so == 0 ? -1.0 : 1.0; }         // sigma_y: <0|s_y|1> = -i
            else { op = to; mr = so == 0 ? 1.0 : -1.0; }                         // sigma_z
            // value = (-s) * i * m / 2   (hop +1: -i G / 2, hop -1: +i G / 2)
            const double fr = -double(s) * (-mi) * 0.5, fi = -double(s) * mr * 0.5;
            push(ns * 4 + op, fr, fi);
        }
    }
}

__global__ void ti_len_kernel(gidx Lx, gidx Ly, gidx Lz, gidx rb, gidx nrows, gidx* lens) {
    const gidx t = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (t > nrows) return;
    lens[t] = t == nrows ? 0 : 13;
}

template <class T>
__global__ void ti_fill_kernel(gidx Lx, gidx Ly, gidx Lz, double disorder, gidx rb, gidx nrows, const gidx* rowptr,
                               gidx* col, T* val) {
    const gidx t = blockIdx.x * gidx(blockDim.x) + threadIdx.x;
    if (t >= nrows) return;
    gidx cols[13];
    double re[13], im[13];
    int cnt = 0;
    ti_entries(rb + t, Lx, Ly, Lz, disorder, cols, re, im, cnt);
    const gidx b = rowptr[t];
    for (int q = 0; q < cnt; ++q) {
        col[b + q] = cols[q];
        if constexpr (scalar_traits<T>::is_complex) {
            using R = typename scalar_traits<T>::real;
            val[b + q] = T{R(re[q]), R(im[q])};
        } else {
            val[b + q] = T(re[q]);  // real surrogate: same pattern, real parts
        }
    }
}

}  // namespace

// C3 generator (rows [rb, re) of the 4*Lx*Ly*Lz Hamiltonian, global columns)
std::unique_ptr<Crs> crs_ti(Datatype dt, gidx Lx, gidx Ly, gidx Lz, double disorder, gidx rb, gidx re) {
    SK_REQUIRE(Lx >= 3 && Ly >= 3 && Lz >= 3, errc::invalid_arg, "lattice extents must be at least 3 (periodic)");
    const gidx N = 4 * Lx * Ly * Lz;
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
        ti_len_kernel<<<int((nrows + 256) / 256), 256, 0, rt.stream>>>(Lx, Ly, Lz, rb, nrows, lens.as<gidx>());
        CK(cudaGetLastError());
        exclusive_scan_i64(lens.as<gidx>(), a->rowptr.as<gidx>(), nrows + 1, rt);
    }
    a->nnz = 13 * nrows;
    a->col = DeviceBuffer(std::max<std::size_t>(std::size_t(a->nnz) * sizeof(gidx), 8), a->device);
    a->val = DeviceBuffer(std::max<std::size_t>(std::size_t(a->nnz) * value_bytes(dt), 16), a->device);
    visit_dt(dt, [&]<class T>() {
        if (nrows > 0)
            ti_fill_kernel<T><<<int((nrows + 255) / 256), 256, 0, rt.stream>>>(Lx, Ly, Lz, disorder, rb, nrows,
                                                                            a->rowptr.as<gidx>(), a->col.as<gidx>(),
                                                                            a->val.as<T>());
        return 0;
    });
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(rt.stream));
    return a;
}

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
