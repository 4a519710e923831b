// Dense block vectors on the device (reference: /root/reference/proj/src/densemat.hpp)
// and the BLAS-1 kernels (densemat.hpp:243-292).
#include <algorithm>

#include "objects.cuh"
#include "ops.cuh"

namespace skb {

namespace {

__device__ __forceinline__ char* elem_ptr(const DAcc& a, gidx i, lidx j, std::size_t es) {
    const gidx c = a.cmap ? a.cmap[j] : gidx(j);
    return a.base + ((a.row_offset + i) * a.rs + c * a.cs) * gidx(es);
}

template <class T>
__global__ void copy_kernel(DAcc dst, DAcc src, lidx nrows, lidx ncols) {
    const gidx total = gidx(nrows) * ncols;
    for (gidx t = blockIdx.x * gidx(blockDim.x) + threadIdx.x; t < total; t += gidx(gridDim.x) * blockDim.x) {
        const gidx i = t / ncols;
        const lidx j = lidx(t - i * ncols);
        *reinterpret_cast<T*>(elem_ptr(dst, i, j, sizeof(T))) =
            *reinterpret_cast<const T*>(elem_ptr(src, i, j, sizeof(T)));
    }
}

template <class T>
__global__ void axpby_kernel(DAcc y, DAcc x, lidx nrows, lidx ncols, const T* alphas, const T* betas,
                             int per_column) {
    using O = Ops<T>;
    const gidx total = gidx(nrows) * ncols;
    for (gidx t = blockIdx.x * gidx(blockDim.x) + threadIdx.x; t < total; t += gidx(gridDim.x) * blockDim.x) {
        const gidx i = t / ncols;
        const lidx j = lidx(t - i * ncols);
        const T a = alphas[per_column ? j : 0];
        const T b = betas[per_column ? j : 0];
        T* yp = reinterpret_cast<T*>(elem_ptr(y, i, j, sizeof(T)));
        const T xv = *reinterpret_cast<const T*>(elem_ptr(x, i, j, sizeof(T)));
        *yp = O::add(O::mul(a, xv), O::mul(b, *yp));  // densemat.hpp:247
    }
}

template <class T>
__global__ void scal_kernel(DAcc x, lidx nrows, lidx ncols, const T* f, int per_column) {
    using O = Ops<T>;
    const gidx total = gidx(nrows) * ncols;
    for (gidx t = blockIdx.x * gidx(blockDim.x) + threadIdx.x; t < total; t += gidx(gridDim.x) * blockDim.x) {
        const gidx i = t / ncols;
        const lidx j = lidx(t - i * ncols);
        T* p = reinterpret_cast<T*>(elem_ptr(x, i, j, sizeof(T)));
        *p = O::mul(*p, f[per_column ? j : 0]);
    }
}

constexpr int kDotThreads = 256;

// Per-block partial column dots (fixed grid => deterministic), then an
// ordered final pass.  out[j] = sum_i conj(a[i,j]) b[i,j] (densemat.hpp:276-292).
template <class T>
__global__ void dot_partial_kernel(DAcc a, DAcc b, lidx nrows, lidx ncols, T* partial) {
    using O = Ops<T>;
    __shared__ T red[kDotThreads];
    for (lidx j = 0; j < ncols; ++j) {
        T s = O::zero();
        for (gidx i = blockIdx.x * gidx(blockDim.x) + threadIdx.x; i < nrows; i += gidx(gridDim.x) * blockDim.x) {
            const T av = *reinterpret_cast<const T*>(elem_ptr(a, i, j, sizeof(T)));
            const T bv = *reinterpret_cast<const T*>(elem_ptr(b, i, j, sizeof(T)));
            s = O::add(s, O::mul(O::conj(av), bv));
        }
        red[threadIdx.x] = s;
        __syncthreads();
        for (int w = kDotThreads / 2; w > 0; w >>= 1) {
            if (int(threadIdx.x) < w) red[threadIdx.x] = O::add(red[threadIdx.x], red[threadIdx.x + w]);
            __syncthreads();
        }
        if (threadIdx.x == 0) partial[gidx(blockIdx.x) * ncols + j] = red[0];
        __syncthreads();
    }
}

template <class T>
__global__ void ordered_sum_kernel(const T* partial, int nparts, int n, T* out) {
    using O = Ops<T>;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    T s = O::zero();
    for (int p = 0; p < nparts; ++p) s = O::add(s, partial[gidx(p) * n + j]);
    out[j] = s;
}

int grid_for(gidx total, int threads, const DeviceRuntime& rt) {
    gidx g = (total + threads - 1) / threads;
    const gidx cap = gidx(rt.num_sms) * 16;
    return int(std::max<gidx>(1, std::min(g, cap)));
}

void upload_cmap(DenseMat& m) {
    if (!m.scattered() || m.col_map_dev) return;
    auto& rt = runtime(m.device);
    m.col_map_dev = std::make_shared<DeviceBuffer>(m.col_map.size() * sizeof(gidx), m.device);
    CK(cudaMemcpyAsync(m.col_map_dev->get(), m.col_map.data(), m.col_map.size() * sizeof(gidx),
                       cudaMemcpyHostToDevice, rt.stream));
}

// Host-side element address (host-resident matrices).
inline char* host_elem(const DenseMat& m, gidx i, lidx j) {
    const gidx c = m.map_col(j);
    const gidx r = m.row_offset + i;
    const gidx off = (m.order == Order::row_major) ? r * m.stride + c : c * m.stride + r;
    return m.data + off * gidx(m.esize());
}

bool contiguous_row_major(const DenseMat& m) {
    return !m.scattered() && m.order == Order::row_major && (m.stride == m.ncols || m.nrows == 1);
}

}  // namespace

DAcc dacc(DenseMat& m) {
    SK_REQUIRE(m.mem == MemKind::device, errc::state, "internal: device accessor on host matrix");
    upload_cmap(m);
    DAcc a;
    a.base = m.data;
    a.row_offset = m.row_offset;
    a.cmap = m.scattered() ? m.col_map_dev->as<gidx>() : nullptr;
    if (m.order == Order::row_major) {
        a.rs = m.stride;
        a.cs = 1;
    } else {
        a.rs = 1;
        a.cs = m.stride;
    }
    return a;
}

// densemat.hpp:29-46
DenseMat densemat_create(Datatype dt, lidx nrows, lidx ncols, Order order) {
    SK_REQUIRE(nrows > 0 && ncols > 0, errc::invalid_arg, "matrix dimensions must be positive");
    DenseMat m;
    m.dt = dt;
    m.nrows = nrows;
    m.ncols = ncols;
    m.order = order;
    m.kind = ViewKind::owned;
    m.mem = MemKind::device;
    m.device = current_device();
    const lidx pad = row_padding();
    const gidx nrows_padded = (gidx(nrows) + pad - 1) / pad * pad;
    m.stride = order == Order::row_major ? ncols : lidx(nrows_padded);
    const std::size_t bytes = std::size_t(nrows_padded) * std::size_t(ncols) * value_bytes(dt);
    m.owner = std::make_shared<DeviceBuffer>(bytes, m.device);
    m.data = m.owner->as<char>();
    auto& rt = runtime(m.device);
    CK(cudaMemsetAsync(m.data, 0, bytes, rt.stream));  // zero-initialised like the reference
    finish(rt);
    return m;
}

// densemat.hpp:50-67
DenseMat densemat_view_plain(Datatype dt, void* buffer, std::size_t nelems, lidx nrows, lidx ncols,
                             lidx stride, Order order) {
    SK_REQUIRE(buffer != nullptr, errc::invalid_arg, "null buffer");
    SK_REQUIRE(nrows > 0 && ncols > 0, errc::invalid_arg, "matrix dimensions must be positive");
    const lidx leading = order == Order::row_major ? ncols : nrows;
    const lidx slow = order == Order::row_major ? nrows : ncols;
    SK_REQUIRE(stride >= leading, errc::invalid_arg, "stride smaller than leading extent");
    SK_REQUIRE(nelems >= std::size_t(stride) * std::size_t(slow), errc::invalid_arg,
               "buffer too small for the requested shape and stride");
    DenseMat m;
    m.dt = dt;
    m.nrows = nrows;
    m.ncols = ncols;
    m.order = order;
    m.stride = stride;
    m.kind = ViewKind::compact_view;
    int dev = 0;
    m.mem = pointer_kind(buffer, &dev);
    m.device = m.mem == MemKind::device ? dev : current_device();
    m.data = static_cast<char*>(buffer);
    return m;
}

// densemat.hpp:72-106
DenseMat densemat_view(const DenseMat& p, lidx row_begin, lidx row_end, const lidx* cols, lidx ncols) {
    SK_REQUIRE(row_begin >= 0 && row_begin < row_end && row_end <= p.nrows, errc::invalid_arg,
               "row range out of bounds");
    SK_REQUIRE(ncols > 0, errc::invalid_arg, "empty column selection");
    for (lidx k = 0; k < ncols; ++k) {
        SK_REQUIRE(cols[k] >= 0 && cols[k] < p.ncols, errc::invalid_arg, "column selection out of bounds");
        if (k > 0) SK_REQUIRE(cols[k] > cols[k - 1], errc::invalid_arg, "column selection must be strictly increasing");
    }
    std::vector<gidx> mapped;
    mapped.reserve(std::size_t(ncols));
    for (lidx k = 0; k < ncols; ++k) mapped.push_back(p.map_col(cols[k]));
    const bool contiguous = mapped.back() - mapped.front() + 1 == gidx(mapped.size());

    DenseMat v;
    v.dt = p.dt;
    v.nrows = row_end - row_begin;
    v.ncols = ncols;
    v.order = p.order;
    v.stride = p.stride;
    v.owner = p.owner;
    v.mem = p.mem;
    v.device = p.device;
    const gidx es = gidx(value_bytes(p.dt));
    if (contiguous) {
        v.kind = ViewKind::compact_view;
        const gidx r = p.row_offset + row_begin;
        const gidx c = mapped.front();
        const gidx off = p.order == Order::row_major ? r * p.stride + c : c * p.stride + r;
        v.data = p.data + off * es;
    } else {
        v.kind = ViewKind::scattered_view;
        v.data = p.data;
        v.row_offset = p.row_offset + row_begin;
        v.col_map = std::move(mapped);
    }
    return v;
}

Staged::Staged(DenseMat& m, bool load, int slot) : orig(&m) {
    if (m.mem == MemKind::device) {
        dev = m;
        return;
    }
    staged = true;
    if (slot >= 0) {
        auto& rt = runtime(current_device());
        const std::size_t n = std::size_t(m.nrows) * m.ncols;
        void* buf = rt.stage_bytes(slot, std::max<std::size_t>(n * m.esize(), 256));
        dev = m.order == Order::row_major
                  ? densemat_view_plain(m.dt, buf, n, m.nrows, m.ncols, m.ncols, Order::row_major)
                  : densemat_view_plain(m.dt, buf, n, m.nrows, m.ncols, m.nrows, Order::col_major);
    } else {
        dev = densemat_create(m.dt, m.nrows, m.ncols, m.order);
    }
    if (load) densemat_copy(dev, m);
}

void Staged::write_back() {
    if (staged) densemat_copy(*orig, dev);
    else *orig = dev;  // keeps lazily uploaded col maps
}

// General logical copy dst(i,j) = src(i,j).
void densemat_copy(DenseMat& dst, const DenseMat& src_in) {
    SK_REQUIRE(dst.same_shape(src_in), errc::shape_mismatch, "shape mismatch");
    SK_REQUIRE(dst.dt == src_in.dt, errc::invalid_arg, "datatype mismatch");
    DenseMat src = src_in;
    const std::size_t es = dst.esize();
    if (dst.mem == MemKind::host && src.mem == MemKind::host) {
        for (lidx i = 0; i < dst.nrows; ++i)
            for (lidx j = 0; j < dst.ncols; ++j) std::memcpy(host_elem(dst, i, j), host_elem(src, i, j), es);
        return;
    }
    const int dev = dst.mem == MemKind::device ? dst.device : src.device;
    DeviceGuard g(dev);
    auto& rt = runtime(dev);
    if (dst.mem == MemKind::device && src.mem == MemKind::device) {
        if (dst.device != src.device) {
            // cross-device: one peer copy (NVLink / PCIe P2P, no host bounce) of a compact
            // row-major image of src, then the layout copy on the destination device
            const std::size_t n = std::size_t(src.nrows) * src.ncols;
            auto& rs = runtime(src.device);
            DeviceBuffer src_tmp;
            const void* image = src.data;
            if (!contiguous_row_major(src)) {
                DeviceGuard gs(src.device);
                src_tmp = DeviceBuffer(std::max<std::size_t>(n * es, 16), src.device);
                DenseMat t = densemat_view_plain(src.dt, src_tmp.get(), n, src.nrows, src.ncols, src.ncols,
                                                 Order::row_major);
                densemat_copy(t, src);
                image = src_tmp.get();
            }
            cudaEvent_t ready;
            {
                DeviceGuard gs(src.device);
                CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
                CK(cudaEventRecord(ready, rs.stream));
            }
            CK(cudaStreamWaitEvent(rt.stream, ready, 0));
            if (contiguous_row_major(dst)) {
                CK(cudaMemcpyPeerAsync(dst.data, dst.device, image, src.device, n * es, rt.stream));
            } else {
                DeviceBuffer dst_tmp(std::max<std::size_t>(n * es, 16), dst.device);
                CK(cudaMemcpyPeerAsync(dst_tmp.get(), dst.device, image, src.device, n * es, rt.stream));
                DenseMat t = densemat_view_plain(dst.dt, dst_tmp.get(), n, dst.nrows, dst.ncols, dst.ncols,
                                                 Order::row_major);
                DAcc d = dacc(dst), s2 = dacc(t);
                visit_dt(dst.dt, [&]<class T>() {
                    copy_kernel<T><<<grid_for(gidx(dst.nrows) * dst.ncols, 256, rt), 256, 0, rt.stream>>>(
                        d, s2, dst.nrows, dst.ncols);
                    return 0;
                });
                CK(cudaGetLastError());
                CK(cudaStreamSynchronize(rt.stream));  // before dst_tmp is freed
            }
            CK(cudaStreamSynchronize(rt.stream));      // before src_tmp / the event go
            CK(cudaEventDestroy(ready));
            return;
        }
        DAcc d = dacc(dst), s = dacc(src);
        visit_dt(dst.dt, [&]<class T>() {
            copy_kernel<T><<<grid_for(gidx(dst.nrows) * dst.ncols, 256, rt), 256, 0, rt.stream>>>(
                d, s, dst.nrows, dst.ncols);
            return 0;
        });
        CK(cudaGetLastError());
        return;
    }
    if (dst.mem == MemKind::device) {  // host -> device
        if (contiguous_row_major(src)) {
            densemat_copy_in(dst, src.data, std::size_t(src.nrows) * src.ncols);
            return;
        }
        std::vector<unsigned char> host(std::size_t(src.nrows) * src.ncols * es);
        for (lidx i = 0; i < src.nrows; ++i)
            for (lidx j = 0; j < src.ncols; ++j)
                std::memcpy(&host[(std::size_t(i) * src.ncols + j) * es], host_elem(src, i, j), es);
        densemat_copy_in(dst, host.data(), std::size_t(src.nrows) * src.ncols);
        return;
    }
    // device -> host
    if (contiguous_row_major(dst)) {
        densemat_copy_out(src, dst.data, std::size_t(dst.nrows) * dst.ncols);
        return;
    }
    std::vector<unsigned char> host(std::size_t(src.nrows) * src.ncols * es);
    densemat_copy_out(src, host.data(), std::size_t(src.nrows) * src.ncols);
    for (lidx i = 0; i < dst.nrows; ++i)
        for (lidx j = 0; j < dst.ncols; ++j)
            std::memcpy(host_elem(dst, i, j), &host[(std::size_t(i) * dst.ncols + j) * es], es);
}

// densemat.hpp:149-154: logical contents from a contiguous row-major host buffer.
void densemat_copy_in(DenseMat& m, const void* buf, std::size_t nelems) {
    SK_REQUIRE(nelems == std::size_t(m.nrows) * std::size_t(m.ncols), errc::shape_mismatch,
               "buffer size does not match matrix shape");
    const std::size_t es = m.esize();
    if (m.mem == MemKind::host) {
        const auto* src = static_cast<const unsigned char*>(buf);
        for (lidx i = 0; i < m.nrows; ++i)
            for (lidx j = 0; j < m.ncols; ++j)
                std::memcpy(host_elem(m, i, j), src + (std::size_t(i) * m.ncols + j) * es, es);
        return;
    }
    DeviceGuard g(m.device);
    auto& rt = runtime(m.device);
    if (!m.scattered() && m.order == Order::row_major) {
        CK(cudaMemcpy2DAsync(m.data, std::size_t(m.stride) * es, buf, std::size_t(m.ncols) * es,
                             std::size_t(m.ncols) * es, std::size_t(m.nrows), cudaMemcpyHostToDevice,
                             rt.stream));
        finish(rt);
        return;
    }
    // col-major or scattered: upload row-major, then permute on the device
    DeviceBuffer tmp(nelems * es, m.device);
    CK(cudaMemcpyAsync(tmp.get(), buf, nelems * es, cudaMemcpyHostToDevice, rt.stream));
    DenseMat t = densemat_view_plain(m.dt, tmp.get(), nelems, m.nrows, m.ncols, m.ncols, Order::row_major);
    densemat_copy(m, t);
    CK(cudaStreamSynchronize(rt.stream));  // tmp dies here
}

// densemat.hpp:156-161
void densemat_copy_out(const DenseMat& m_in, void* buf, std::size_t nelems) {
    DenseMat m = m_in;
    SK_REQUIRE(nelems == std::size_t(m.nrows) * std::size_t(m.ncols), errc::shape_mismatch,
               "buffer size does not match matrix shape");
    const std::size_t es = m.esize();
    if (m.mem == MemKind::host) {
        auto* dst = static_cast<unsigned char*>(buf);
        for (lidx i = 0; i < m.nrows; ++i)
            for (lidx j = 0; j < m.ncols; ++j)
                std::memcpy(dst + (std::size_t(i) * m.ncols + j) * es, host_elem(m, i, j), es);
        return;
    }
    DeviceGuard g(m.device);
    auto& rt = runtime(m.device);
    if (!m.scattered() && m.order == Order::row_major) {
        CK(cudaMemcpy2DAsync(buf, std::size_t(m.ncols) * es, m.data, std::size_t(m.stride) * es,
                             std::size_t(m.ncols) * es, std::size_t(m.nrows), cudaMemcpyDeviceToHost,
                             rt.stream));
        CK(cudaStreamSynchronize(rt.stream));
        return;
    }
    DeviceBuffer tmp(nelems * es, m.device);
    DenseMat t = densemat_view_plain(m.dt, tmp.get(), nelems, m.nrows, m.ncols, m.ncols, Order::row_major);
    densemat_copy(t, m);
    CK(cudaMemcpyAsync(buf, tmp.get(), nelems * es, cudaMemcpyDeviceToHost, rt.stream));
    CK(cudaStreamSynchronize(rt.stream));
}

// densemat.hpp:117-122
DenseMat densemat_compact_clone(const DenseMat& m) {
    DeviceGuard g(m.mem == MemKind::device ? m.device : current_device());
    DenseMat out = densemat_create(m.dt, m.nrows, m.ncols, m.order);
    densemat_copy(out, m);
    finish(runtime(out.device));
    return out;
}

// densemat.hpp:213-224
DenseMat densemat_convert_order(DenseMat& v, Order new_order, bool in_place) {
    SK_REQUIRE(!v.scattered(), errc::invalid_arg, "convert_order requires a compact matrix");
    DeviceGuard g(v.mem == MemKind::device ? v.device : current_device());
    DenseMat out = densemat_create(v.dt, v.nrows, v.ncols, new_order);
    densemat_copy(out, v);
    finish(runtime(out.device));
    if (in_place) {
        SK_REQUIRE(v.kind == ViewKind::owned, errc::invalid_arg, "in-place conversion requires an owned matrix");
        v = out;
    }
    return out;
}

// ------------------------------------------------------------------ BLAS-1 --

void blas_axpby(DenseMat& y, const DenseMat& x_in, const void* alpha, const void* beta, bool per_column) {
    SK_REQUIRE(y.same_shape(x_in), errc::shape_mismatch, per_column ? "vaxpby shape mismatch" : "axpby shape mismatch");
    DenseMat x = x_in;
    Staged ys(y, true);
    Staged xs(x, true);
    const int dev = ys.dev.device;
    DeviceGuard g(dev);
    auto& rt = runtime(dev);
    const std::size_t es = y.esize();
    const std::size_t ns = per_column ? std::size_t(y.ncols) : 1;
    auto* sc = static_cast<char*>(rt.scratch_bytes(2 * ns * es));
    std::vector<unsigned char> hs(2 * ns * es);
    std::memcpy(hs.data(), alpha, ns * es);
    std::memcpy(hs.data() + ns * es, beta, ns * es);
    CK(cudaMemcpyAsync(sc, hs.data(), hs.size(), cudaMemcpyHostToDevice, rt.stream));
    DAcc ya = dacc(ys.dev), xa = dacc(xs.dev);
    visit_dt(y.dt, [&]<class T>() {
        axpby_kernel<T><<<grid_for(gidx(y.nrows) * y.ncols, 256, rt), 256, 0, rt.stream>>>(
            ya, xa, y.nrows, y.ncols, reinterpret_cast<const T*>(sc), reinterpret_cast<const T*>(sc + ns * es),
            per_column ? 1 : 0);
        return 0;
    });
    CK(cudaGetLastError());
    ys.write_back();
    CK(cudaStreamSynchronize(rt.stream));  // host scalars / staging buffers
}

void blas_scal(DenseMat& x, const void* factor, bool per_column) {
    Staged xs(x, true);
    const int dev = xs.dev.device;
    DeviceGuard g(dev);
    auto& rt = runtime(dev);
    const std::size_t es = x.esize();
    const std::size_t ns = per_column ? std::size_t(x.ncols) : 1;
    auto* sc = static_cast<char*>(rt.scratch_bytes(ns * es));
    CK(cudaMemcpyAsync(sc, factor, ns * es, cudaMemcpyHostToDevice, rt.stream));
    DAcc xa = dacc(xs.dev);
    visit_dt(x.dt, [&]<class T>() {
        scal_kernel<T><<<grid_for(gidx(x.nrows) * x.ncols, 256, rt), 256, 0, rt.stream>>>(
            xa, x.nrows, x.ncols, reinterpret_cast<const T*>(sc), per_column ? 1 : 0);
        return 0;
    });
    CK(cudaGetLastError());
    xs.write_back();
    CK(cudaStreamSynchronize(rt.stream));
}

void blas_dot(const DenseMat& a_in, const DenseMat& b_in, void* out) {
    SK_REQUIRE(a_in.same_shape(b_in), errc::shape_mismatch, "dot shape mismatch");
    DenseMat a = a_in, b = b_in;
    Staged as(a, true), bs(b, true);
    const int dev = as.dev.device;
    DeviceGuard g(dev);
    auto& rt = runtime(dev);
    const std::size_t es = a.esize();
    const int nblocks = std::max(1, std::min(rt.num_sms * 2, int((a.nrows + kDotThreads - 1) / kDotThreads)));
    const std::size_t w = std::size_t(a.ncols);
    auto* sc = static_cast<char*>(rt.scratch_bytes((std::size_t(nblocks) + 1) * w * es));
    DAcc aa = dacc(as.dev), ba = dacc(bs.dev);
    visit_dt(a.dt, [&]<class T>() {
        T* partial = reinterpret_cast<T*>(sc);
        T* res = partial + std::size_t(nblocks) * w;
        dot_partial_kernel<T><<<nblocks, kDotThreads, 0, rt.stream>>>(aa, ba, a.nrows, a.ncols, partial);
        ordered_sum_kernel<T><<<int((w + 127) / 128), 128, 0, rt.stream>>>(partial, nblocks, int(w), res);
        CK(cudaMemcpyAsync(out, res, w * es, cudaMemcpyDeviceToHost, rt.stream));
        return 0;
    });
    CK(cudaStreamSynchronize(rt.stream));
}

}  // namespace skb
