// Fused SELL-C-sigma SpMV driver: validation (spmv.hpp:98-125), staging of
// host-resident vectors, kernel dispatch and the ordered dot reduction.
#include "spmv_kernels.cuh"

namespace skb {

using namespace spmv_detail;

namespace {

template <class T>
T scalar_of(const unsigned char* b) {
    T v;
    std::memcpy(&v, b, sizeof(T));
    return v;
}

// 16-B aligned view: every vector access of the specialised kernel is legal.
// Every row segment a specialised kernel touches with one vector access must be
// aligned to the access width: min(32 B, width * element bytes) (widths are powers of 2).
bool aligned_for_vectors(const DenseMat& m) {
    const std::size_t req = std::min<std::size_t>(32, std::size_t(m.ncols) * m.esize());
    if (req & (req - 1)) return false;
    return (reinterpret_cast<std::uintptr_t>(m.data) % req == 0) && ((std::size_t(m.stride) * m.esize()) % req == 0);
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
        if (hooks.x_self) {
            a.xs = reinterpret_cast<const T*>(hooks.x_self->data);
            a.xs_rs = hooks.x_self->row_stride();
            a.xs_cs = hooks.x_self->col_step();
        }
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
        const LaunchShape ls = launch_spmv<T>(a, spec, rt, st, A.max_chunk_len);
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
