// The extern "C" surface (include/sellkit.h, include/sellkit_ext.h).
// Mirrors /root/reference/proj/src/capi.cpp: exceptions are mapped to error
// codes at this boundary (capi.cpp:50-62), NULL scalars select the documented
// defaults (capi.cpp:64-70, 124-140), datatype mismatches between handles are
// SELLKIT_ERR_INVALID_ARG (capi.cpp:142-147).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <new>
#include <numeric>
#include <string>
#include <thread>

#include "handles.cuh"
#include "ops.cuh"
#include "spmv.cuh"
#include "tsm.cuh"

namespace skb {
std::unique_ptr<Crs> crs_stencil(Datatype dt, int points, gidx n, gidx rb, gidx re);
std::unique_ptr<Crs> crs_ti(Datatype dt, gidx Lx, gidx Ly, gidx Lz, double disorder, gidx rb, gidx re);
void densemat_fill_hash(DenseMat& m, unsigned long long seed);
void crs_validate_impl(const Crs& a, bool check_sorted);
std::unique_ptr<Crs> crs_read_mm(const char* path, Datatype dt);
std::unique_ptr<Crs> crs_read_bin(const char* path);
void crs_write_bin(const char* path, const Crs& a, bool wide_cols);
}  // namespace skb

namespace sk = skb;
using sk::dt_from;
using sk::guarded;
using sk::order_from;
using sk::require;
using sk::same_dt;

namespace {

// RowSource -> host CRS (capi.cpp:149-183 / sellcs.hpp:248-265): two passes
// over the callback (lengths, entries); lengths checked against max_rowlen.
std::unique_ptr<sk::Crs> crs_from_rowfunc(sk::Datatype dt, sk::gidx nrows, sk::gidx ncols, sk::lidx max_rowlen,
                                          sellkit_row_fn fn, void* arg, bool check_sorted) {
    require(fn != nullptr, "row callback must not be null");
    require(nrows >= 0 && ncols >= 0, "negative dimension");
    require(max_rowlen >= 0, "negative max_rowlen");
    const std::size_t es = sk::value_bytes(dt);
    std::vector<sk::gidx> rowptr(std::size_t(nrows) + 1, 0), cbuf(std::size_t(std::max(max_rowlen, 1)));
    std::vector<unsigned char> vbuf(std::size_t(std::max(max_rowlen, 1)) * es);
    std::vector<sk::gidx> col;
    std::vector<unsigned char> val;
    for (sk::gidx r = 0; r < nrows; ++r) {
        sk::lidx len = 0;
        if (fn(r, &len, cbuf.data(), vbuf.data(), arg) != 0) sk::fail(sk::errc::invalid_arg, "row callback reported failure");
        SK_REQUIRE(len >= 0 && len <= max_rowlen, sk::errc::invalid_arg, "row longer than max_rowlen");
        rowptr[r + 1] = rowptr[r] + len;
        col.insert(col.end(), cbuf.begin(), cbuf.begin() + len);
        val.insert(val.end(), vbuf.begin(), vbuf.begin() + std::size_t(len) * es);
    }
    if (!check_sorted) {
        // build(RowSource) checks only column ranges (sellcs.hpp:213-215)
        for (sk::gidx c : col) SK_REQUIRE(c >= 0 && c < ncols, sk::errc::invalid_arg, "column index out of range");
    }
    auto a = std::make_unique<sk::Crs>();
    a->dt = dt;
    a->nrows = nrows;
    a->ncols = ncols;
    a->nnz = rowptr.back();
    a->device = sk::current_device();
    auto& rt = sk::runtime(a->device);
    a->rowptr = sk::DeviceBuffer(rowptr.size() * sizeof(sk::gidx), a->device);
    a->col = sk::DeviceBuffer(std::max<std::size_t>(col.size() * sizeof(sk::gidx), 8), a->device);
    a->val = sk::DeviceBuffer(std::max<std::size_t>(val.size(), 16), a->device);
    CK(cudaMemcpyAsync(a->rowptr.get(), rowptr.data(), rowptr.size() * sizeof(sk::gidx), cudaMemcpyHostToDevice, rt.stream));
    if (!col.empty()) {
        CK(cudaMemcpyAsync(a->col.get(), col.data(), col.size() * sizeof(sk::gidx), cudaMemcpyHostToDevice, rt.stream));
        CK(cudaMemcpyAsync(a->val.get(), val.data(), val.size(), cudaMemcpyHostToDevice, rt.stream));
    }
    CK(cudaStreamSynchronize(rt.stream));
    if (check_sorted) sk::crs_validate_impl(*a, true);
    return a;
}

std::atomic<int>& worker_slot() {
    static std::atomic<int> n{[] {
        if (const char* env = std::getenv("SELLKIT_NUM_WORKERS")) {
            int v = std::atoi(env);
            if (v >= 1) return v;
        }
        return int(std::max(1u, std::thread::hardware_concurrency()));
    }()};
    return n;
}

std::atomic<double (*)(void*)> g_timer_fn{nullptr};
std::atomic<void*> g_timer_arg{nullptr};

std::string sci(double v) {
    char buf[32];
    std::snprintf(buf, sizeof(buf), "%.2e", v);
    return buf;
}

char* dup_string(const std::string& s) {
    char* out = new char[s.size() + 1];
    std::memcpy(out, s.c_str(), s.size() + 1);
    return out;
}

}  // namespace

extern "C" {

/* ------------------------------------------------------------------ basics */

const char* sellkit_error_name(sellkit_error err) { return sk::errc_name(static_cast<sk::errc>(static_cast<int>(err))); }

sellkit_error sellkit_narrow_index(sellkit_gidx g, sellkit_lidx* out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        *out = sk::narrow_index(g);
    });
}

sellkit_error sellkit_buildconfig_chunk_heights(const int** out, size_t* n) {
    return guarded([&] {
        require(out && n, "null output");
        *out = sk::config_chunk_heights(n);
    });
}

sellkit_error sellkit_buildconfig_block_widths(const int** out, size_t* n) {
    return guarded([&] {
        require(out && n, "null output");
        *out = sk::config_block_widths(n);
    });
}

sellkit_error sellkit_set_num_workers(int n) {
    return guarded([&] {
        SK_REQUIRE(n >= 1, sk::errc::invalid_arg, "worker count must be positive");
        worker_slot().store(n);
    });
}

int sellkit_num_workers(void) { return worker_slot().load(); }

double sellkit_now_seconds(void) {
    if (auto* fn = g_timer_fn.load(std::memory_order_acquire)) return fn(g_timer_arg.load());
    using clock = std::chrono::steady_clock;
    return std::chrono::duration<double>(clock::now().time_since_epoch()).count();
}

void sellkit_set_timer_override(double (*now_fn)(void*), void* arg) {
    g_timer_arg.store(arg);
    g_timer_fn.store(now_fn, std::memory_order_release);
}

/* --------------------------------------------------------------------- crs */

sellkit_error sellkit_crs_create(sellkit_datatype dt, sellkit_gidx nrows, sellkit_gidx ncols,
                                 const sellkit_gidx* rowptr, const sellkit_gidx* col, const void* val,
                                 sellkit_crs** out) {
    return guarded([&] {
        require(out && rowptr, "null argument");
        require(nrows >= 0 && ncols >= 0, "negative dimension");
        const sk::gidx nnz = rowptr[nrows];
        require(nnz >= 0, "negative nonzero count");
        require(nnz == 0 || (col && val), "null payload");
        *out = new sellkit_crs{sk::crs_from_host(dt_from(dt), nrows, ncols, rowptr, col, val)};
    });
}

sellkit_error sellkit_crs_from_rowfunc(sellkit_datatype dt, sellkit_gidx nrows, sellkit_gidx ncols,
                                       sellkit_lidx max_rowlen, sellkit_row_fn fn, void* arg, sellkit_crs** out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        *out = new sellkit_crs{crs_from_rowfunc(dt_from(dt), nrows, ncols, max_rowlen, fn, arg, true)};
    });
}

sellkit_error sellkit_crs_read_mm(const char* path, sellkit_datatype dt, sellkit_crs** out) {
    return guarded([&] {
        require(path && out, "null argument");
        *out = new sellkit_crs{sk::crs_read_mm(path, dt_from(dt))};
    });
}

sellkit_error sellkit_crs_read_bin(const char* path, sellkit_crs** out) {
    return guarded([&] {
        require(path && out, "null argument");
        *out = new sellkit_crs{sk::crs_read_bin(path)};
    });
}

sellkit_error sellkit_crs_write_bin(const char* path, const sellkit_crs* crs, int wide_cols) {
    return guarded([&] {
        require(path && crs, "null argument");
        sk::crs_write_bin(path, *crs->p, wide_cols != 0);
    });
}

sellkit_error sellkit_crs_dims(const sellkit_crs* crs, sellkit_gidx* nrows, sellkit_gidx* ncols, sellkit_gidx* nnz) {
    return guarded([&] {
        require(crs != nullptr, "null handle");
        if (nrows) *nrows = crs->p->nrows;
        if (ncols) *ncols = crs->p->ncols;
        if (nnz) *nnz = crs->p->nnz;
    });
}

sellkit_datatype sellkit_crs_datatype(const sellkit_crs* crs) {
    return static_cast<sellkit_datatype>(static_cast<int>(crs->p->dt));
}

void sellkit_crs_destroy(sellkit_crs* crs) { delete crs; }

/* -------------------------------------------------------------------- sell */

sellkit_error sellkit_mat_build(const sellkit_crs* crs, int chunk_height, int sigma, sellkit_mat** out) {
    return guarded([&] {
        require(crs && out, "null argument");
        *out = new sellkit_mat{sk::sell_build(*crs->p, chunk_height, sigma, sk::BuildOptions{})};
    });
}

sellkit_error sellkit_mat_build_rowfunc(sellkit_datatype dt, sellkit_gidx nrows, sellkit_gidx ncols,
                                        sellkit_lidx max_rowlen, sellkit_row_fn fn, void* arg, int chunk_height,
                                        int sigma, sellkit_mat** out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        auto crs = crs_from_rowfunc(dt_from(dt), nrows, ncols, max_rowlen, fn, arg, false);
        *out = new sellkit_mat{sk::sell_build(*crs, chunk_height, sigma, sk::BuildOptions{})};
    });
}

sellkit_error sellkit_mat_stats(const sellkit_mat* m, double* beta, uint64_t* bytes_total) {
    return guarded([&] {
        require(m != nullptr, "null handle");
        if (beta) *beta = m->p->beta;
        if (bytes_total) *bytes_total = sk::sell_bytes_total(*m->p);
    });
}

sellkit_error sellkit_mat_update_values(sellkit_mat* m, const sellkit_crs* crs) {
    return guarded([&] {
        require(m && crs, "null argument");
        same_dt(m->p->dt, crs->p->dt, "matrix and CRS data");
        sk::sell_update_values(*m->p, *crs->p);
    });
}

sellkit_error sellkit_mat_to_crs(const sellkit_mat* m, sellkit_crs** out) {
    return guarded([&] {
        require(m && out, "null argument");
        *out = new sellkit_crs{sk::sell_to_crs(*m->p)};
    });
}

sellkit_error sellkit_mat_dims(const sellkit_mat* m, sellkit_lidx* nrows, sellkit_lidx* ncols, sellkit_gidx* nnz) {
    return guarded([&] {
        require(m != nullptr, "null handle");
        if (nrows) *nrows = m->p->nrows;
        if (ncols) *ncols = m->p->ncols;
        if (nnz) *nnz = m->p->nnz;
    });
}

void sellkit_mat_destroy(sellkit_mat* m) { delete m; }

/* ---------------------------------------------------------------- densemat */

sellkit_error sellkit_densemat_create(sellkit_datatype dt, sellkit_lidx nrows, sellkit_lidx ncols, sellkit_order order,
                                      sellkit_densemat** out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        *out = new sellkit_densemat{sk::densemat_create(dt_from(dt), nrows, ncols, order_from(order))};
    });
}

sellkit_error sellkit_densemat_view_plain(sellkit_datatype dt, void* buffer, size_t nelems, sellkit_lidx nrows,
                                          sellkit_lidx ncols, sellkit_lidx stride, sellkit_order order,
                                          sellkit_densemat** out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        *out = new sellkit_densemat{
            sk::densemat_view_plain(dt_from(dt), buffer, nelems, nrows, ncols, stride, order_from(order))};
    });
}

sellkit_error sellkit_densemat_view(const sellkit_densemat* parent, sellkit_lidx row_begin, sellkit_lidx row_end,
                                    const sellkit_lidx* cols, sellkit_lidx ncols, sellkit_densemat** out) {
    return guarded([&] {
        require(parent && cols && out, "null argument");
        *out = new sellkit_densemat{sk::densemat_view(parent->m, row_begin, row_end, cols, ncols)};
    });
}

sellkit_error sellkit_densemat_compact_clone(const sellkit_densemat* m, sellkit_densemat** out) {
    return guarded([&] {
        require(m && out, "null argument");
        *out = new sellkit_densemat{sk::densemat_compact_clone(m->m)};
    });
}

sellkit_error sellkit_densemat_convert_order(sellkit_densemat* m, sellkit_order new_order, int in_place,
                                             sellkit_densemat** out) {
    return guarded([&] {
        require(m != nullptr, "null handle");
        require(in_place || out, "out-of-place conversion needs an output handle");
        auto converted = sk::densemat_convert_order(m->m, order_from(new_order), in_place != 0);
        if (out) *out = new sellkit_densemat{std::move(converted)};
    });
}

int sellkit_densemat_is_scattered(const sellkit_densemat* m) { return m && m->m.scattered() ? 1 : 0; }

sellkit_error sellkit_densemat_dims(const sellkit_densemat* m, sellkit_lidx* nrows, sellkit_lidx* ncols) {
    return guarded([&] {
        require(m != nullptr, "null handle");
        if (nrows) *nrows = m->m.nrows;
        if (ncols) *ncols = m->m.ncols;
    });
}

sellkit_error sellkit_densemat_copy_in(sellkit_densemat* m, const void* buf, size_t nelems) {
    return guarded([&] {
        require(m && buf, "null argument");
        sk::densemat_copy_in(m->m, buf, nelems);
    });
}

sellkit_error sellkit_densemat_copy_out(const sellkit_densemat* m, void* buf, size_t nelems) {
    return guarded([&] {
        require(m && buf, "null argument");
        sk::densemat_copy_out(m->m, buf, nelems);
    });
}

void sellkit_densemat_destroy(sellkit_densemat* m) { delete m; }

sellkit_error sellkit_axpby(sellkit_densemat* y, const sellkit_densemat* x, const void* alpha, const void* beta) {
    return guarded([&] {
        require(y && x, "null argument");
        same_dt(y->m.dt, x->m.dt, "y and x");
        unsigned char one[16] = {}, a[16], b[16];
        sk::visit_dt(y->m.dt, [&]<class T>() {
            T o = sk::Ops<T>::one();
            std::memcpy(one, &o, sizeof(T));
            return 0;
        });
        const std::size_t es = y->m.esize();
        std::memcpy(a, alpha ? alpha : one, es);
        std::memcpy(b, beta ? beta : one, es);  // capi.cpp:511: beta defaults to 1
        sk::blas_axpby(y->m, x->m, a, b, false);
    });
}

sellkit_error sellkit_vaxpby(sellkit_densemat* y, const sellkit_densemat* x, const void* alphas, const void* betas) {
    return guarded([&] {
        require(y && x && alphas && betas, "null argument");
        same_dt(y->m.dt, x->m.dt, "y and x");
        sk::blas_axpby(y->m, x->m, alphas, betas, true);
    });
}

sellkit_error sellkit_scal(sellkit_densemat* x, const void* factor) {
    return guarded([&] {
        require(x && factor, "null argument");
        sk::blas_scal(x->m, factor, false);
    });
}

sellkit_error sellkit_vscal(sellkit_densemat* x, const void* factors) {
    return guarded([&] {
        require(x && factors, "null argument");
        sk::blas_scal(x->m, factors, true);
    });
}

sellkit_error sellkit_dot(const sellkit_densemat* a, const sellkit_densemat* b, void* out) {
    return guarded([&] {
        require(a && b && out, "null argument");
        same_dt(a->m.dt, b->m.dt, "a and b");
        sk::blas_dot(a->m, b->m, out);
    });
}

/* --------------------------------------------------------------------- tsm */

sellkit_error sellkit_tsmttsm(sellkit_densemat* x, const sellkit_densemat* v, const sellkit_densemat* w,
                              const void* alpha, const void* beta, int kahan) {
    return guarded([&] {
        require(x && v && w, "null argument");
        same_dt(x->m.dt, v->m.dt, "x and v");
        same_dt(x->m.dt, w->m.dt, "x and w");
        sk::tsmttsm(x->m, v->m, w->m, alpha, beta, kahan != 0);
    });
}

sellkit_error sellkit_tsmm(sellkit_densemat* w, const sellkit_densemat* v, const sellkit_densemat* x, const void* alpha,
                           const void* beta) {
    return guarded([&] {
        require(w && v && x, "null argument");
        same_dt(w->m.dt, v->m.dt, "w and v");
        same_dt(w->m.dt, x->m.dt, "w and x");
        sk::tsmm(w->m, v->m, x->m, alpha, beta);
    });
}

sellkit_error sellkit_tsmm_inplace(sellkit_densemat* v, const sellkit_densemat* x, const void* alpha,
                                   const void* beta) {
    return guarded([&] {
        require(v && x, "null argument");
        same_dt(v->m.dt, x->m.dt, "v and x");
        sk::tsmm_inplace(v->m, x->m, alpha, beta);
    });
}

sellkit_error sellkit_gemm(sellkit_densemat* c, const sellkit_densemat* a, const sellkit_densemat* b, const void* alpha,
                           const void* beta, sellkit_trans ta, sellkit_trans tb) {
    return guarded([&] {
        require(c && a && b, "null argument");
        same_dt(c->m.dt, a->m.dt, "c and a");
        same_dt(c->m.dt, b->m.dt, "c and b");
        auto conv = [](sellkit_trans t) {
            switch (t) {
                case SELLKIT_TRANS_NONE: return sk::Trans::none;
                case SELLKIT_TRANS_T: return sk::Trans::transpose;
                case SELLKIT_TRANS_C: return sk::Trans::conj_transpose;
            }
            sk::fail(sk::errc::invalid_arg, "unknown transpose mode");
        };
        sk::gemm(c->m, a->m, b->m, alpha, beta, conv(ta), conv(tb));
    });
}

/* -------------------------------------------------------------------- spmv */

void sellkit_spmv_opts_init(sellkit_spmv_opts* opts) {
    if (opts) std::memset(opts, 0, sizeof(*opts));
}

sellkit_error sellkit_spmv(sellkit_densemat* y, const sellkit_mat* a, const sellkit_densemat* x,
                           const sellkit_spmv_opts* opts) {
    return guarded([&] {
        require(y && a && x, "null argument");
        same_dt(y->m.dt, a->p->dt, "y and A");
        same_dt(y->m.dt, x->m.dt, "y and x");
        sk::SpmvOptions o;
        if (opts) {
            sk::spmv_options_from(y->m.dt, opts->flags, opts->alpha, opts->beta, opts->gamma, opts->delta, opts->eta, o);
            o.dot = opts->dot;
            if (opts->z) {
                same_dt(y->m.dt, opts->z->m.dt, "y and z");
                o.z = &opts->z->m;
            }
        } else {
            sk::spmv_options_from(y->m.dt, 0, nullptr, nullptr, nullptr, nullptr, nullptr, o);
        }
        if (a->apply_override) {
            // spmv.hpp:131-135: validate, then hand the whole fused operation to the override
            sk::spmv_validate(y->m, *a->p, x->m, o);
            sellkit_spmv_opts dflt;
            sellkit_spmv_opts_init(&dflt);
            sk::DeviceGuard g(a->p->device);
            auto& rt = sk::runtime(a->p->device);
            const sellkit_error e = a->apply_override(y, x, opts ? opts : &dflt, rt.stream, a->apply_ctx);
            SK_REQUIRE(e == SELLKIT_OK, static_cast<sk::errc>(int(e)), "apply override failed");
            sk::finish(rt);
            return;
        }
        sk::spmv(y->m, *a->p, x->m, o);
    });
}

sellkit_error sellkit_ext_mat_set_apply_override(sellkit_mat* m, sellkit_ext_apply_fn fn, void* ctx) {
    return guarded([&] {
        require(m != nullptr, "null handle");
        m->apply_override = fn;
        m->apply_ctx = fn ? ctx : nullptr;
    });
}

sellkit_error sellkit_select_kernel(int chunk_height, sellkit_lidx block_width, sellkit_order order, int* variant_chunk,
                                    int* variant_width, int* vectorized) {
    return guarded([&] {
        const auto v = sk::select_kernel(chunk_height, block_width, order_from(order));
        if (variant_chunk) *variant_chunk = v.chunk_height;
        if (variant_width) *variant_width = v.block_width;
        if (vectorized) *vectorized = v.vectorized ? 1 : 0;
    });
}

/* ---------------------------------------------------------------- task pool */

sellkit_error sellkit_pool_create(int, const int*, int, sellkit_pool** out) {
    if (out) *out = nullptr;
    return SELLKIT_ERR_UNSUPPORTED;
}
sellkit_error sellkit_task_create(sellkit_pool*, sellkit_task_fn, void*, int, int, uint32_t, sellkit_task** out) {
    if (out) *out = nullptr;
    return SELLKIT_ERR_UNSUPPORTED;
}
sellkit_error sellkit_task_add_dependency(sellkit_task*, sellkit_task*) { return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_task_enqueue(sellkit_pool*, sellkit_task*) { return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_task_spawn_child(sellkit_pool*, sellkit_task*) { return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_task_wait(sellkit_pool*, sellkit_task*, void**) { return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_pool_current_task(sellkit_pool*, sellkit_task** out) {
    if (out) *out = nullptr;
    return SELLKIT_ERR_UNSUPPORTED;
}
sellkit_error sellkit_task_state_of(const sellkit_task*, sellkit_task_state*) { return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_task_destroy(sellkit_pool*, sellkit_task*) { return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_pool_shutdown(sellkit_pool*) { return SELLKIT_ERR_UNSUPPORTED; }
int sellkit_pool_npus(const sellkit_pool*) { return 0; }
int sellkit_pool_num_numa_nodes(const sellkit_pool*) { return 0; }
sellkit_error sellkit_pool_numa_node_of(const sellkit_pool*, int, int*) { return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_pool_trace(const sellkit_pool*, char** out) {
    if (out) *out = nullptr;
    return SELLKIT_ERR_UNSUPPORTED;
}
void sellkit_pool_destroy(sellkit_pool*) {}

void sellkit_string_free(char* s) { delete[] s; }

/* -------------------------------------------------------- performance model */
// perfmodel.cpp:11-45

sellkit_error sellkit_spmv_code_balance(sellkit_datatype dt, int index_bytes, int include_vectors,
                                        double avg_nnz_per_row, double* out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        const sk::Datatype d = dt_from(dt);
        SK_REQUIRE(index_bytes > 0, sk::errc::invalid_arg, "index bytes must be positive");
        const double vb = double(sk::value_bytes(d));
        const double flops = sk::is_complex(d) ? 8.0 : 2.0;
        double balance = (vb + index_bytes) / flops;
        if (include_vectors) {
            SK_REQUIRE(avg_nnz_per_row > 0, sk::errc::invalid_arg, "average row length must be positive");
            balance += (2.0 * vb + vb) / (flops * avg_nnz_per_row);
        }
        *out = balance;
    });
}

sellkit_error sellkit_index_width_saving(int value_bytes, double* out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        SK_REQUIRE(value_bytes == 4 || value_bytes == 8 || value_bytes == 16, sk::errc::unsupported,
                   "unsupported value width");
        *out = 4.0 / (value_bytes + 8.0);
    });
}

sellkit_error sellkit_roofline_bound(double bandwidth_gbs, double peak_gflops, double code_balance, double* out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        SK_REQUIRE(bandwidth_gbs > 0 && peak_gflops > 0, sk::errc::invalid_arg,
                   "machine model parameters must be positive");
        SK_REQUIRE(code_balance >= 0, sk::errc::invalid_arg, "negative code balance");
        *out = code_balance == 0.0 ? peak_gflops : std::min(peak_gflops, bandwidth_gbs / code_balance);
    });
}

sellkit_error sellkit_crs_refresh_cost(sellkit_gidx nnz, int value_bytes, double spmv_traffic_per_call, double* out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        SK_REQUIRE(nnz > 0 && value_bytes > 0 && spmv_traffic_per_call > 0, sk::errc::invalid_arg,
                   "refresh cost inputs must be positive");
        *out = 3.0 * double(nnz) * value_bytes / spmv_traffic_per_call;
    });
}

sellkit_error sellkit_region_create(const char* name, sellkit_region** out) {
    return guarded([&] {
        require(name && out, "null argument");
        *out = new sellkit_region{name, {}};
    });
}

sellkit_error sellkit_region_record(sellkit_region* region, double sample) {
    return guarded([&] {
        require(region != nullptr, "null handle");
        region->samples.push_back(sample);
    });
}

// perfmodel.cpp:47-56
sellkit_error sellkit_region_p_max(const sellkit_region* region, double* out) {
    return guarded([&] {
        require(region && out, "null argument");
        SK_REQUIRE(!region->samples.empty(), sk::errc::state, "region has no samples");
        *out = *std::max_element(region->samples.begin(), region->samples.end());
    });
}

sellkit_error sellkit_region_p_skip10(const sellkit_region* region, double* out) {
    return guarded([&] {
        require(region && out, "null argument");
        SK_REQUIRE(region->samples.size() > 10, sk::errc::state, "P_skip10 needs more than ten calls");
        *out = std::accumulate(region->samples.begin() + 10, region->samples.end(), 0.0) /
               double(region->samples.size() - 10);
    });
}

// perfmodel.cpp:58-77: byte-stable table format
sellkit_error sellkit_region_table(const sellkit_region* const* regions, int nregions, char** out) {
    return guarded([&] {
        require(regions && out, "null argument");
        std::string text;
        char line[160];
        std::snprintf(line, sizeof(line), "%-12s| %5s | %8s | %8s\n", "Region", "Calls", "P_max", "P_skip10");
        text += line;
        text += std::string(41, '-') + "\n";
        for (int i = 0; i < nregions; ++i) {
            const sellkit_region* r = regions[i];
            SK_REQUIRE(!r->samples.empty(), sk::errc::state, "region has no samples");
            const double pmax = *std::max_element(r->samples.begin(), r->samples.end());
            std::string skip = "n/a";
            if (r->samples.size() > 10)
                skip = sci(std::accumulate(r->samples.begin() + 10, r->samples.end(), 0.0) /
                           double(r->samples.size() - 10));
            std::snprintf(line, sizeof(line), "%-12s| %5zu | %8s | %8s\n", r->name.c_str(), r->samples.size(),
                          sci(pmax).c_str(), skip.c_str());
            text += line;
        }
        *out = dup_string(text);
    });
}

void sellkit_region_destroy(sellkit_region* region) { delete region; }

/* ------------------------------------------------------------ extensions -- */

const char* sellkit_ext_last_error(void) { return sk::last_error_message(); }

sellkit_error sellkit_ext_set_sync(int sync) {
    return guarded([&] { sk::set_sync_mode(sync != 0); });
}

sellkit_error sellkit_ext_synchronize(void) {
    return guarded([&] { CK(cudaStreamSynchronize(sk::runtime(sk::current_device()).stream)); });
}

sellkit_error sellkit_ext_release_cached(void) {
    return guarded([&] { sk::release_cached_all(); });
}

sellkit_error sellkit_ext_stream(void** stream) {
    return guarded([&] {
        require(stream != nullptr, "null output");
        *stream = sk::runtime(sk::current_device()).stream;
    });
}

sellkit_error sellkit_ext_device_info(int* device, int* num_sms, size_t* l2_bytes) {
    return guarded([&] {
        auto& rt = sk::runtime(sk::current_device());
        if (device) *device = rt.device;
        if (num_sms) *num_sms = rt.num_sms;
        if (l2_bytes) *l2_bytes = rt.l2_bytes;
    });
}

sellkit_error sellkit_ext_crs_create_device(sellkit_datatype dt, sellkit_gidx nrows, sellkit_gidx ncols,
                                            const sellkit_gidx* rowptr, const sellkit_gidx* col, const void* val,
                                            sellkit_crs** out) {
    return guarded([&] {
        require(out && rowptr, "null argument");
        *out = new sellkit_crs{sk::crs_from_device(dt_from(dt), nrows, ncols, rowptr, col, val)};
    });
}

sellkit_error sellkit_ext_crs_stencil(sellkit_datatype dt, int points, sellkit_gidx n, sellkit_gidx row_begin,
                                      sellkit_gidx row_end, sellkit_crs** out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        *out = new sellkit_crs{sk::crs_stencil(dt_from(dt), points, n, row_begin, row_end)};
    });
}

sellkit_error sellkit_ext_crs_ti(sellkit_datatype dt, sellkit_gidx lx, sellkit_gidx ly, sellkit_gidx lz,
                                 double disorder, sellkit_gidx row_begin, sellkit_gidx row_end, sellkit_crs** out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        *out = new sellkit_crs{sk::crs_ti(dt_from(dt), lx, ly, lz, disorder, row_begin, row_end)};
    });
}

sellkit_error sellkit_ext_mat_info(const sellkit_mat* m, int* chunk_height, int* sigma, sellkit_lidx* nrows_padded,
                                   sellkit_gidx* nchunks, sellkit_gidx* slots, int* cols_permuted) {
    return guarded([&] {
        require(m != nullptr, "null handle");
        const auto& a = *m->p;
        if (chunk_height) *chunk_height = a.C;
        if (sigma) *sigma = a.sigma;
        if (nrows_padded) *nrows_padded = a.nrows_padded;
        if (nchunks) *nchunks = a.nchunks;
        if (slots) *slots = a.slots;
        if (cols_permuted) *cols_permuted = a.cols_permuted ? 1 : 0;
    });
}

sellkit_error sellkit_ext_mat_export(const sellkit_mat* m, int32_t* row_perm_inv, int32_t* row_perm, int32_t* rowlen,
                                     int32_t* chunk_len, int64_t* chunk_offset, void* val, int32_t* col) {
    return guarded([&] {
        require(m != nullptr, "null handle");
        const auto& a = *m->p;
        sk::DeviceGuard g(a.device);
        auto& rt = sk::runtime(a.device);
        auto cp = [&](void* dst, const sk::DeviceBuffer& src, std::size_t bytes) {
            if (dst && bytes) CK(cudaMemcpyAsync(dst, src.get(), bytes, cudaMemcpyDeviceToHost, rt.stream));
        };
        cp(row_perm_inv, a.row_perm_inv, std::size_t(a.nrows) * 4);
        cp(row_perm, a.row_perm, std::size_t(a.nrows) * 4);
        cp(rowlen, a.rowlen, std::size_t(a.nrows_padded) * 4);
        cp(chunk_len, a.chunk_len, std::size_t(a.nchunks) * 4);
        cp(chunk_offset, a.chunk_offset, std::size_t(a.nchunks + 1) * 8);
        cp(val, a.val, std::size_t(a.slots) * sk::value_bytes(a.dt));
        cp(col, a.col, std::size_t(a.slots) * 4);
        CK(cudaStreamSynchronize(rt.stream));
    });
}

sellkit_error sellkit_ext_mat_set_sweep_order(sellkit_mat* m, sellkit_lidx block_rows, const int32_t* order,
                                              sellkit_gidx nblocks) {
    return guarded([&] {
        require(m != nullptr, "null handle");
        auto& a = *m->p;
        if (!order) {
            // block_rows == 0: back to the automatic locality order; otherwise natural row order
            a.sweep_order = sk::DeviceBuffer();
            a.sweep_block_rgs = 0;
            a.sweep_blocks = 0;
            a.sweep_policy = block_rows == 0 ? 0 : 1;
            return;
        }
        SK_REQUIRE(block_rows > 0 && block_rows % 32 == 0 && block_rows <= 32 * 4096, sk::errc::invalid_arg,
                   "block_rows must be a positive multiple of 32");
        const sellkit_gidx want = (sellkit_gidx(a.nrows_padded) + block_rows - 1) / block_rows;
        SK_REQUIRE(nblocks == want, sk::errc::shape_mismatch, "nblocks must be ceil(nrows_padded / block_rows)");
        std::vector<char> seen(std::size_t(nblocks), 0);
        for (sellkit_gidx i = 0; i < nblocks; ++i) {
            SK_REQUIRE(order[i] >= 0 && order[i] < nblocks && !seen[std::size_t(order[i])], sk::errc::invalid_arg,
                       "order must be a permutation of the block indices");
            seen[std::size_t(order[i])] = 1;
        }
        sk::DeviceGuard g(a.device);
        auto& rt = sk::runtime(a.device);
        sk::DeviceBuffer buf(std::size_t(nblocks) * sizeof(int32_t), a.device);
        CK(cudaMemcpyAsync(buf.get(), order, std::size_t(nblocks) * sizeof(int32_t), cudaMemcpyHostToDevice, rt.stream));
        CK(cudaStreamSynchronize(rt.stream));
        a.sweep_order = std::move(buf);
        a.sweep_block_rgs = int(block_rows / 32);
        a.sweep_blocks = nblocks;
        a.sweep_policy = 2;
    });
}

sellkit_error sellkit_ext_densemat_storage(const sellkit_densemat* m, void** data, sellkit_lidx* stride, int* order,
                                           int* device, int* on_device) {
    return guarded([&] {
        require(m != nullptr, "null handle");
        if (data) *data = m->m.data;
        if (stride) *stride = m->m.stride;
        if (order) *order = int(m->m.order);
        if (device) *device = m->m.device;
        if (on_device) *on_device = m->m.mem == sk::MemKind::device ? 1 : 0;
    });
}

sellkit_error sellkit_ext_densemat_fill_hash(sellkit_densemat* m, uint64_t seed) {
    return guarded([&] {
        require(m != nullptr, "null handle");
        sk::densemat_fill_hash(m->m, seed);
    });
}

}  // extern "C"
