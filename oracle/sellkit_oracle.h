/*
 * sellkit_oracle -- CPU restatement of the reference's SELL-C-sigma hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load this library, and only as the checker.
 * The product library (paper_1507_08101_b200/lib/libsellkit_b200.so) never
 * links it and has no CPU fallback.
 *
 * Parity pinning: every function below is checked against the reference's own
 * known-answer tests and against golden fixtures produced by the reference
 * itself (oracle/_ref, tests/golden/make_golden.py) in tests/test_oracle.py.
 *
 * Floating point: compiled with -ffp-contract=off so that every a*b+c is two
 * roundings, exactly like the reference's Release build (x86-64 baseline, no
 * FMA).  Summation orders follow the reference line by line, so results are
 * bit-identical to the reference for a given worker count.
 *
 * Complex values (dt == 1) are interleaved (re, im) doubles, like
 * std::complex<double> in the reference.
 */
#ifndef SELLKIT_ORACLE_H
#define SELLKIT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype selector: 0 = real double (R64), 1 = complex double (C64) */

/* sellcs.hpp:80-91 */
void or_sigma_permutation(const int32_t* lens, int64_t n, int32_t sigma, int32_t* order);

typedef struct or_sell {
    int32_t nrows, ncols, nrows_padded, C, sigma, cols_permuted, dt;
    int64_t nnz, nchunks, slots;
    int32_t* row_perm_inv; /* [nrows]   stored -> original   */
    int32_t* row_perm;     /* [nrows]   original -> stored   */
    int32_t* rowlen;       /* [nrows_padded]                 */
    int32_t* chunk_len;    /* [nchunks]                      */
    int64_t* chunk_offset; /* [nchunks+1]                    */
    double* val;           /* [slots] (x2 for complex)       */
    int32_t* col;          /* [slots]                        */
    double beta;
} or_sell;

/* sellcs.hpp:143-232 (build_sell) via build(CrsData) :236-246.
 * imposed_order may be NULL.  Returns 0 or a sellkit error code
 * (1 invalid_arg, 2 overflow). */
int or_sell_build(int dt, int64_t nrows, int64_t ncols, const int64_t* rowptr, const int64_t* col,
                  const double* val, int32_t C, int32_t sigma, int permute_columns,
                  const int32_t* imposed_order, or_sell** out);
void or_sell_free(or_sell* m);

/* detail::worker_blocks densemat.hpp:230-238: number of blocks and block b's range */
int64_t or_worker_blocks(int64_t n, int workers, int64_t b, int64_t* begin, int64_t* end);

/* Fused SpMV spmv.hpp:129-202 + spmv_generic :68-92 + spmv_store_row
 * spmv_epilogue.hpp:12-36.  x/y/z are block vectors addressed as
 * base + row*rs + col*cs (elements).  Dots follow the reference's per-worker
 * partial order for `workers` workers.  flags as in sellkit.h. */
void or_spmv(const or_sell* A, double* y, int64_t y_rs, int64_t y_cs, const double* x,
             int64_t x_rs, int64_t x_cs, double* z, int64_t z_rs, int64_t z_cs, int32_t width,
             uint32_t flags, const double* alpha, const double* beta, const double* gamma,
             const double* gamma_list, const double* delta, const double* eta, double* dot,
             int workers);

/* tsm.hpp:105-178: X(m x k, element (i,j) at x[i*x_rs + j*x_cs]) = alpha V^H W + beta X.
 * V (n x m), W (n x k) row-major with row strides v_rs / w_rs. */
void or_tsmttsm(int dt, int64_t n, int32_t m, int32_t k, double* x, int64_t x_rs, int64_t x_cs,
                const double* v, int64_t v_rs, const double* w, int64_t w_rs, const double* alpha,
                const double* beta, int kahan, int workers);

/* tsm.hpp:182-225: W(n x k) = alpha V X + beta W, X (m x k) at x[i*x_rs + j*x_cs]. */
void or_tsmm(int dt, int64_t n, int32_t m, int32_t k, double* w, int64_t w_rs, const double* v,
             int64_t v_rs, const double* x, int64_t x_rs, int64_t x_cs, const double* alpha,
             const double* beta);

/* tsm.hpp:230-249: V(n x m) = alpha V X + beta V, X (m x m). */
void or_tsmm_inplace(int dt, int64_t n, int32_t m, double* v, int64_t v_rs, const double* x,
                     int64_t x_rs, int64_t x_cs, const double* alpha, const double* beta);

/* densemat.hpp:276-292: out[j] = sum_i conj(a[i,j]) b[i,j], worker-block order. */
void or_dot(int dt, int64_t n, int32_t w, const double* a, int64_t a_rs, int64_t a_cs,
            const double* b, int64_t b_rs, int64_t b_cs, double* out, int workers);

/* partition.hpp:45-94.  rowlens may be NULL for BY_ROWS.  Returns 0 or an error code. */
int or_partition(int64_t n, const int32_t* rowlens, const double* weights, int k, int by_nnz,
                 int64_t* row_offset);

#ifdef __cplusplus
}
#endif

#endif
