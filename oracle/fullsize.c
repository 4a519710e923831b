/*
 * fullsize -- CPU checkers for the BASELINE-size parity tests.
 *
 * TEST INFRASTRUCTURE ONLY (like sellkit_oracle.c): only tests/, smoke() and
 * bench.py's cpu_baseline / reference legs may load it, and only as the checker
 * or the input generator of the reference arm.  The product library never links it.
 *
 * At the BASELINE sizes (64 M-row stencil, N = 1e8 tall-skinny blocks) the host
 * copies of every operand would not fit a test, so the checkers REGENERATE the
 * operands from the same counter hash the device fills them with
 * (sellkit_ext_densemat_fill_hash: U(-1,1) from splitmix64(seed ^ (i*ncols+j)),
 * mapped by (h >> 11) * 2^-53 * 2 - 1), and OpenMP parallelises over rows --
 * every row's arithmetic is sequential, so results do not depend on the thread
 * count.
 *
 *  - fs_stencil7_crs: the 3-D 7-point Laplacian CRS rows [r0, r1) (diagonal 6,
 *    neighbours -1, columns ascending, Dirichlet) -- the matrix of
 *    sellkit_ext_crs_stencil / oracle.stencil_crs, for the reference library.
 *  - fs_hash_block: the hash fill of an n x w block.
 *  - fs_tsmm_rows: TSMM rows W[i,:] = alpha * sum_m V[i,m] X[m,:] + beta * W0[i,:]
 *    in the reference's order (proj/src/tsm.hpp:51-68: tmp[k] += V[i,m] * X[m,k]
 *    over m ascending from 0, then alpha * tmp + beta * W), V and W0 regenerated.
 *  - fs_tsmttsm: X = V^T W over all rows with long-double accumulation (the
 *    "true" value for the tolerance check; the reference's own order depends on
 *    its worker count, tsm.hpp:105-178), plus sum_i |V[i,a]| |W[i,b]| per cell.
 *
 * Compiled with -ffp-contract=off (two roundings per a*b+c, like the reference).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

static inline uint64_t fs_splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline double fs_hash(uint64_t seed, uint64_t idx) {
    const uint64_t h = fs_splitmix64(seed ^ idx);
    return (double)(h >> 11) * 0x1p-53 * 2.0 - 1.0;
}

void fs_hash_block(int64_t nrows, int32_t ncols, uint64_t seed, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; ++i)
        for (int32_t j = 0; j < ncols; ++j) out[i * ncols + j] = fs_hash(seed, (uint64_t)(i * ncols + j));
}

/* rows [r0, r1) of the n^3 7-point Laplacian; rowptr[r1 - r0 + 1] starts at 0 */
void fs_stencil7_crs(int64_t n, int64_t r0, int64_t r1, int64_t* rowptr, int64_t* col, double* val) {
    const int64_t n2 = n * n;
    const int64_t rows = r1 - r0;
    /* row lengths are 7 minus the number of boundary faces: prefix sum first */
    rowptr[0] = 0;
    for (int64_t k = 0; k < rows; ++k) {
        const int64_t r = r0 + k;
        const int64_t x = r % n, y = (r / n) % n, z = r / n2;
        rowptr[k + 1] = rowptr[k] + 1 + (z > 0) + (y > 0) + (x > 0) + (x + 1 < n) + (y + 1 < n) + (z + 1 < n);
    }
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < rows; ++k) {
        const int64_t r = r0 + k;
        const int64_t x = r % n, y = (r / n) % n, z = r / n2;
        int64_t p = rowptr[k];
        if (z > 0) { col[p] = r - n2; val[p++] = -1.0; }
        if (y > 0) { col[p] = r - n; val[p++] = -1.0; }
        if (x > 0) { col[p] = r - 1; val[p++] = -1.0; }
        col[p] = r; val[p++] = 6.0;
        if (x + 1 < n) { col[p] = r + 1; val[p++] = -1.0; }
        if (y + 1 < n) { col[p] = r + n; val[p++] = -1.0; }
        if (z + 1 < n) { col[p] = r + n2; val[p++] = -1.0; }
    }
}

/* TSMM rows [i0, i1): out[(i - i0) * k + c]; X row-major m x k (x[a*k + c]).
 * V[i,a] = hash(seed_v, i*m + a); W0[i,c] = hash(seed_w, i*k + c) (read only if beta != 0,
 * but always multiplied like the reference: beta * W). */
void fs_tsmm_rows(int64_t i0, int64_t i1, int32_t m, int32_t k, uint64_t seed_v, const double* x, double alpha,
                  double beta, uint64_t seed_w, double* out) {
#pragma omp parallel
    {
        double* tmp = (double*)malloc(sizeof(double) * (size_t)k);
#pragma omp for schedule(static)
        for (int64_t i = i0; i < i1; ++i) {
            for (int32_t c = 0; c < k; ++c) tmp[c] = 0.0;
            for (int32_t a = 0; a < m; ++a) {
                const double va = fs_hash(seed_v, (uint64_t)(i * m + a));
                for (int32_t c = 0; c < k; ++c) tmp[c] += va * x[a * k + c];
            }
            for (int32_t c = 0; c < k; ++c) {
                const double w0 = fs_hash(seed_w, (uint64_t)(i * k + c));
                out[(i - i0) * k + c] = alpha * tmp[c] + beta * w0;
            }
        }
        free(tmp);
    }
}

/* X[a*k + b] = sum_i V[i,a] W[i,b] (long double), scale[a*k + b] = sum_i |V[i,a]| |W[i,b]| */
void fs_tsmttsm(int64_t n, int32_t m, int32_t k, uint64_t seed_v, uint64_t seed_w, double* x, double* scale) {
    const int64_t cells = (int64_t)m * k;
    long double* acc = (long double*)calloc((size_t)cells, sizeof(long double));
    long double* sc = (long double*)calloc((size_t)cells, sizeof(long double));
#pragma omp parallel
    {
        long double* la = (long double*)calloc((size_t)cells, sizeof(long double));
        long double* ls = (long double*)calloc((size_t)cells, sizeof(long double));
        double* vr = (double*)malloc(sizeof(double) * (size_t)m);
        double* wr = (double*)malloc(sizeof(double) * (size_t)k);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            for (int32_t a = 0; a < m; ++a) vr[a] = fs_hash(seed_v, (uint64_t)(i * m + a));
            for (int32_t b = 0; b < k; ++b) wr[b] = fs_hash(seed_w, (uint64_t)(i * k + b));
            for (int32_t a = 0; a < m; ++a)
                for (int32_t b = 0; b < k; ++b) {
                    const long double p = (long double)vr[a] * (long double)wr[b];
                    la[a * k + b] += p;
                    ls[a * k + b] += fabsl(p);
                }
        }
#pragma omp critical
        for (int64_t c = 0; c < cells; ++c) {
            acc[c] += la[c];
            sc[c] += ls[c];
        }
        free(la);
        free(ls);
        free(vr);
        free(wr);
    }
    for (int64_t c = 0; c < cells; ++c) {
        x[c] = (double)acc[c];
        scale[c] = (double)sc[c];
    }
    free(acc);
    free(sc);
}

/* Long-double column dots of row-major n x w blocks: out[j] = sum_i a[i,j] b[i,j],
 * scale[j] = sum_i |a[i,j] b[i,j]| (the reference value for dot tolerances). */
void fs_dot_cols(int64_t n, int32_t w, const double* a, const double* b, double* out, double* scale) {
    long double* acc = (long double*)calloc((size_t)w, sizeof(long double));
    long double* sc = (long double*)calloc((size_t)w, sizeof(long double));
#pragma omp parallel
    {
        long double* la = (long double*)calloc((size_t)w, sizeof(long double));
        long double* ls = (long double*)calloc((size_t)w, sizeof(long double));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i)
            for (int32_t j = 0; j < w; ++j) {
                const long double p = (long double)a[i * w + j] * (long double)b[i * w + j];
                la[j] += p;
                ls[j] += fabsl(p);
            }
#pragma omp critical
        for (int32_t j = 0; j < w; ++j) {
            acc[j] += la[j];
            sc[j] += ls[j];
        }
        free(la);
        free(ls);
    }
    for (int32_t j = 0; j < w; ++j) {
        out[j] = (double)acc[j];
        scale[j] = (double)sc[j];
    }
    free(acc);
    free(sc);
}

/* complex interleaved (re, im): out[2j..2j+1] = sum_i conj(a[i,j]) b[i,j], scale[j] = sum_i |a[i,j]| |b[i,j]| */
void fs_zdot_cols(int64_t n, int32_t w, const double* a, const double* b, double* out, double* scale) {
    long double* acc = (long double*)calloc(2 * (size_t)w, sizeof(long double));
    long double* sc = (long double*)calloc((size_t)w, sizeof(long double));
#pragma omp parallel
    {
        long double* la = (long double*)calloc(2 * (size_t)w, sizeof(long double));
        long double* ls = (long double*)calloc((size_t)w, sizeof(long double));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i)
            for (int32_t j = 0; j < w; ++j) {
                const long double ar = a[2 * (i * w + j)], ai = a[2 * (i * w + j) + 1];
                const long double br = b[2 * (i * w + j)], bi = b[2 * (i * w + j) + 1];
                la[2 * j] += ar * br + ai * bi;
                la[2 * j + 1] += ar * bi - ai * br;
                ls[j] += sqrtl(ar * ar + ai * ai) * sqrtl(br * br + bi * bi);
            }
#pragma omp critical
        for (int32_t j = 0; j < w; ++j) {
            acc[2 * j] += la[2 * j];
            acc[2 * j + 1] += la[2 * j + 1];
            sc[j] += ls[j];
        }
        free(la);
        free(ls);
    }
    for (int32_t j = 0; j < w; ++j) {
        out[2 * j] = (double)acc[2 * j];
        out[2 * j + 1] = (double)acc[2 * j + 1];
        scale[j] = (double)sc[j];
    }
    free(acc);
    free(sc);
}
