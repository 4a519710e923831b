/*
 * sellkit_oracle.c -- CPU restatement of the reference's SELL-C-sigma hot path.
 * TEST INFRASTRUCTURE ONLY (see sellkit_oracle.h).  Compiled with
 * -ffp-contract=off.  Every function cites the reference file:line it follows
 * (paths relative to /root/reference/proj).
 */
#include "sellkit_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double complex zdouble;

/* ------------------------------------------------------------ sigma sort -- */

/* Stable merge sort of idx[lo,hi) by descending lens[idx]. */
static void msort_desc(int32_t* idx, int32_t* tmp, int64_t lo, int64_t hi, const int32_t* lens) {
    if (hi - lo < 2) return;
    const int64_t mid = lo + (hi - lo) / 2;
    msort_desc(idx, tmp, lo, mid, lens);
    msort_desc(idx, tmp, mid, hi, lens);
    int64_t i = lo, j = mid, o = lo;
    while (i < mid && j < hi) {
        /* take from the right only if strictly longer: stability */
        if (lens[idx[j]] > lens[idx[i]])
            tmp[o++] = idx[j++];
        else
            tmp[o++] = idx[i++];
    }
    while (i < mid) tmp[o++] = idx[i++];
    while (j < hi) tmp[o++] = idx[j++];
    memcpy(idx + lo, tmp + lo, (size_t)(hi - lo) * sizeof(int32_t));
}

/* sellcs.hpp:80-91: per-scope stable sort by descending row length. */
void or_sigma_permutation(const int32_t* lens, int64_t n, int32_t sigma, int32_t* order) {
    for (int64_t i = 0; i < n; ++i) order[i] = (int32_t)i;
    if (sigma <= 1) return;
    int32_t* tmp = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    for (int64_t s = 0; s < n; s += sigma) {
        const int64_t e = (s + sigma < n) ? s + sigma : n;
        msort_desc(order, tmp, s, e, lens);
    }
    free(tmp);
}

/* ----------------------------------------------------------------- build -- */

void or_sell_free(or_sell* m) {
    if (!m) return;
    free(m->row_perm_inv);
    free(m->row_perm);
    free(m->rowlen);
    free(m->chunk_len);
    free(m->chunk_offset);
    free(m->val);
    free(m->col);
    free(m);
}

/* sellcs.hpp:28-33 (validate), :143-232 (build_sell), :236-246 (build from CRS). */
int or_sell_build(int dt, int64_t nrows, int64_t ncols, const int64_t* rowptr, const int64_t* col,
                  const double* val, int32_t C, int32_t sigma, int permute_columns,
                  const int32_t* imposed_order, or_sell** out) {
    *out = NULL;
    if (C < 1 || sigma < 1) return 1;
    if (!(sigma == 1 || sigma % C == 0 || sigma >= nrows)) return 1;
    if (nrows < 0 || ncols < 0) return 1;
    if (nrows >= ((int64_t)1 << 31) || ncols >= ((int64_t)1 << 31)) return 2;
    if (nrows <= 0) return 1;
    if (permute_columns && nrows != ncols) return 1;
    const int vw = dt ? 2 : 1; /* doubles per value */

    or_sell* m = (or_sell*)calloc(1, sizeof(or_sell));
    m->nrows = (int32_t)nrows;
    m->ncols = (int32_t)ncols;
    m->C = C;
    m->sigma = sigma;
    m->dt = dt;
    m->cols_permuted = permute_columns ? 1 : 0;
    const int32_t n = m->nrows;

    int32_t* lens = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    for (int32_t r = 0; r < n; ++r) lens[r] = (int32_t)(rowptr[r + 1] - rowptr[r]);

    m->row_perm_inv = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    if (imposed_order)
        memcpy(m->row_perm_inv, imposed_order, (size_t)n * sizeof(int32_t));
    else
        or_sigma_permutation(lens, n, sigma, m->row_perm_inv);
    m->row_perm = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    for (int32_t k = 0; k < n; ++k) m->row_perm[m->row_perm_inv[k]] = k;

    const int64_t nchunks = ((int64_t)n + C - 1) / C;
    m->nchunks = nchunks;
    m->nrows_padded = (int32_t)(nchunks * C);
    m->rowlen = (int32_t*)calloc((size_t)m->nrows_padded, sizeof(int32_t));
    for (int32_t k = 0; k < n; ++k) m->rowlen[k] = lens[m->row_perm_inv[k]];

    m->chunk_len = (int32_t*)calloc((size_t)nchunks, sizeof(int32_t));
    m->chunk_offset = (int64_t*)calloc((size_t)nchunks + 1, sizeof(int64_t));
    for (int64_t c = 0; c < nchunks; ++c) {
        int32_t lc = 0;
        for (int32_t i = 0; i < C; ++i)
            if (m->rowlen[c * C + i] > lc) lc = m->rowlen[c * C + i];
        m->chunk_len[c] = lc;
        m->chunk_offset[c + 1] = m->chunk_offset[c] + (int64_t)C * lc;
    }
    m->slots = m->chunk_offset[nchunks];
    m->val = (double*)calloc((size_t)(m->slots > 0 ? m->slots : 1) * vw, sizeof(double));
    m->col = (int32_t*)calloc((size_t)(m->slots > 0 ? m->slots : 1), sizeof(int32_t));
    int64_t nnz = 0;
    for (int32_t r = 0; r < n; ++r) nnz += lens[r];
    m->nnz = nnz;
    m->beta = m->slots > 0 ? (double)nnz / (double)m->slots : 1.0;

    int err = 0;
    for (int64_t c = 0; c < nchunks && !err; ++c) {
        for (int32_t i = 0; i < C; ++i) {
            const int64_t stored = c * C + i;
            if (stored >= n) continue;
            const int32_t orig = m->row_perm_inv[stored];
            const int32_t len = lens[orig];
            for (int32_t j = 0; j < len; ++j) {
                const int64_t g = col[rowptr[orig] + j];
                if (g < 0 || g >= ncols) { err = 1; break; }
                const int32_t sc = m->cols_permuted ? m->row_perm[g] : (int32_t)g;
                const int64_t slot = m->chunk_offset[c] + (int64_t)j * C + i;
                for (int q = 0; q < vw; ++q) m->val[slot * vw + q] = val[(rowptr[orig] + j) * vw + q];
                m->col[slot] = sc;
            }
            if (err) break;
        }
    }
    free(lens);
    if (err) {
        or_sell_free(m);
        return 1;
    }
    *out = m;
    return 0;
}

/* densemat.hpp:230-238 */
int64_t or_worker_blocks(int64_t n, int workers, int64_t b, int64_t* begin, int64_t* end) {
    if (n <= 0) return 0;
    const int64_t w = workers > 1 ? workers : 1;
    const int64_t chunk = (n + w - 1) / w;
    int64_t nb = 0;
    while (nb * chunk < n) ++nb;
    if (begin && end && b < nb) {
        *begin = b * chunk;
        *end = (b + 1) * chunk < n ? (b + 1) * chunk : n;
    }
    return nb;
}

/* ------------------------------------------------------------------ spmv -- */

#define F_AXPBY 0x01u
#define F_SHIFT 0x02u
#define F_VSHIFT 0x04u
#define F_DOT_YY 0x08u
#define F_DOT_XY 0x10u
#define F_DOT_XX 0x20u
#define F_CHAIN 0x40u

/* spmv_generic (spmv.hpp:68-92) + spmv_store_row (spmv_epilogue.hpp:12-36), real. */
static void spmv_real(const or_sell* A, double* y, int64_t y_rs, int64_t y_cs, const double* x,
                      int64_t x_rs, int64_t x_cs, double* z, int64_t z_rs, int64_t z_cs, int32_t w,
                      uint32_t f, double alpha, double beta, double gamma0, const double* gl,
                      double delta, double eta, double* dot, int workers) {
    const int32_t C = A->C;
    int64_t nb = or_worker_blocks(A->nchunks, workers, 0, NULL, NULL);
    const int64_t dotn = 3 * (int64_t)w;
    double* partials = (double*)calloc((size_t)(nb > 0 ? nb : 1) * dotn, sizeof(double));
    double* acc = (double*)malloc((size_t)C * w * sizeof(double));
    for (int64_t bi = 0; bi < nb; ++bi) {
        int64_t c0, c1;
        or_worker_blocks(A->nchunks, workers, bi, &c0, &c1);
        double* dotp = partials + bi * dotn;
        for (int64_t c = c0; c < c1; ++c) {
            const int64_t off = A->chunk_offset[c];
            const int32_t len = A->chunk_len[c];
            for (int64_t q = 0; q < (int64_t)C * w; ++q) acc[q] = 0.0;
            for (int32_t j = 0; j < len; ++j) {
                const double* vj = A->val + off + (int64_t)j * C;
                const int32_t* cj = A->col + off + (int64_t)j * C;
                for (int32_t r = 0; r < C; ++r) {
                    const double mv = vj[r];
                    const double* xr = x + (int64_t)cj[r] * x_rs;
                    double* ar = acc + (int64_t)r * w;
                    for (int32_t v = 0; v < w; ++v) ar[v] += mv * xr[v * x_cs];
                }
            }
            for (int32_t r = 0; r < C; ++r) {
                const int64_t row = c * C + r;
                if (row >= A->nrows) continue;
                double* yr = y + row * y_rs;
                const double* xr = x + row * x_rs;
                for (int32_t v = 0; v < w; ++v) {
                    double t = acc[(int64_t)r * w + v];
                    if (f & F_SHIFT) t -= gamma0 * xr[v * x_cs];
                    if (f & F_VSHIFT) t -= gl[v] * xr[v * x_cs];
                    t *= alpha;
                    if (f & F_AXPBY) t += beta * yr[v * y_cs];
                    yr[v * y_cs] = t;
                    if (f & F_CHAIN) {
                        double* zr = z + row * z_rs;
                        zr[v * z_cs] = delta * zr[v * z_cs] + eta * t;
                    }
                    if (f & F_DOT_YY) dotp[v] += t * t;
                    if (f & F_DOT_XY) dotp[w + v] += xr[v * x_cs] * t;
                    if (f & F_DOT_XX) dotp[2 * w + v] += xr[v * x_cs] * xr[v * x_cs];
                }
            }
        }
    }
    /* spmv.hpp:188-201: combine block partials in block order */
    for (int seg = 0; seg < 3; ++seg) {
        const uint32_t want = seg == 0 ? F_DOT_YY : seg == 1 ? F_DOT_XY : F_DOT_XX;
        if (!(f & want)) continue;
        for (int32_t v = 0; v < w; ++v) {
            double s = 0.0;
            for (int64_t bi = 0; bi < nb; ++bi) s += partials[bi * dotn + seg * w + v];
            dot[seg * w + v] = s;
        }
    }
    free(acc);
    free(partials);
}

static inline zdouble zload(const double* p) { return CMPLX(p[0], p[1]); }
static inline void zstore(double* p, zdouble v) {
    p[0] = creal(v);
    p[1] = cimag(v);
}

/* Same, complex double (conjugated dots: spmv_epilogue.hpp:31-34). Strides in complex elements. */
static void spmv_cplx(const or_sell* A, double* y, int64_t y_rs, int64_t y_cs, const double* x,
                      int64_t x_rs, int64_t x_cs, double* z, int64_t z_rs, int64_t z_cs, int32_t w,
                      uint32_t f, zdouble alpha, zdouble beta, zdouble gamma0, const double* gl,
                      zdouble delta, zdouble eta, double* dot, int workers) {
    const int32_t C = A->C;
    int64_t nb = or_worker_blocks(A->nchunks, workers, 0, NULL, NULL);
    const int64_t dotn = 3 * (int64_t)w;
    zdouble* partials = (zdouble*)calloc((size_t)(nb > 0 ? nb : 1) * dotn, sizeof(zdouble));
    zdouble* acc = (zdouble*)malloc((size_t)C * w * sizeof(zdouble));
    for (int64_t bi = 0; bi < nb; ++bi) {
        int64_t c0, c1;
        or_worker_blocks(A->nchunks, workers, bi, &c0, &c1);
        zdouble* dotp = partials + bi * dotn;
        for (int64_t c = c0; c < c1; ++c) {
            const int64_t off = A->chunk_offset[c];
            const int32_t len = A->chunk_len[c];
            for (int64_t q = 0; q < (int64_t)C * w; ++q) acc[q] = 0.0;
            for (int32_t j = 0; j < len; ++j) {
                for (int32_t r = 0; r < C; ++r) {
                    const int64_t slot = off + (int64_t)j * C + r;
                    const zdouble mv = zload(A->val + 2 * slot);
                    const double* xr = x + 2 * ((int64_t)A->col[slot] * x_rs);
                    zdouble* ar = acc + (int64_t)r * w;
                    for (int32_t v = 0; v < w; ++v) ar[v] += mv * zload(xr + 2 * (v * x_cs));
                }
            }
            for (int32_t r = 0; r < C; ++r) {
                const int64_t row = c * C + r;
                if (row >= A->nrows) continue;
                double* yr = y + 2 * (row * y_rs);
                const double* xr = x + 2 * (row * x_rs);
                for (int32_t v = 0; v < w; ++v) {
                    zdouble t = acc[(int64_t)r * w + v];
                    const zdouble xv = zload(xr + 2 * (v * x_cs));
                    if (f & F_SHIFT) t -= gamma0 * xv;
                    if (f & F_VSHIFT) t -= zload(gl + 2 * v) * xv;
                    t *= alpha;
                    if (f & F_AXPBY) t += beta * zload(yr + 2 * (v * y_cs));
                    zstore(yr + 2 * (v * y_cs), t);
                    if (f & F_CHAIN) {
                        double* zr = z + 2 * (row * z_rs);
                        zstore(zr + 2 * (v * z_cs), delta * zload(zr + 2 * (v * z_cs)) + eta * t);
                    }
                    if (f & F_DOT_YY) dotp[v] += conj(t) * t;
                    if (f & F_DOT_XY) dotp[w + v] += conj(xv) * t;
                    if (f & F_DOT_XX) dotp[2 * w + v] += conj(xv) * xv;
                }
            }
        }
    }
    for (int seg = 0; seg < 3; ++seg) {
        const uint32_t want = seg == 0 ? F_DOT_YY : seg == 1 ? F_DOT_XY : F_DOT_XX;
        if (!(f & want)) continue;
        for (int32_t v = 0; v < w; ++v) {
            zdouble s = 0.0;
            for (int64_t bi = 0; bi < nb; ++bi) s += partials[bi * dotn + seg * w + v];
            zstore(dot + 2 * (seg * w + v), s);
        }
    }
    free(acc);
    free(partials);
}

/* spmv.hpp:129-202 with opts_from capi.cpp:124-140 (NULL scalars -> alpha 1, others 0). */
void or_spmv(const or_sell* A, double* y, int64_t y_rs, int64_t y_cs, const double* x,
             int64_t x_rs, int64_t x_cs, double* z, int64_t z_rs, int64_t z_cs, int32_t width,
             uint32_t flags, const double* alpha, const double* beta, const double* gamma,
             const double* gamma_list, const double* delta, const double* eta, double* dot,
             int workers) {
    if (A->dt == 0) {
        spmv_real(A, y, y_rs, y_cs, x, x_rs, x_cs, z, z_rs, z_cs, width, flags,
                  alpha ? *alpha : 1.0, beta ? *beta : 0.0, gamma ? *gamma : 0.0, gamma_list,
                  delta ? *delta : 0.0, eta ? *eta : 0.0, dot, workers);
    } else {
        spmv_cplx(A, y, y_rs, y_cs, x, x_rs, x_cs, z, z_rs, z_cs, width, flags,
                  alpha ? zload(alpha) : 1.0, beta ? zload(beta) : 0.0,
                  gamma ? zload(gamma) : 0.0, gamma_list, delta ? zload(delta) : 0.0,
                  eta ? zload(eta) : 0.0, dot, workers);
    }
}

/* ------------------------------------------------------------------- tsm -- */

typedef struct {
    zdouble sum, comp;
} ksum;

/* CompensatedSum tsm.hpp:73-87 (Kahan-Babuska-Neumaier), complex-aware via abs. */
static void ksum_add(ksum* s, zdouble x) {
    const zdouble t = s->sum + x;
    if (cabs(s->sum) >= cabs(x))
        s->comp += (s->sum - t) + x;
    else
        s->comp += (x - t) + s->sum;
    s->sum = t;
}

typedef struct {
    double sum, comp;
} rsum;

static void rsum_add(rsum* s, double x) {
    const double t = s->sum + x;
    if (fabs(s->sum) >= fabs(x))
        s->comp += (s->sum - t) + x;
    else
        s->comp += (x - t) + s->sum;
    s->sum = t;
}

/* tsm.hpp:105-178.  The fixed (m,k) kernels (:37-49) and the generic loop
 * (:142-146) accumulate in the same order (rows ascending, then m, then k). */
void or_tsmttsm(int dt, int64_t n, int32_t m, int32_t k, double* x, int64_t x_rs, int64_t x_cs,
                const double* v, int64_t v_rs, const double* w, int64_t w_rs, const double* alpha,
                const double* beta, int kahan, int workers) {
    const int64_t nb = or_worker_blocks(n, workers, 0, NULL, NULL);
    const int64_t cells = (int64_t)m * k;
    if (dt == 0) {
        const double a = alpha ? *alpha : 1.0, b = beta ? *beta : 0.0;
        if (!kahan) {
            double* part = (double*)calloc((size_t)(nb ? nb : 1) * cells, sizeof(double));
            for (int64_t bi = 0; bi < nb; ++bi) {
                int64_t r0, r1;
                or_worker_blocks(n, workers, bi, &r0, &r1);
                double* acc = part + bi * cells;
                for (int64_t i = r0; i < r1; ++i)
                    for (int32_t mm = 0; mm < m; ++mm) {
                        const double vm = v[i * v_rs + mm];
                        for (int32_t kk = 0; kk < k; ++kk) acc[(int64_t)kk * m + mm] += vm * w[i * w_rs + kk];
                    }
            }
            for (int32_t kk = 0; kk < k; ++kk)
                for (int32_t mm = 0; mm < m; ++mm) {
                    double s = 0.0;
                    for (int64_t bi = 0; bi < nb; ++bi) s += part[bi * cells + (int64_t)kk * m + mm];
                    double* xo = x + mm * x_rs + kk * x_cs;
                    *xo = a * s + b * *xo;
                }
            free(part);
        } else {
            rsum* part = (rsum*)calloc((size_t)(nb ? nb : 1) * cells, sizeof(rsum));
            for (int64_t bi = 0; bi < nb; ++bi) {
                int64_t r0, r1;
                or_worker_blocks(n, workers, bi, &r0, &r1);
                rsum* acc = part + bi * cells;
                for (int64_t i = r0; i < r1; ++i)
                    for (int32_t mm = 0; mm < m; ++mm) {
                        const double vm = v[i * v_rs + mm];
                        for (int32_t kk = 0; kk < k; ++kk)
                            rsum_add(&acc[(int64_t)kk * m + mm], vm * w[i * w_rs + kk]);
                    }
            }
            for (int32_t kk = 0; kk < k; ++kk)
                for (int32_t mm = 0; mm < m; ++mm) {
                    rsum tot = {0.0, 0.0};
                    for (int64_t bi = 0; bi < nb; ++bi) {
                        rsum_add(&tot, part[bi * cells + (int64_t)kk * m + mm].sum);
                        rsum_add(&tot, part[bi * cells + (int64_t)kk * m + mm].comp);
                    }
                    double* xo = x + mm * x_rs + kk * x_cs;
                    *xo = a * (tot.sum + tot.comp) + b * *xo;
                }
            free(part);
        }
        return;
    }
    const zdouble a = alpha ? zload(alpha) : 1.0, b = beta ? zload(beta) : 0.0;
    ksum* part = (ksum*)calloc((size_t)(nb ? nb : 1) * cells, sizeof(ksum));
    for (int64_t bi = 0; bi < nb; ++bi) {
        int64_t r0, r1;
        or_worker_blocks(n, workers, bi, &r0, &r1);
        ksum* acc = part + bi * cells;
        for (int64_t i = r0; i < r1; ++i)
            for (int32_t mm = 0; mm < m; ++mm) {
                const zdouble vm = conj(zload(v + 2 * (i * v_rs + mm)));
                for (int32_t kk = 0; kk < k; ++kk) {
                    const zdouble p = vm * zload(w + 2 * (i * w_rs + kk));
                    if (kahan)
                        ksum_add(&acc[(int64_t)kk * m + mm], p);
                    else
                        acc[(int64_t)kk * m + mm].sum += p;
                }
            }
    }
    for (int32_t kk = 0; kk < k; ++kk)
        for (int32_t mm = 0; mm < m; ++mm) {
            zdouble s;
            if (kahan) {
                ksum tot = {0.0, 0.0};
                for (int64_t bi = 0; bi < nb; ++bi) {
                    ksum_add(&tot, part[bi * cells + (int64_t)kk * m + mm].sum);
                    ksum_add(&tot, part[bi * cells + (int64_t)kk * m + mm].comp);
                }
                s = tot.sum + tot.comp;
            } else {
                s = 0.0;
                for (int64_t bi = 0; bi < nb; ++bi) s += part[bi * cells + (int64_t)kk * m + mm].sum;
            }
            double* xo = x + 2 * (mm * x_rs + kk * x_cs);
            zstore(xo, a * s + b * zload(xo));
        }
    free(part);
}

/* tsm.hpp:182-225 (tsmm_fixed :51-68 has the same order: tmp over m, then alpha*tmp+beta*w). */
void or_tsmm(int dt, int64_t n, int32_t m, int32_t k, double* w, int64_t w_rs, const double* v,
             int64_t v_rs, const double* x, int64_t x_rs, int64_t x_cs, const double* alpha,
             const double* beta) {
    if (dt == 0) {
        const double a = alpha ? *alpha : 1.0, b = beta ? *beta : 0.0;
        double* tmp = (double*)malloc((size_t)k * sizeof(double));
        for (int64_t i = 0; i < n; ++i) {
            for (int32_t kk = 0; kk < k; ++kk) tmp[kk] = 0.0;
            for (int32_t mm = 0; mm < m; ++mm) {
                const double vm = v[i * v_rs + mm];
                for (int32_t kk = 0; kk < k; ++kk) tmp[kk] += vm * x[mm * x_rs + kk * x_cs];
            }
            for (int32_t kk = 0; kk < k; ++kk) w[i * w_rs + kk] = a * tmp[kk] + b * w[i * w_rs + kk];
        }
        free(tmp);
        return;
    }
    const zdouble a = alpha ? zload(alpha) : 1.0, b = beta ? zload(beta) : 0.0;
    zdouble* tmp = (zdouble*)malloc((size_t)k * sizeof(zdouble));
    for (int64_t i = 0; i < n; ++i) {
        for (int32_t kk = 0; kk < k; ++kk) tmp[kk] = 0.0;
        for (int32_t mm = 0; mm < m; ++mm) {
            const zdouble vm = zload(v + 2 * (i * v_rs + mm));
            for (int32_t kk = 0; kk < k; ++kk) tmp[kk] += vm * zload(x + 2 * (mm * x_rs + kk * x_cs));
        }
        for (int32_t kk = 0; kk < k; ++kk) {
            double* wo = w + 2 * (i * w_rs + kk);
            zstore(wo, a * tmp[kk] + b * zload(wo));
        }
    }
    free(tmp);
}

/* tsm.hpp:230-249: per row, s = sum_mm v[mm]*x[mm,kk] (mm ascending), then alpha*s + beta*v. */
void or_tsmm_inplace(int dt, int64_t n, int32_t m, double* v, int64_t v_rs, const double* x,
                     int64_t x_rs, int64_t x_cs, const double* alpha, const double* beta) {
    if (dt == 0) {
        const double a = alpha ? *alpha : 1.0, b = beta ? *beta : 0.0;
        double* tmp = (double*)malloc((size_t)m * sizeof(double));
        for (int64_t i = 0; i < n; ++i) {
            for (int32_t kk = 0; kk < m; ++kk) {
                double s = 0.0;
                for (int32_t mm = 0; mm < m; ++mm) s += v[i * v_rs + mm] * x[mm * x_rs + kk * x_cs];
                tmp[kk] = s;
            }
            for (int32_t kk = 0; kk < m; ++kk) v[i * v_rs + kk] = a * tmp[kk] + b * v[i * v_rs + kk];
        }
        free(tmp);
        return;
    }
    const zdouble a = alpha ? zload(alpha) : 1.0, b = beta ? zload(beta) : 0.0;
    zdouble* tmp = (zdouble*)malloc((size_t)m * sizeof(zdouble));
    for (int64_t i = 0; i < n; ++i) {
        for (int32_t kk = 0; kk < m; ++kk) {
            zdouble s = 0.0;
            for (int32_t mm = 0; mm < m; ++mm)
                s += zload(v + 2 * (i * v_rs + mm)) * zload(x + 2 * (mm * x_rs + kk * x_cs));
            tmp[kk] = s;
        }
        for (int32_t kk = 0; kk < m; ++kk) {
            double* vo = v + 2 * (i * v_rs + kk);
            zstore(vo, a * tmp[kk] + b * zload(vo));
        }
    }
    free(tmp);
}

/* densemat.hpp:276-292 */
void or_dot(int dt, int64_t n, int32_t w, const double* a, int64_t a_rs, int64_t a_cs,
            const double* b, int64_t b_rs, int64_t b_cs, double* out, int workers) {
    const int64_t nb = or_worker_blocks(n, workers, 0, NULL, NULL);
    if (dt == 0) {
        double* part = (double*)calloc((size_t)(nb ? nb : 1) * w, sizeof(double));
        for (int64_t bi = 0; bi < nb; ++bi) {
            int64_t r0, r1;
            or_worker_blocks(n, workers, bi, &r0, &r1);
            for (int64_t i = r0; i < r1; ++i)
                for (int32_t j = 0; j < w; ++j) part[bi * w + j] += a[i * a_rs + j * a_cs] * b[i * b_rs + j * b_cs];
        }
        for (int32_t j = 0; j < w; ++j) out[j] = 0.0;
        for (int64_t bi = 0; bi < nb; ++bi)
            for (int32_t j = 0; j < w; ++j) out[j] += part[bi * w + j];
        free(part);
        return;
    }
    zdouble* part = (zdouble*)calloc((size_t)(nb ? nb : 1) * w, sizeof(zdouble));
    for (int64_t bi = 0; bi < nb; ++bi) {
        int64_t r0, r1;
        or_worker_blocks(n, workers, bi, &r0, &r1);
        for (int64_t i = r0; i < r1; ++i)
            for (int32_t j = 0; j < w; ++j)
                part[bi * w + j] += conj(zload(a + 2 * (i * a_rs + j * a_cs))) * zload(b + 2 * (i * b_rs + j * b_cs));
    }
    for (int32_t j = 0; j < w; ++j) {
        zdouble s = 0.0;
        for (int64_t bi = 0; bi < nb; ++bi) s += part[bi * w + j];
        zstore(out + 2 * j, s);
    }
    free(part);
}

/* ------------------------------------------------------------- partition -- */

/* partition.hpp:45-94 */
int or_partition(int64_t n, const int32_t* rowlens, const double* weights, int k, int by_nnz,
                 int64_t* row_offset) {
    if (n <= 0 || k < 1 || (int64_t)k > n) return 1;
    double total_w = 0.0;
    for (int i = 0; i < k; ++i) {
        if (!(weights[i] > 0.0)) return 1;
        total_w += weights[i];
    }
    int64_t* prefix = NULL;
    int64_t total_nnz = 0;
    if (by_nnz) {
        if (!rowlens) return 1;
        prefix = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
        for (int64_t r = 0; r < n; ++r) prefix[r + 1] = prefix[r] + rowlens[r];
        total_nnz = prefix[n];
    }
    row_offset[0] = 0;
    row_offset[k] = n;
    double cum = 0.0;
    for (int i = 1; i < k; ++i) {
        cum += weights[i - 1];
        const double share = cum / total_w;
        int64_t b;
        if (!by_nnz || total_nnz == 0) {
            b = (int64_t)floor((double)n * share + 0.5);
        } else {
            const double target = (double)total_nnz * share;
            int64_t p = 0;
            while (p < n && (double)prefix[p] < target) ++p;
            if (p > 0 && fabs((double)prefix[p - 1] - target) <= fabs((double)prefix[p] - target))
                b = p - 1;
            else
                b = p;
        }
        if (b < row_offset[i - 1] + 1) b = row_offset[i - 1] + 1;
        if (b > n - (k - i)) b = n - (k - i);
        row_offset[i] = b;
    }
    free(prefix);
    return 0;
}
