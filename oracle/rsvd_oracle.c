/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference randomized k-SVD.
 *
 * This is the checker for the B200 path, never the thing measured or shipped:
 * only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
 * reference legs) load it. Every function cites the reference file:line it
 * restates (paths relative to /root/reference/proj). It keeps the reference's
 * per-element evaluation order (and so, compiled with the same FMA contraction
 * as the reference, its exact bits); tests/test_oracle.py pins that against
 * the reference library and the golden vectors in tests/golden/.
 *
 * Build: oracle/Makefile (gcc -O3 -march=x86-64-v3 -std=gnu11, shared library).
 */
#define _GNU_SOURCE
#include "rsvd_oracle.h"

#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* orc_last_error(void) { return g_err; }

static inline size_t nz(size_t n) { return n ? n : 1; }
#define XMALLOC(T, n) ((T*)malloc(sizeof(T) * nz(n)))

/* ---------------------------------------------------------------- rng.cpp:9-51 */

static const uint64_t kGolden = 0x9E3779B97F4A7C15ULL; /* rng.cpp:11 */

static inline uint64_t mix64(uint64_t z) { /* rng.cpp:13-20 */
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

/* The counter is pre-incremented, so the first word uses counter 1 (rng.cpp:24-27). */
static inline uint64_t word_at(uint64_t seed, uint64_t counter) {
    return mix64(seed + counter * kGolden);
}

static inline double uniform_from_word(uint64_t w) { /* rng.cpp:29-32, (0, 1] */
    return (double)((w >> 11) + 1) * 0x1.0p-53;
}

void orc_splitmix_words(uint64_t seed, uint64_t first_counter, size_t count, uint64_t* out) {
    for (size_t i = 0; i < count; ++i) out[i] = word_at(seed, first_counter + i);
}

void orc_uniforms(uint64_t seed, uint64_t first_counter, size_t count, double* out) {
    for (size_t i = 0; i < count; ++i) out[i] = uniform_from_word(word_at(seed, first_counter + i));
}

/* Box-Muller with the sine half cached (rng.cpp:34-46); element i of the row-major fill
 * (rng.cpp:48-53) is normal #i of a fresh sampler. */
void orc_gaussian_matrix(uint64_t seed, size_t rows, size_t cols, double* out) {
    const size_t total = rows * cols;
    uint64_t counter = 0;
    for (size_t i = 0; i < total; i += 2) {
        const double u1 = uniform_from_word(word_at(seed, ++counter));
        const double u2 = uniform_from_word(word_at(seed, ++counter));
        const double radius = sqrt(-2.0 * log(u1));
        const double angle = 2.0 * M_PI * u2;
        out[i] = radius * cos(angle);
        if (i + 1 < total) out[i + 1] = radius * sin(angle);
    }
}

/* ---------------------------------------------------------- matrix.cpp:17-102 */

__attribute__((noinline)) static double pairwise_sum_impl(const double* x, size_t n) {
    if (n <= 64) {
        double acc = 0.0;
        for (size_t i = 0; i < n; ++i) acc += x[i];
        return acc;
    }
    const size_t half = n / 2;
    return pairwise_sum_impl(x, half) + pairwise_sum_impl(x + half, n - half);
}

__attribute__((noinline)) static double pairwise_dot_impl(const double* x, const double* y, size_t n) {
    if (n <= 64) {
        double acc = 0.0;
        for (size_t i = 0; i < n; ++i) acc += x[i] * y[i];
        return acc;
    }
    const size_t half = n / 2;
    return pairwise_dot_impl(x, y, half) + pairwise_dot_impl(x + half, y + half, n - half);
}

double orc_pairwise_sum(const double* x, size_t n) { return pairwise_sum_impl(x, n); }
double orc_pairwise_dot(const double* x, const double* y, size_t n) {
    return pairwise_dot_impl(x, y, n);
}
double orc_frobenius_norm(const double* a, size_t count) {
    return sqrt(pairwise_dot_impl(a, a, count));
}

static void transpose(const double* a, size_t r, size_t c, double* t) { /* matrix.cpp:66-71 */
    for (size_t i = 0; i < r; ++i)
        for (size_t j = 0; j < c; ++j) t[j * r + i] = a[i * c + j];
}

static int all_finite(const double* a, size_t count) { /* matrix.cpp:83-87 */
    for (size_t i = 0; i < count; ++i)
        if (!isfinite(a[i])) return 0;
    return 1;
}

/* ---------------------------------------------------------------- gemm.cpp:24-100 */

/* Per output element the k index runs in ascending order, c += (alpha*a_ik)*b_kj
 * (gemm.cpp:32-40); the 64-blocking only changes locality, not that order. */
static void kernel_rows(double* cdat, const double* adat, const double* bdat, size_t m, size_t k,
                        size_t n, double alpha) {
    for (size_t i0 = 0; i0 < m; i0 += 64) {
        const size_t i1 = i0 + 64 < m ? i0 + 64 : m;
        for (size_t k0 = 0; k0 < k; k0 += 64) {
            const size_t k1 = k0 + 64 < k ? k0 + 64 : k;
            for (size_t i = i0; i < i1; ++i) {
                double* crow = cdat + i * n;
                const double* arow = adat + i * k;
                for (size_t kk = k0; kk < k1; ++kk) {
                    const double aik = alpha * arow[kk];
                    const double* brow = bdat + kk * n;
                    for (size_t j = 0; j < n; ++j) crow[j] += aik * brow[j];
                }
            }
        }
    }
}

int orc_gemm(double alpha, const double* a, size_t ar, size_t ac, int ta, const double* b,
             size_t br, size_t bc, int tb, double beta, const double* c, double* out) {
    const size_t m = ta ? ac : ar;
    const size_t inner_a = ta ? ar : ac;
    const size_t inner_b = tb ? bc : br;
    const size_t n = tb ? br : bc;
    if (inner_a != inner_b)
        return fail(ORC_DIMENSION, "gemm inner dimensions disagree: %zu vs %zu", inner_a, inner_b);
    for (size_t i = 0; i < m * n; ++i) out[i] = 0.0;
    if (beta != 0.0)
        for (size_t i = 0; i < m * n; ++i) out[i] = beta * c[i];
    double* at = NULL;
    double* bt = NULL;
    const double* ap = a;
    const double* bp = b;
    if (ta) {
        at = XMALLOC(double, ar * ac);
        if (!at) return fail(ORC_NOMEM, "out of memory");
        transpose(a, ar, ac, at);
        ap = at;
    }
    if (tb) {
        bt = XMALLOC(double, br * bc);
        if (!bt) {
            free(at);
            return fail(ORC_NOMEM, "out of memory");
        }
        transpose(b, br, bc, bt);
        bp = bt;
    }
    kernel_rows(out, ap, bp, m, inner_a, n, alpha);
    free(at);
    free(bt);
    return ORC_OK;
}

/* ----------------------------------------------------------------- qr.cpp:27-102 */

int orc_householder_qr(const double* a, size_t m, size_t n, double* qout, double* rout) {
    if (m < n)
        return fail(ORC_DIMENSION, "householder_qr needs rows >= cols, got %zux%zu", m, n);
    double* w = XMALLOC(double, m * n);
    double* refl = (double*)calloc(nz(m * n), sizeof(double));
    char* active = (char*)calloc(nz(n), 1);
    double* q = (double*)calloc(nz(m * n), sizeof(double));
    if (!w || !refl || !active || !q) {
        free(w); free(refl); free(active); free(q);
        return fail(ORC_NOMEM, "out of memory");
    }
    for (size_t i = 0; i < m; ++i) /* column-major working copy, qr.cpp:36-38 */
        for (size_t j = 0; j < n; ++j) w[j * m + i] = a[i * n + j];

    for (size_t k = 0; k < n; ++k) { /* qr.cpp:44-68 */
        double* col = w + k * m;
        const size_t len = m - k;
        const double norm_x = sqrt(pairwise_dot_impl(col + k, col + k, len));
        if (norm_x == 0.0) continue;
        double* v = refl + k * m + k;
        for (size_t i = 0; i < len; ++i) v[i] = col[k + i];
        const double sign = col[k] >= 0.0 ? 1.0 : -1.0;
        v[0] += sign * norm_x;
        const double norm_v = sqrt(pairwise_dot_impl(v, v, len));
        for (size_t i = 0; i < len; ++i) v[i] /= norm_v;
        active[k] = 1;
        col[k] = -sign * norm_x;
        for (size_t t = 0; t + k + 1 < n; ++t) {
            double* cj = w + (k + 1 + t) * m + k;
            const double d = 2.0 * pairwise_dot_impl(v, cj, len);
            for (size_t i = 0; i < len; ++i) cj[i] -= d * v[i];
        }
    }
    for (size_t j = 0; j < n; ++j) q[j * m + j] = 1.0; /* backward accumulation, qr.cpp:71-84 */
    for (size_t kk = n; kk-- > 0;) {
        if (!active[kk]) continue;
        const double* v = refl + kk * m + kk;
        const size_t len = m - kk;
        for (size_t t = 0; t + kk < n; ++t) {
            double* cj = q + (kk + t) * m + kk;
            const double d = 2.0 * pairwise_dot_impl(v, cj, len);
            for (size_t i = 0; i < len; ++i) cj[i] -= d * v[i];
        }
    }
    for (size_t k = 0; k < n; ++k) { /* diag(R) >= 0, qr.cpp:86-93 */
        if (w[k * m + k] < 0.0) {
            for (size_t j = k; j < n; ++j) w[j * m + k] = -w[j * m + k];
            double* qc = q + k * m;
            for (size_t i = 0; i < m; ++i) qc[i] = -qc[i];
        }
    }
    if (qout)
        for (size_t i = 0; i < m; ++i)
            for (size_t j = 0; j < n; ++j) qout[i * n + j] = q[j * m + i];
    if (rout)
        for (size_t i = 0; i < n; ++i)
            for (size_t j = 0; j < n; ++j) rout[i * n + j] = j >= i ? w[j * m + i] : 0.0;
    free(w); free(refl); free(active); free(q);
    return ORC_OK;
}

/* ---------------------------------------------------------------- svd.cpp:35-297 */

static const double kAbsGramTol = 1e-14; /* svd.cpp:35 */
static const double kRelGramTol = 1e-13; /* svd.cpp:36 */
enum { kPairBlock = 32, kSvdMaxSweeps = 30 }; /* svd.cpp:37, svd.hpp:20 */

/* Stable sort of an index permutation by key, descending (desc=1) or ascending. */
static void stable_argsort(const double* key, size_t n, size_t* perm, int desc) {
    /* insertion sort is stable; n is small (sketch widths) in every caller that is hot, and
     * row_load sorts (fill_null_columns) use merge sort below when n is large */
    for (size_t i = 0; i < n; ++i) perm[i] = i;
    if (n < 2) return;
    size_t* tmp = XMALLOC(size_t, n);
    for (size_t width = 1; width < n; width *= 2) { /* bottom-up merge sort: stable */
        for (size_t lo = 0; lo < n; lo += 2 * width) {
            size_t mid = lo + width < n ? lo + width : n;
            size_t hi = lo + 2 * width < n ? lo + 2 * width : n;
            size_t i = lo, j = mid, o = lo;
            while (i < mid && j < hi) {
                const int take_right = desc ? (key[perm[j]] > key[perm[i]])
                                            : (key[perm[j]] < key[perm[i]]);
                tmp[o++] = take_right ? perm[j++] : perm[i++];
            }
            while (i < mid) tmp[o++] = perm[i++];
            while (j < hi) tmp[o++] = perm[j++];
        }
        memcpy(perm, tmp, n * sizeof(size_t));
    }
    free(tmp);
}

static void permute_cols(double* src, double* scratch, size_t m, const size_t* perm, size_t n) {
    for (size_t j = 0; j < n; ++j) memcpy(scratch + j * m, src + perm[j] * m, m * sizeof(double));
    memcpy(src, scratch, m * n * sizeof(double));
}

typedef struct {
    double* w;
    double* v;
    double* colsq;
    size_t m, n;
    double abs_thresh;
    size_t rotations;
} PairSweep;

static void sweep_visit(PairSweep* s, size_t i, size_t j) { /* svd.cpp:60-90 */
    const size_t m = s->m, n = s->n;
    double* wi = s->w + i * m;
    double* wj = s->w + j * m;
    const double d = pairwise_dot_impl(wi, wj, m);
    const double ad = fabs(d);
    if (ad <= s->abs_thresh && d * d <= kRelGramTol * kRelGramTol * s->colsq[i] * s->colsq[j])
        return;
    const double zeta = (s->colsq[j] - s->colsq[i]) / (2.0 * d);
    const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
    const double c = 1.0 / sqrt(1.0 + t * t);
    const double sn = c * t;
    for (size_t r = 0; r < m; ++r) {
        const double a = wi[r], b = wj[r];
        wi[r] = c * a - sn * b;
        wj[r] = sn * a + c * b;
    }
    double* vi = s->v + i * n;
    double* vj = s->v + j * n;
    for (size_t r = 0; r < n; ++r) {
        const double a = vi[r], b = vj[r];
        vi[r] = c * a - sn * b;
        vj[r] = sn * a + c * b;
    }
    s->colsq[i] -= t * d;
    s->colsq[j] += t * d;
    ++s->rotations;
}

static void sweep_run(PairSweep* s) { /* svd.cpp:93-106 */
    const size_t n = s->n;
    s->rotations = 0;
    for (size_t bi = 0; bi < n; bi += kPairBlock) {
        const size_t bi_end = bi + kPairBlock < n ? bi + kPairBlock : n;
        for (size_t i = bi; i < bi_end; ++i)
            for (size_t j = i + 1; j < bi_end; ++j) sweep_visit(s, i, j);
        for (size_t bj = bi_end; bj < n; bj += kPairBlock) {
            const size_t bj_end = bj + kPairBlock < n ? bj + kPairBlock : n;
            for (size_t i = bi; i < bi_end; ++i)
                for (size_t j = bj; j < bj_end; ++j) sweep_visit(s, i, j);
        }
    }
}

/* svd.cpp:111-151. u col-major m x width; valid holds nvalid column ids (capacity width). */
static int fill_null_columns(double* u, size_t m, size_t* valid, size_t nvalid, const size_t* nulls,
                             size_t nnulls) {
    double* row_load = XMALLOC(double, m);
    size_t* order = XMALLOC(size_t, m);
    double* cand = XMALLOC(double, m);
    int rc = ORC_OK;
    for (size_t si = 0; si < nnulls && rc == ORC_OK; ++si) {
        const size_t slot = nulls[si];
        for (size_t r = 0; r < m; ++r) row_load[r] = 0.0;
        for (size_t ci = 0; ci < nvalid; ++ci) {
            const double* col = u + valid[ci] * m;
            for (size_t r = 0; r < m; ++r) row_load[r] += col[r] * col[r];
        }
        stable_argsort(row_load, m, order, 0);
        int placed = 0;
        for (size_t oi = 0; oi < m; ++oi) {
            const size_t t = order[oi];
            for (size_t r = 0; r < m; ++r) cand[r] = 0.0;
            cand[t] = 1.0;
            for (int pass = 0; pass < 2; ++pass) {
                for (size_t ci = 0; ci < nvalid; ++ci) {
                    const double* col = u + valid[ci] * m;
                    const double d = pairwise_dot_impl(cand, col, m);
                    for (size_t r = 0; r < m; ++r) cand[r] -= d * col[r];
                }
            }
            const double nrm = sqrt(pairwise_dot_impl(cand, cand, m));
            if (nrm >= 1e-4) {
                double* dst = u + slot * m;
                for (size_t r = 0; r < m; ++r) dst[r] = cand[r] / nrm;
                valid[nvalid++] = slot;
                placed = 1;
                break;
            }
        }
        if (!placed) rc = fail(ORC_CONVERGENCE, "dense_svd could not complete an orthonormal basis");
    }
    free(row_load); free(order); free(cand);
    return rc;
}

/* svd.cpp:153-263; a is m x n row-major with m >= n; u m x n, sigma n, v n x n. */
static int jacobi_svd_tall(const double* a, size_t m, size_t n, double* uout, double* sigma,
                           double* vout) {
    double* w = XMALLOC(double, m * n);
    double* v = (double*)calloc(n * n, sizeof(double));
    double* colsq = XMALLOC(double, n);
    double* reordered = XMALLOC(double, n);
    double* scratch = XMALLOC(double, (m > n ? m : n) * n);
    size_t* perm = XMALLOC(size_t, n);
    size_t* valid = XMALLOC(size_t, n);
    size_t* nulls = (size_t*)calloc(nz(n), sizeof(size_t));  /* zeroed: silences -Wmaybe-uninitialized */
    int rc = ORC_OK;
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) w[j * m + i] = a[i * n + j];
    for (size_t j = 0; j < n; ++j) v[j * n + j] = 1.0;
    for (size_t j = 0; j < n; ++j) colsq[j] = pairwise_dot_impl(w + j * m, w + j * m, m);
    const double total = pairwise_sum_impl(colsq, n);
    PairSweep sw = {w, v, colsq, m, n, kAbsGramTol * total, 0};
    int converged = 0, sweeps = 0;
    while (sweeps < kSvdMaxSweeps) { /* svd.cpp:178-200 */
        ++sweeps;
        for (size_t j = 0; j < n; ++j) colsq[j] = pairwise_dot_impl(w + j * m, w + j * m, m);
        stable_argsort(colsq, n, perm, 1);
        permute_cols(w, scratch, m, perm, n);
        permute_cols(v, scratch, n, perm, n);
        for (size_t j = 0; j < n; ++j) reordered[j] = colsq[perm[j]];
        memcpy(colsq, reordered, n * sizeof(double));
        sweep_run(&sw);
        if (sw.rotations == 0) {
            converged = 1;
            break;
        }
    }
    if (!converged) {
        rc = fail(ORC_CONVERGENCE, "one-sided Jacobi SVD did not converge within %d sweeps",
                  kSvdMaxSweeps);
        goto done;
    }
    for (size_t j = 0; j < n; ++j) sigma[j] = sqrt(pairwise_dot_impl(w + j * m, w + j * m, m));
    stable_argsort(sigma, n, perm, 1); /* svd.cpp:210-219 */
    permute_cols(w, scratch, m, perm, n);
    permute_cols(v, scratch, n, perm, n);
    for (size_t j = 0; j < n; ++j) reordered[j] = sigma[perm[j]];
    memcpy(sigma, reordered, n * sizeof(double));
    {
        const double sigma_max = n ? sigma[0] : 0.0; /* svd.cpp:221-234 */
        const double null_thresh = sigma_max * (double)(m > n ? m : n) * DBL_EPSILON;
        size_t nvalid = 0, nnull = 0;
        for (size_t j = 0; j < n; ++j) {
            if (sigma[j] > null_thresh) {
                double* col = w + j * m;
                for (size_t r = 0; r < m; ++r) col[r] /= sigma[j];
                valid[nvalid++] = j;
            } else {
                nulls[nnull++] = j;
            }
        }
        rc = fill_null_columns(w, m, valid, nvalid, nulls, nnull);
        if (rc != ORC_OK) goto done;
    }
    for (size_t j = 0; j < n; ++j) { /* sign convention, svd.cpp:237-254 */
        double* uc = w + j * m;
        size_t arg = 0;
        double best = fabs(uc[0]);
        for (size_t r = 1; r < m; ++r) {
            if (fabs(uc[r]) > best) {
                best = fabs(uc[r]);
                arg = r;
            }
        }
        if (uc[arg] < 0.0) {
            for (size_t r = 0; r < m; ++r) uc[r] = -uc[r];
            double* vc = v + j * n;
            for (size_t r = 0; r < n; ++r) vc[r] = -vc[r];
        }
    }
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) uout[i * n + j] = w[j * m + i];
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < n; ++j) vout[i * n + j] = v[j * n + i];
done:
    free(w); free(v); free(colsq); free(reordered); free(scratch); free(perm); free(valid);
    free(nulls);
    return rc;
}

int orc_dense_svd(const double* a, size_t m, size_t n, double* u, double* sigma, double* v) {
    if (!all_finite(a, m * n)) return fail(ORC_ARGUMENT, "dense_svd input contains NaN or Inf");
    if (m >= n) return jacobi_svd_tall(a, m, n, u, sigma, v);
    double* at = XMALLOC(double, m * n); /* wide: factor the transpose, swap roles (svd.cpp:267-273) */
    transpose(a, m, n, at);
    const int rc = jacobi_svd_tall(at, n, m, v, sigma, u);
    free(at);
    return rc;
}

int orc_extend_orthonormal(const double* u, size_t m, size_t r0, size_t target, double* out) {
    if (target < r0 || target > m)
        return fail(ORC_DIMENSION, "extend_orthonormal from %zu to %zu columns of height %zu", r0,
                    target, m);
    double* cols = (double*)calloc(m * target, sizeof(double));
    size_t* valid = XMALLOC(size_t, target);
    size_t* nulls = XMALLOC(size_t, target);
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < r0; ++j) cols[j * m + i] = u[i * r0 + j];
    for (size_t j = 0; j < r0; ++j) valid[j] = j;
    for (size_t j = r0; j < target; ++j) nulls[j - r0] = j;
    const int rc = fill_null_columns(cols, m, valid, r0, nulls, target - r0);
    if (rc == ORC_OK)
        for (size_t i = 0; i < m; ++i)
            for (size_t j = 0; j < target; ++j) out[i * target + j] = cols[j * m + i];
    free(cols); free(valid); free(nulls);
    return rc;
}

/* ---------------------------------------------------------------- rsvd.cpp:28-174 */

size_t orc_sketch_width(size_t k, size_t oversample, double epsilon, int epsilon_mode, size_t m,
                        size_t n) {
    const size_t cap = m < n ? m : n;
    if (epsilon_mode) {
        const double raw = ceil((double)k / epsilon);
        const size_t w = (size_t)raw;
        return w < cap ? w : cap;
    }
    return k + oversample < cap ? k + oversample : cap;
}

int orc_sketch(const double* a, size_t m, size_t n, size_t s, uint64_t seed, double* y0) {
    const size_t md = m < n ? m : n; /* rsvd.cpp:51-59 */
    if (s < 1 || s > md)
        return fail(ORC_ARGUMENT, "sketch width %zu outside [1, %zu] for a %zux%zu input", s, md, m,
                    n);
    double* omega = XMALLOC(double, n * s);
    orc_gaussian_matrix(seed, n, s, omega);
    const int rc = orc_gemm(1.0, a, m, n, 0, omega, n, s, 0, 0.0, NULL, y0);
    free(omega);
    return rc;
}

int orc_power_iterate(const double* a, size_t m, size_t n, const double* y0, size_t s, size_t q,
                      double* wout) { /* rsvd.cpp:61-73 */
    if (q == 0) return orc_householder_qr(y0, m, s, wout, NULL);
    double* w = XMALLOC(double, m * s);
    double* z = XMALLOC(double, n * s);
    double* tmp = XMALLOC(double, (m > n ? m : n) * s);
    int rc = ORC_OK;
    memcpy(w, y0, m * s * sizeof(double));
    for (size_t round = 0; round < q && rc == ORC_OK; ++round) {
        rc = orc_gemm(1.0, a, m, n, 1, w, m, s, 0, 0.0, NULL, tmp);
        if (rc == ORC_OK) rc = orc_householder_qr(tmp, n, s, z, NULL);
        if (rc == ORC_OK) rc = orc_gemm(1.0, a, m, n, 0, z, n, s, 0, 0.0, NULL, tmp);
        if (rc == ORC_OK) rc = orc_householder_qr(tmp, m, s, w, NULL);
    }
    if (rc == ORC_OK) memcpy(wout, w, m * s * sizeof(double));
    free(w); free(z); free(tmp);
    return rc;
}

int orc_range_basis(const double* y, size_t m, size_t s, double* qout, size_t* cols_out) {
    double* q = XMALLOC(double, m * s); /* rsvd.cpp:75-87 */
    double* r = XMALLOC(double, s * s);
    size_t* keep = XMALLOC(size_t, s);
    int rc = orc_householder_qr(y, m, s, q, r);
    if (rc == ORC_OK) {
        const double drop = 1e-13 * orc_frobenius_norm(y, m * s);
        size_t nk = 0;
        for (size_t j = 0; j < s; ++j)
            if (fabs(r[j * s + j]) > drop) keep[nk++] = j;
        if (nk == s) {
            memcpy(qout, q, m * s * sizeof(double));
        } else {
            if (nk == 0) keep[nk++] = 0;
            for (size_t i = 0; i < m; ++i)
                for (size_t j = 0; j < nk; ++j) qout[i * nk + j] = q[i * s + keep[j]];
        }
        *cols_out = nk;
    }
    free(q); free(r); free(keep);
    return rc;
}

int orc_project_and_solve(const double* a, size_t m, size_t n, const double* qb, size_t sq,
                          size_t k, double* u, double* sigma, double* v, size_t* sketch_width) {
    if (k < 1 || k > sq) /* rsvd.cpp:89-109 */
        return fail(ORC_ARGUMENT, "rank k=%zu exceeds the basis width %zu", k, sq);
    double* b = XMALLOC(double, sq * n);
    const size_t p = sq < n ? sq : n;
    double* ub = XMALLOC(double, sq * p);
    double* sb = XMALLOC(double, p);
    double* vb = XMALLOC(double, n * p);
    double* ubk = XMALLOC(double, sq * k);
    int rc = orc_gemm(1.0, qb, m, sq, 1, a, m, n, 0, 0.0, NULL, b);
    if (rc == ORC_OK) rc = orc_dense_svd(b, sq, n, ub, sb, vb);
    if (rc == ORC_OK) {
        const size_t avail = k < p ? k : p;
        for (size_t i = 0; i < avail; ++i) sigma[i] = sb[i];
        for (size_t i = 0; i < sq; ++i)
            for (size_t j = 0; j < avail; ++j) ubk[i * avail + j] = ub[i * p + j];
        if (u) rc = orc_gemm(1.0, qb, m, sq, 0, ubk, sq, avail, 0, 0.0, NULL, u);
        if (v)
            for (size_t i = 0; i < n; ++i)
                for (size_t j = 0; j < avail; ++j) v[i * avail + j] = vb[i * p + j];
        *sketch_width = sq;
    }
    free(b); free(ub); free(sb); free(vb); free(ubk);
    return rc;
}

/* solve_tall + pad_to_rank (rsvd.cpp:117-134); a is tall m x n. */
static int solve_tall(const double* a, size_t m, size_t n, size_t k, size_t oversample,
                      size_t power_q, uint64_t seed, double epsilon, int epsilon_mode,
                      int values_only, double* u, double* sigma, double* v, size_t* sketch_width) {
    const size_t s = orc_sketch_width(k, oversample, epsilon, epsilon_mode, m, n);
    double* y0 = XMALLOC(double, m * s);
    double* w = XMALLOC(double, m * s);
    double* qb = XMALLOC(double, m * s);
    int rc = orc_sketch(a, m, n, s, seed, y0);
    if (rc == ORC_OK) rc = orc_power_iterate(a, m, n, y0, s, power_q, w);
    size_t sq = 0;
    if (rc == ORC_OK) rc = orc_range_basis(w, m, s, qb, &sq);
    if (rc == ORC_OK) {
        const size_t k_eff = k < sq ? k : sq;
        double* ue = values_only ? NULL : XMALLOC(double, m * k_eff);
        double* ve = values_only ? NULL : XMALLOC(double, n * k_eff);
        size_t sw = 0;
        rc = orc_project_and_solve(a, m, n, qb, sq, k_eff, ue, sigma, ve, &sw);
        if (rc == ORC_OK) {
            for (size_t i = k_eff; i < k; ++i) sigma[i] = 0.0;
            if (!values_only) {
                if (k_eff < k) {
                    rc = orc_extend_orthonormal(ue, m, k_eff, k, u);
                    if (rc == ORC_OK) rc = orc_extend_orthonormal(ve, n, k_eff, k, v);
                } else {
                    memcpy(u, ue, m * k * sizeof(double));
                    memcpy(v, ve, n * k * sizeof(double));
                }
            }
            *sketch_width = sw;
        }
        free(ue); free(ve);
    }
    free(y0); free(w); free(qb);
    return rc;
}

int orc_randomized_ksvd(const double* a, size_t m, size_t n, size_t k, size_t oversample,
                        size_t power_q, uint64_t seed, double epsilon, int epsilon_mode,
                        int values_only, double* u, double* sigma, double* v,
                        size_t* sketch_width) {
    const size_t md = m < n ? m : n; /* validate, rsvd.cpp:136-146 */
    if (k < 1 || k > md)
        return fail(ORC_ARGUMENT, "target rank k=%zu outside [1, %zu] for a %zux%zu input", k, md,
                    m, n);
    if (!(epsilon > 0.0 && epsilon < 1.0)) return fail(ORC_ARGUMENT, "epsilon must lie in (0, 1)");
    if (!all_finite(a, m * n))
        return fail(ORC_ARGUMENT, "randomized_ksvd input contains NaN or Inf");
    size_t sw = 0;
    if (m >= n) {
        const int rc = solve_tall(a, m, n, k, oversample, power_q, seed, epsilon, epsilon_mode,
                                  values_only, u, sigma, v, &sw);
        if (sketch_width) *sketch_width = sw;
        return rc;
    }
    double* at = XMALLOC(double, m * n); /* wide: transpose, swap U/V (rsvd.cpp:150-156) */
    if (!at) return fail(ORC_NOMEM, "out of memory");
    transpose(a, m, n, at);
    const int rc = solve_tall(at, n, m, k, oversample, power_q, seed, epsilon, epsilon_mode,
                              values_only, v, sigma, u, &sw);
    free(at);
    if (sketch_width) *sketch_width = sw;
    return rc;
}

double orc_residual_fro(const double* a, size_t m, size_t n, const double* u, const double* sigma,
                        const double* v, size_t k) {
    double* us = XMALLOC(double, m * k); /* rsvd.cpp:37-49 */
    double* out = XMALLOC(double, m * n);
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < k; ++j) us[i * k + j] = u[i * k + j] * sigma[j];
    orc_gemm(-1.0, us, m, k, 0, v, n, k, 1, 1.0, a, out);
    const double r = orc_frobenius_norm(out, m * n);
    free(us); free(out);
    return r;
}
