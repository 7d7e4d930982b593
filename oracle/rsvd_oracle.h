/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the randomized k-SVD path.
 *
 * A plain-C restatement of the reference algorithm
 * (/root/reference/proj/src/{rng,matrix,gemm,qr,svd,rsvd}.cpp) used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER.
 * Nothing in paper_2110_03423_b200/ links, loads or calls it.
 *
 * Parity pin: tests/test_oracle.py checks every function here bit-for-bit
 * against the reference library itself (oracle/_ref/libranddsvd_ref.so, built
 * by oracle/Makefile from the reference sources) and against the committed
 * golden vectors in tests/golden/ (made by tests/golden/make_golden.py).
 *
 * All matrices are row-major doubles, like randsvd::DenseMatrix
 * (include/randsvd/matrix.hpp:12-31). Status codes follow rsvd_b200.h:
 * 0 ok, 1 ArgumentError, 2 DimensionError, 3 ConvergenceError.
 */
#ifndef RSVD_ORACLE_H
#define RSVD_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_ARGUMENT = 1, ORC_DIMENSION = 2, ORC_CONVERGENCE = 3, ORC_NOMEM = 9 };

/* SplitMix64 counter stream + Box-Muller (rng.cpp:9-51). */
void orc_splitmix_words(uint64_t seed, uint64_t first_counter, size_t count, uint64_t* out);
void orc_uniforms(uint64_t seed, uint64_t first_counter, size_t count, double* out);
void orc_gaussian_matrix(uint64_t seed, size_t rows, size_t cols, double* out);

/* Pairwise reductions (matrix.cpp:17-38, 100-102). */
double orc_pairwise_sum(const double* x, size_t n);
double orc_pairwise_dot(const double* x, const double* y, size_t n);
double orc_frobenius_norm(const double* a, size_t count);

/* gemm.cpp:48-100: out = alpha * op(a) * op(b) + beta * c (c may be NULL when beta == 0). */
int orc_gemm(double alpha, const double* a, size_t ar, size_t ac, int ta, const double* b,
             size_t br, size_t bc, int tb, double beta, const double* c, double* out);

/* qr.cpp:27-102: thin Householder QR, q m x n, r n x n upper with diag >= 0. */
int orc_householder_qr(const double* a, size_t m, size_t n, double* q, double* r);

/* svd.cpp:153-273: compact SVD; u m x p, sigma p, v n x p, p = min(m, n). */
int orc_dense_svd(const double* a, size_t m, size_t n, double* u, double* sigma, double* v);

/* svd.cpp:275-297 */
int orc_extend_orthonormal(const double* u, size_t m, size_t r0, size_t target, double* out);

/* rsvd.cpp:28-35 */
size_t orc_sketch_width(size_t k, size_t oversample, double epsilon, int epsilon_mode, size_t m,
                        size_t n);

/* Step functions (rsvd.cpp:51-109). Outputs are caller-allocated at the maximal size;
 * range_basis writes the kept width to *cols_out. */
int orc_sketch(const double* a, size_t m, size_t n, size_t s, uint64_t seed, double* y0);
int orc_power_iterate(const double* a, size_t m, size_t n, const double* y0, size_t s, size_t q,
                      double* w);
int orc_range_basis(const double* y, size_t m, size_t s, double* q, size_t* cols_out);
int orc_project_and_solve(const double* a, size_t m, size_t n, const double* qb, size_t sq,
                          size_t k, double* u, double* sigma, double* v, size_t* sketch_width);

/* Full pipeline (rsvd.cpp:150-174). u m x k, sigma k, v n x k. values_only => u/v unused. */
int orc_randomized_ksvd(const double* a, size_t m, size_t n, size_t k, size_t oversample,
                        size_t power_q, uint64_t seed, double epsilon, int epsilon_mode,
                        int values_only, double* u, double* sigma, double* v,
                        size_t* sketch_width);

/* rsvd.cpp:37-49 */
double orc_residual_fro(const double* a, size_t m, size_t n, const double* u, const double* sigma,
                        const double* v, size_t k);

/* Last error message (thread-local). */
const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
