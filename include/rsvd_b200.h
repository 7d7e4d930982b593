/* rsvd_b200.h — C-ABI of the B200-native randomized truncated SVD.
 *
 * This is the drop-in boundary for the reference's hot path
 *   randsvd::randomized_ksvd(const DenseMatrix&, const RsvdConfig&)
 *       (/root/reference/proj/include/randsvd/rsvd.hpp:58, src/rsvd.cpp:150-156)
 *   randsvd::singular_values_only(const DenseMatrix&, const RsvdConfig&)
 *       (rsvd.hpp:62-63, rsvd.cpp:158-174)
 * and the step functions its tests drive (rsvd.hpp:36-53). Plain pointers and
 * sizes only: every matrix is row-major FP64 exactly like randsvd::DenseMatrix
 * (matrix.hpp:12-31, element (i, j) at data[i * cols + j]) unless a leading
 * dimension is given. The C++ drop-in (include/randsvd/rsvd.hpp) and the Python
 * host mirror (paper_2110_03423_b200/rsvd.py) are thin layers over this file.
 *
 * Errors: every entry point returns an rsvd_b200_status. The reference's
 * exception types map 1:1 — ArgumentError, DimensionError, ConvergenceError
 * (errors.hpp:16-37) — plus CUDA/NCCL/allocation failures. The message of the
 * last failure on the calling thread is rsvd_b200_last_error().
 *
 * Threading: a handle owns one CUDA stream and its workspace; one solve at a
 * time per handle, independent handles are independent (cf. SPEC "safe
 * concurrent independent solves").
 */
#ifndef RSVD_B200_H
#define RSVD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RSVD_B200_OK = 0,
    RSVD_B200_ARGUMENT_ERROR = 1,    /* randsvd::ArgumentError    */
    RSVD_B200_DIMENSION_ERROR = 2,   /* randsvd::DimensionError   */
    RSVD_B200_CONVERGENCE_ERROR = 3, /* randsvd::ConvergenceError */
    RSVD_B200_CUDA_ERROR = 4,
    RSVD_B200_NCCL_ERROR = 5,
    RSVD_B200_ALLOC_ERROR = 6
} rsvd_b200_status;

/* Mirrors randsvd::RsvdConfig (rsvd.hpp:13-23) field for field. */
typedef struct {
    size_t k;          /* target rank, >= 1                         */
    size_t oversample; /* p, reference default 10                   */
    size_t power_q;    /* q, reference default 2                    */
    uint64_t seed;     /* reference default 0                       */
    double epsilon;    /* must lie in (0, 1); reference default 0.5 */
    int epsilon_mode;  /* sketch width ceil(k / epsilon)            */
} rsvd_b200_config;

/* Fills the reference defaults (k = 1, p = 10, q = 2, seed 0, eps 0.5, off). */
void rsvd_b200_config_default(rsvd_b200_config* cfg);

/* RsvdConfig::sketch_width (rsvd.cpp:28-35). */
size_t rsvd_b200_sketch_width(const rsvd_b200_config* cfg, size_t m, size_t n);

typedef struct rsvd_b200_handle rsvd_b200_handle;

/* Create a solver bound to CUDA device `device` (its own stream and workspace). */
rsvd_b200_status rsvd_b200_create(int device, rsvd_b200_handle** out);
rsvd_b200_status rsvd_b200_destroy(rsvd_b200_handle* h);
const char* rsvd_b200_last_error(void);
/* The handle's CUDA stream (a cudaStream_t) so callers can order work around it. */
void* rsvd_b200_stream(rsvd_b200_handle* h);
/* Order the handle's stream after all work already enqueued on `other` (a cudaStream_t,
 * e.g. the framework stream that produced a device A). The _device entry points read
 * their inputs on the handle's (non-blocking) stream. */
rsvd_b200_status rsvd_b200_wait_stream(rsvd_b200_handle* h, void* other);

/* Validation mode: use the caller's Omega (n x s row-major, host memory) for the
 * next solves instead of the on-device generator, making the sketch bit-identical
 * to the reference's (rng.cpp's glibc log/sin/cos can differ from the device's in
 * the last bit). Pass NULL to return to the device generator. */
rsvd_b200_status rsvd_b200_set_omega(rsvd_b200_handle* h, const double* omega_host, size_t rows,
                                     size_t cols);

/* ---------------------------------------------------------------------------
 * The drop-in entry points, host buffers (H2D/D2H inside the call):
 *   a      m x n input (borrowed)
 *   u      m x k, sigma k, v n x k outputs (caller allocated); sketch_width may be NULL.
 * Wide inputs (m < n) are solved on the transpose with U/V swapped back, exactly
 * as rsvd.cpp:150-156 does.
 * ------------------------------------------------------------------------- */
rsvd_b200_status rsvd_b200_randomized_ksvd(rsvd_b200_handle* h, const double* a, size_t m,
                                           size_t n, const rsvd_b200_config* cfg, double* u,
                                           double* sigma, double* v, size_t* sketch_width);

/* sigma (k) only; bit-identical to randomized_ksvd's sigma under the same config. */
rsvd_b200_status rsvd_b200_singular_values_only(rsvd_b200_handle* h, const double* a, size_t m,
                                                size_t n, const rsvd_b200_config* cfg,
                                                double* sigma);

/* Same solve with every buffer already in device memory (A resident in HBM):
 * a_dev with leading dimension lda (>= n, lda*8 a multiple of 16 bytes, 16-byte
 * aligned base), u_dev (m x k) / v_dev (n x k) may be NULL for values-only.
 * Work is enqueued on the handle's stream; the call returns after the solve
 * completes (status flags are checked on the host). */
rsvd_b200_status rsvd_b200_randomized_ksvd_device(rsvd_b200_handle* h, const double* a_dev,
                                                  size_t m, size_t n, size_t lda,
                                                  const rsvd_b200_config* cfg, double* u_dev,
                                                  double* sigma_dev, double* v_dev,
                                                  size_t* sketch_width);

/* ---------------------------------------------------------------------------
 * FP32 input (BASELINE config C4). Same solve for an FP32 A: every product with an
 * m-dimension runs on the 5th-generation tensor cores (tcgen05.mma kind::tf32) as
 * 3xTF32 split products (FP32-class accuracy), the (k+p)-sized side in FP64; outputs
 * are FP64. Tolerance bar (BASELINE.json): sigma 1e-4 relative, angles 1e-3. No
 * reference counterpart (the reference is FP64-only); rsvd.hpp:58 semantics otherwise.
 * Device A: lda a multiple of 4 floats and 16-byte aligned base (else copied).
 * ------------------------------------------------------------------------- */
rsvd_b200_status rsvd_b200_randomized_ksvd_f32(rsvd_b200_handle* h, const float* a, size_t m,
                                               size_t n, const rsvd_b200_config* cfg, double* u,
                                               double* sigma, double* v, size_t* sketch_width);
rsvd_b200_status rsvd_b200_randomized_ksvd_f32_device(rsvd_b200_handle* h, const float* a_dev,
                                                      size_t m, size_t n, size_t lda,
                                                      const rsvd_b200_config* cfg, double* u_dev,
                                                      double* sigma_dev, double* v_dev,
                                                      size_t* sketch_width);

/* ---------------------------------------------------------------------------
 * Row-sharded solves across GPUs (no reference counterpart: the reference is one
 * host process; this is §8e's data-parallel split of the same
 * randomized_ksvd, rsvd.hpp:58). Rank g holds a contiguous row block A_g of the
 * m_total x n input (m_total >= n); every rank calls the solve collectively with the
 * same n, m_total and config. Only sums over rows cross ranks (the s x s Gram of each
 * CholeskyQR pass, the n x s partials of A^T Q and Q^T A, the TSQR R stack of the
 * Householder fallback, the status flags), as in-place FP64 sum all-reduces on the
 * handle's stream. sigma and V are returned replicated, U sharded like A
 * (m_local x k). Results agree with the single-device solve to rounding.
 * ------------------------------------------------------------------------- */
/* 128-byte NCCL unique id, created on rank 0 and distributed out of band. */
rsvd_b200_status rsvd_b200_nccl_unique_id(unsigned char* id128);
/* Attach an NCCL communicator (the process's libnccl.so.2) to the handle's device. */
rsvd_b200_status rsvd_b200_comm_init_nccl(rsvd_b200_handle* h, const unsigned char* id128,
                                          int rank, int world);
/* In-process group of handles (one host thread per rank; buffers on one device or
 * P2P-reachable devices): reductions are fixed-order device sums. For testing the
 * sharded pipeline on one GPU. */
typedef struct rsvd_b200_local_group rsvd_b200_local_group;
rsvd_b200_status rsvd_b200_local_group_create(int world, rsvd_b200_local_group** out);
void rsvd_b200_local_group_destroy(rsvd_b200_local_group* g);
rsvd_b200_status rsvd_b200_comm_init_local(rsvd_b200_handle* h, rsvd_b200_local_group* g,
                                           int rank);
/* rank / world of the attached communicator (0 / 1 without one). */
rsvd_b200_status rsvd_b200_comm_info(rsvd_b200_handle* h, int* rank, int* world);
/* Detach and destroy the handle's communicator. */
void rsvd_b200_comm_free(rsvd_b200_handle* h);
/* Host buffers: a (m_local x n) in, u (m_local x k), sigma (k), v (n x k) out. */
rsvd_b200_status rsvd_b200_randomized_ksvd_sharded(rsvd_b200_handle* h, const double* a,
                                                   size_t m_local, size_t m_total, size_t n,
                                                   const rsvd_b200_config* cfg, double* u,
                                                   double* sigma, double* v,
                                                   size_t* sketch_width);
/* Device buffers (A shard resident in HBM, same layout rules as the _device solve). */
rsvd_b200_status rsvd_b200_randomized_ksvd_sharded_device(
    rsvd_b200_handle* h, const double* a_dev, size_t m_local, size_t m_total, size_t n,
    size_t lda, const rsvd_b200_config* cfg, double* u_dev, double* sigma_dev, double* v_dev,
    size_t* sketch_width);

/* FP32 row-sharded solves (host / device buffers). */
rsvd_b200_status rsvd_b200_randomized_ksvd_sharded_f32(rsvd_b200_handle* h, const float* a,
                                                       size_t m_local, size_t m_total, size_t n,
                                                       const rsvd_b200_config* cfg, double* u,
                                                       double* sigma, double* v,
                                                       size_t* sketch_width);
rsvd_b200_status rsvd_b200_randomized_ksvd_sharded_f32_device(
    rsvd_b200_handle* h, const float* a_dev, size_t m_local, size_t m_total, size_t n,
    size_t lda, const rsvd_b200_config* cfg, double* u_dev, double* sigma_dev, double* v_dev,
    size_t* sketch_width);

/* ---------------------------------------------------------------------------
 * RsvdResult::residual_fro (rsvd.hpp:31-32, rsvd.cpp:37-49): ||a - u diag(sigma) v^T||_F
 * for a m x n, u m x k, v n x k (row-major FP64), sigma k. On the device the product is
 * never formed: a fused GEMM epilogue subtracts it chunk by chunk and reduces the squares
 * in a fixed order (deterministic).
 * ------------------------------------------------------------------------- */
rsvd_b200_status rsvd_b200_residual_fro(rsvd_b200_handle* h, const double* a, size_t m, size_t n,
                                       const double* u, const double* sigma, const double* v,
                                       size_t k, double* out);
rsvd_b200_status rsvd_b200_residual_fro_device(rsvd_b200_handle* h, const double* a_dev,
                                              size_t m, size_t n, size_t lda,
                                              const double* u_dev, const double* sigma_dev,
                                              const double* v_dev, size_t k, double* out);

/* ---------------------------------------------------------------------------
 * PCA, the paper's CelebA application (randsvd::pca, pca.hpp:13-28, pca.cpp:10-52):
 * fit_pca centers the N x d samples-as-rows x on the device (column sums by the atx GEMM,
 * then X - 1 mean^T), runs the randomized k-SVD of the centered data and returns
 * mean (d), components = V (d x k, row-major) and explained_variance = sigma^2 / (N - 1).
 * Errors as the reference: N < 2 or k outside [1, min(N, d)] -> ArgumentError.
 * transform: out (N x k) = (x - mean) components (DimensionError on a feature mismatch).
 * ------------------------------------------------------------------------- */
rsvd_b200_status rsvd_b200_fit_pca(rsvd_b200_handle* h, const double* x, size_t N, size_t d,
                                   size_t k, const rsvd_b200_config* cfg, double* mean,
                                   double* components, double* explained_variance);
rsvd_b200_status rsvd_b200_pca_transform(rsvd_b200_handle* h, const double* x, size_t N,
                                         size_t d, const double* mean, const double* components,
                                         size_t k, double* out);

/* ---------------------------------------------------------------------------
 * DMAT files (the reference's interchange format, dmat.hpp:10-19) straight into HBM:
 * rows [row0, row0 + nrows) of the file (a rank's shard) stream through two pinned
 * staging buffers into a_dev (lda >= cols doubles), file reads overlapping the copies.
 * Return 0, or 7 (randsvd::IoError: bad magic / header / truncation, with the byte offset
 * in rsvd_b200_dmat_last_error()).
 * ------------------------------------------------------------------------- */
int rsvd_b200_dmat_shape(const char* path, uint64_t* rows, uint64_t* cols);
int rsvd_b200_load_dmat_device(rsvd_b200_handle* h, const char* path, uint64_t row0,
                               uint64_t nrows, double* a_dev, size_t lda);
const char* rsvd_b200_dmat_last_error(void);

/* ---------------------------------------------------------------------------
 * Step functions (rsvd.hpp:36-53), host buffers, for the reference's step-level
 * tests.  range_basis writes the kept width to *cols_out (q must hold m x s).
 * ------------------------------------------------------------------------- */
rsvd_b200_status rsvd_b200_gaussian_matrix(rsvd_b200_handle* h, uint64_t seed, size_t rows,
                                           size_t cols, double* out);
rsvd_b200_status rsvd_b200_sketch(rsvd_b200_handle* h, const double* a, size_t m, size_t n,
                                  size_t s, uint64_t seed, double* y0);
/* The same from a sampler part-way through its stream (GaussianSampler state,
 * rng.hpp:21-42): `counter` words already drawn, and, if has_cached, the cached sine half
 * `cached` that the sampler's next normal() returns first (rng.cpp:35-38). A fresh sampler
 * is (0, 0, 0.0). The reference's sketch/gaussian_matrix continue a sampler this way
 * (rng.cpp:48-53); after drawing N normals the caller advances its sampler state. */
rsvd_b200_status rsvd_b200_gaussian_stream(rsvd_b200_handle* h, uint64_t seed, uint64_t counter,
                                           int has_cached, double cached, size_t rows,
                                           size_t cols, double* out);
rsvd_b200_status rsvd_b200_sketch_stream(rsvd_b200_handle* h, const double* a, size_t m,
                                         size_t n, size_t s, uint64_t seed, uint64_t counter,
                                         int has_cached, double cached, double* y0);
rsvd_b200_status rsvd_b200_power_iterate(rsvd_b200_handle* h, const double* a, size_t m, size_t n,
                                         const double* y0, size_t s, size_t q, double* w);
/* Householder thin QR (replaces randsvd::householder_qr, qr.hpp:16 / qr.cpp:27-102):
 * a m x n row-major (m >= n) -> q m x n with orthonormal columns and r n x n
 * upper triangular with a non-negative diagonal (strictly-lower entries exact zeros).
 * The blocked (compact WY) Householder kernel of the CholeskyQR2 fallback. m < n is
 * RSVD_B200_DIMENSION_ERROR (the reference's DimensionError). The _device variant takes
 * device pointers with leading dimensions and is stream-ordered (rsvd_b200_stream). */
rsvd_b200_status rsvd_b200_householder_qr(rsvd_b200_handle* h, const double* a, size_t m,
                                          size_t n, double* q, double* r);
rsvd_b200_status rsvd_b200_householder_qr_device(rsvd_b200_handle* h, const double* a, size_t lda,
                                                 size_t m, size_t n, double* q, size_t ldq,
                                                 double* r, size_t ldr);
/* Test-matrix generator (replaces randsvd::synth::synth_matrix, synth.cpp:58-71, for the
 * paper's §4 grids): A = U diag(sigma) V^T, rows x cols (rows >= cols), U the Householder Q
 * of a rows x cols draw of GaussianSampler(seed), V that of the next cols x cols draw,
 * sigma_j = spectrum_value(kind, j + 1) with kind 0 = fast (1/i^2), 1 = sharp
 * (1e-4 + 1/(1 + e^(i+1-beta)), beta > 0), 2 = slow (1/i^0.1). out row-major (host), or
 * device memory with leading dimension ld (_device; returns after the copy completes). */
rsvd_b200_status rsvd_b200_synth_matrix(rsvd_b200_handle* h, size_t rows, size_t cols, int kind,
                                        double beta, uint64_t seed, double* out);
rsvd_b200_status rsvd_b200_synth_matrix_device(rsvd_b200_handle* h, size_t rows, size_t cols,
                                               int kind, double beta, uint64_t seed, double* out,
                                               size_t ld);
rsvd_b200_status rsvd_b200_range_basis(rsvd_b200_handle* h, const double* y, size_t m, size_t s,
                                       double* q, size_t* cols_out);
rsvd_b200_status rsvd_b200_project_and_solve(rsvd_b200_handle* h, const double* a, size_t m,
                                             size_t n, const double* qb, size_t sq, size_t k,
                                             double* u, double* sigma, double* v,
                                             size_t* sketch_width);

/* ---------------------------------------------------------------------------
 * Raw sampler stream on the device (rng.cpp:22-32), for bit-exactness tests:
 * words / uniforms for counters first_counter .. first_counter + count - 1.
 * ------------------------------------------------------------------------- */
rsvd_b200_status rsvd_b200_splitmix_words(rsvd_b200_handle* h, uint64_t seed,
                                          uint64_t first_counter, size_t count, uint64_t* out);
rsvd_b200_status rsvd_b200_uniforms(rsvd_b200_handle* h, uint64_t seed, uint64_t first_counter,
                                    size_t count, double* out);

/* ---------------------------------------------------------------------------
 * Instrumentation: per-stage device times (ms) of the last solve on this handle,
 * measured with CUDA events on the handle's stream, and the dominant GEMM's
 * launch count/total ms.  names[i] are static strings.  Returns the count.
 * ------------------------------------------------------------------------- */
int rsvd_b200_last_profile(rsvd_b200_handle* h, const char** names, double* ms, int max);
/* Event timing level: 0 off (default), 1 per-stage events, 2 additionally one event
 * pair around every launch of the passes over A (tag "gemm_A"). Adds event records only. */
void rsvd_b200_set_profiling(rsvd_b200_handle* h, int level);
/* Accumulated per-launch stats for a tag since the last reset: launches, summed device
 * ms (CUDA events on the handle's stream) and summed algorithmic flops (2*m*n*s per pass).
 * Returns 1 if the tag was seen. */
int rsvd_b200_kernel_stats(rsvd_b200_handle* h, const char* tag, long* count, double* total_ms,
                           double* total_flops);
void rsvd_b200_reset_stats(rsvd_b200_handle* h);
/* Number of kernels launched by the last solve. */
long rsvd_b200_last_launch_count(rsvd_b200_handle* h);

/* Diagnostics of the last solve: "jacobi_sweeps", "householder_fallbacks",
 * "robust_reruns" (optimistic pipeline repeated on the robust path), "launches"; and,
 * cumulative over the handle, "graph_launches" (device-resident solves that ran as one
 * launch of the handle's cached CUDA graph of the pipeline; RSVD_B200_NO_GRAPH disables it),
 * "upload_aty_splits" (host-buffer solves: split count of the first power iteration's A^T Y0
 * produced during the chunked upload, 0 if that pass ran after it), "oz_passes" (passes over A
 * of the last solve that ran as INT8-emulated FP64 products) and "oz_stored_passes" (of those,
 * the ones that read A's digit planes converted once per solve).
 * Returns -1 for an unknown key. */
long rsvd_b200_last_info(rsvd_b200_handle* h, const char* key);
/* Force the robust path (host-checked Cholesky, Householder fallback) for every solve. */
void rsvd_b200_set_robust(rsvd_b200_handle* h, int on);
/* Enable (default) or disable the CUDA-graph replay of repeated device-resident solves. */
void rsvd_b200_set_graphs(rsvd_b200_handle* h, int on);

/* Measured FP64 tensor-core peak of the handle's GPU (TFLOP/s): an issue-bound
 * mma.sync m16n8k16 f64 loop on every SM — the roofline denominator of the GEMMs. */
rsvd_b200_status rsvd_b200_dmma_peak(rsvd_b200_handle* h, double* tflops);
/* Measured INT8 tensor-core peak (TOPS; tcgen05 kind::i8 M 128 N 256 K 32 issue loop on every
 * SM): the roofline denominator of the INT8-emulated FP64 passes over A. */
rsvd_b200_status rsvd_b200_imma_peak(rsvd_b200_handle* h, double* tops);

/* Test hook for the FP32-input 3xTF32 tcgen05 GEMM (device pointers; see csrc/kernels.h
 * GemmTf32): mn = 0: out = A (M x K) * Bt^T, Bt NP x K; mn = 1: out = A^T W, A K x M,
 * W K x NP. out FP64 (out64) or FP32, row-major or transposed (out_t); splits > 1 = split-K
 * with a fixed-order reduce (FP64 only). Synchronous. */
rsvd_b200_status rsvd_b200_debug_gemm_tf32(rsvd_b200_handle* h, int mn, const float* A, long M,
                                          long K, long lda, const float* B, long ldb, int NP,
                                          void* out, long ldo, int out64, int out_t, int splits);

/* Test hook for the INT8-emulated FP64 GEMM (Ozaki scheme, csrc/gemm_oz.cu; device pointers):
 * mn = 0: out (M x NP) = A (M x K) * B^T with B = Xt (NP x K, ldb; rows >= cols zero);
 * mn = 1: out = A^T W, A (K x M), W = B (K x NP, ldb; columns >= cols zero), out Z (M x NP) or
 * Z^T (NP x M) with out_t; splits > 1 = split-K with a fixed-order reduce. NP a multiple of 16,
 * <= 256. Scales (row / column maxima) and digits are computed in the call. Synchronous. */
rsvd_b200_status rsvd_b200_debug_gemm_oz(rsvd_b200_handle* h, int mn, const double* A, long M,
                                        long K, long lda, const double* B, long ldb, int NP,
                                        int cols, double* out, long ldo, int out_t, int splits);

/* The same with A converted once to stored row-scaled digit planes (the GEMM reads digits,
 * A^T W takes A's row scales through W). */
rsvd_b200_status rsvd_b200_debug_gemm_ozd(rsvd_b200_handle* h, int mn, const double* A, long M,
                                         long K, long lda, const double* B, long ldb, int NP,
                                         int cols, double* out, long ldo, int out_t, int splits);

/* Test hook for the single-CTA Cholesky kernel (device pointers, row-major NP x NP buffers):
 * G (s x s SPD block of an NP x NP buffer) -> R (upper, zero padded) and Rinv^T; *status = 0
 * or 1 (a pivot below tol * max_i G_ii). s up to the shared-memory width limit. Synchronous. */
rsvd_b200_status rsvd_b200_debug_cholesky(rsvd_b200_handle* h, const double* G, int s, int NP,
                                         double* R, double* RinvT, double tol, int* status);

/* Test hook for the one-sided Jacobi SVD kernels (single CTA up to s = 112, multi-CTA block
 * Jacobi beyond): R (s x s block of an NP x NP row-major device buffer) = U diag(sigma) W^T with
 * sigma descending (NP entries, zero padded), U and W NP x NP row-major (columns = vectors).
 * *sweeps = sweeps used, or -1 if 30 sweeps did not converge. Synchronous. */
rsvd_b200_status rsvd_b200_debug_jacobi(rsvd_b200_handle* h, const double* R, int s, int NP,
                                       double* sigma, double* U, double* W, int* sweeps);

/* Library build identification (sm_100a). */
const char* rsvd_b200_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RSVD_B200_H */
