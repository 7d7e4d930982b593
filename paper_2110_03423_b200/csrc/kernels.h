// Internal (C++) launch interface of the sm_100a kernels. Not part of the C-ABI:
// include/rsvd_b200.h is the public boundary; rsvd_b200.cpp orchestrates these.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rsvdb200 {

// Y = A * X.  A: M x K row-major (lda), Xt: NP x K row-major (ldx) holding X^T,
// Y: M x NP row-major (ldy).  splits > 1 writes split slab s at Y + s*split_stride.
// flag != nullptr additionally ORs 1 into *flag if any element of A is NaN/Inf.
struct GemmAx {
    const double* A;
    long M, K, lda;
    const double* Xt;
    long ldx;
    int NP;
    double* Y;
    long ldy;
    int splits = 1;
    long split_stride = 0;
    int* flag = nullptr;
    // Fused Gram epilogue (NP <= 96, splits == 1): per-CTA partials Y_tile^T Y_tile,
    // NP x NP each, at gram + blockIdx * NP * NP (ceil(M / 128) partials).
    double* gram = nullptr;
    // Fused residual (NP == 96, splits == 1): Y is not stored; resid_out[cta] =
    // sum over the CTA's rows < M, columns < resid_cols of (resid[r][c] - Y[r][c])^2.
    const double* resid = nullptr;
    long resid_ld = 0;
    int resid_cols = 0;
    double* resid_out = nullptr;
    // > 0: rows >= cols of Xt are zero (a sketch of width cols < NP). NP <= 96 then runs the
    // last cols % 8 (<= 4) columns as DFMA instead of a padded DMMA tile; output columns
    // >= cols come out zero as before.
    int cols = 0;
    // != nullptr and set on entry: return without touching the output (an optimistic
    // pipeline that already aborted on a Cholesky breakdown skips its remaining passes)
    const int* abort = nullptr;
};

// Z = A^T * W.  A: K x N row-major (lda), W: K x NP row-major (ldw).
// out_transposed: Z^T stored NP x N (ldz) else Z stored N x NP (ldz).
struct GemmAtx {
    const double* A;
    long K, N, lda;
    const double* W;
    long ldw;
    int NP;
    double* Z;
    long ldz;
    bool out_transposed = true;
    int splits = 1;
    long split_stride = 0;
    // (out_transposed, splits == 1) start from the Z^T already in Z instead of zero: a K
    // range processed by consecutive launches accumulates exactly like one launch
    bool accumulate = false;
    const int* abort = nullptr;  // as GemmAx::abort
    // > 0: W's columns >= cols are zero (the sketch width s of an A-pass); when the last
    // MMA column tile would hold at most 2 of them they run as DFMA (gemm_atx_kernel TAIL)
    int cols = 0;
};

// FP32-input 3xTF32 tensor-core GEMM (tcgen05, gemm_tf32.cu), D = op(A) * B (M x NP):
//   mn = false (ax):  A M x K row-major (lda), B given as Bt NP x K row-major (ldb);
//   mn = true  (atx): A K x M row-major (lda) read in place, B = W K x NP row-major (ldb).
// out: FP64 (out64) or FP32, row-major M x NP (ldo) or transposed NP x M (out_t); split-K
// writes slab s at out + s*split_stride (FP64 only). NP multiple of 16, <= 288.
// flag != nullptr ORs 1 into *flag if A holds a NaN/Inf. Blo (required): B's lo parts
// x - trunc_tf32(x), same shape and ldb as B. out_lo (FP32 row-major outputs only): also
// write the output's lo parts there (same ldo), ready to be the B operand of a later product.
struct GemmTf32 {
    const float* A;
    long M, K, lda;
    const float* B;
    long ldb;
    int NP;
    void* out;
    long ldo;
    const float* Blo = nullptr;
    void* out_lo = nullptr;
    bool mn = false, out64 = true, out_t = false;
    int splits = 1;
    long split_stride = 0;
    int* flag = nullptr;
    // mn with A == B (a Gram X^T X): compute only the column tiles at or right of each
    // 128-row tile's diagonal block; everything left of it is written as zero (the upper
    // triangle, all a Cholesky reads, is exact)
    bool upper = false;
    // > 0: split K into runs of this many 16-row k-tiles (the split count follows), so a row
    // range of a larger split-K product reproduces that product's slabs exactly
    int k_per_split = 0;
    const int* abort = nullptr;  // as GemmAx::abort
};
cudaError_t launch_gemm_tf32(const GemmTf32& p, cudaStream_t st);
// out (rows x cols, FP32, ldo) = in (FP64, ldi) for r < rows_valid and c < cols_valid, else 0.
// lo (optional): also the TF32 lo parts of out, same ldo.
cudaError_t launch_cvt_f64_f32(const double* in, long ldi, long rows, long cols, long rows_valid,
                               long cols_valid, float* out, long ldo, cudaStream_t st,
                               float* lo = nullptr);
// lo = x - trunc_tf32(x) elementwise (rows x cols, same ld).
cudaError_t launch_split_lo(const float* in, long rows, long cols, long ld, float* lo,
                            cudaStream_t st);
cudaError_t launch_cvt_f32_f64(const float* in, long ldi, long rows, long cols, double* out,
                               long ldo, cudaStream_t st);
cudaError_t launch_transpose_f32(const float* in, long rows, long cols, long ldi, float* out,
                                 long ldo, cudaStream_t st);

// FP64 GEMM on the INT8 tensor cores (Ozaki scheme, gemm_oz.cu). A (FP64) is split into 7
// balanced base-256 digits at a per-row (ax) / per-column (atx) scale inside the kernel; the
// small operand comes as digit planes bdig[7][NP][ldb] (K contiguous, ldb = oz_ldb(K) bytes)
// with per-column scales b_ef[NP] (launch_oz_digits_rows / _cols). a_ef / b_ef hold biased
// FP64 exponents of the row / column maxima (launch_oz_scan).
//   mn = false (ax):  out (M x NP, ldo) = A (M x K, lda) X,  a_ef[M] per row of A.
//   mn = true  (atx): out = A^T W, A (K x M, lda); out_t: Z^T (NP x M, ldo) else Z (M x NP);
//                     a_ef[M] per column of A; split-K slabs at out + s * split_stride.
// K per split <= kOzMaxKTiles * 32 (int32 accumulator headroom of a digit group: 7 products of
// balanced digits, |.| <= 2^14 each, per k). Measured: unsigned two's-complement A digits would
// save the bias add and XOR (2.6 -> 2.3 ms per C2 pass) but make the dropped low-order products
// biased (3x the Frobenius error), so the digits stay balanced.
constexpr int kOzMaxKTiles = 512;
struct GemmOz {
    bool mn = false;
    const double* A = nullptr;
    long M = 0, K = 0, lda = 0;
    const int* a_ef = nullptr;
    const uint8_t* bdig = nullptr;
    long ldb = 0;
    const int* b_ef = nullptr;
    int NP = 0;
    double* out = nullptr;
    long ldo = 0;
    bool out_t = false;
    int splits = 1;
    long split_stride = 0;
    const int* abort = nullptr;
};
cudaError_t launch_gemm_oz(const GemmOz& p, cudaStream_t st);
long oz_ldb(long K);
size_t oz_digits_bytes(int NP, long K);
void oz_chunks(int NP, int* nch, int* nfirst);
// Row / column maxima (biased exponents) of A (rows x cols, lda) and the NaN/Inf flag; `part`
// holds oz_scan_part_ints(rows, cols) ints of scratch.
// col_acc: max the column maxima into col_ef (row chunks of one A scanned as they arrive).
cudaError_t launch_oz_scan(const double* A, long rows, long cols, long lda, int* row_ef,
                           int* col_ef, int* part, int* flag, cudaStream_t st,
                           bool col_acc = false);
size_t oz_scan_part_ints(long rows, long cols);
// Digit planes of the rows of Xt (NP x K, ldx; rows >= cols zero), one scale per row.
// nfirst = 0: plain layout [plane][row][k] (gemm_oz); > 0: the stored-digit GEMM's tiled layout
// for column chunks of nfirst (oz_chunks).
cudaError_t launch_oz_digits_rows(const double* Xt, long ldx, int NP, int cols, long K,
                                  uint8_t* dig, int* b_ef, cudaStream_t st, int nfirst = 0);
// Digit planes of the columns of W (K x NP, ldw; columns >= cols zero), one scale per column;
// colmax: NP ints of scratch. row_ef (optional): digitise W' = diag(2^(row_ef[k] - 1076)) W,
// which carries A's row scales into the stored-digit atx GEMM. nfirst as above.
cudaError_t launch_oz_digits_cols(const double* W, long ldw, int NP, int cols, long K,
                                  uint8_t* dig, int* b_ef, int* colmax, cudaStream_t st,
                                  const int* row_ef = nullptr, int nfirst = 0);

// Stored digits: rows [r0, r1) of A (rows x cols <= 16384, lda) -> A's 7 row-scaled digit
// planes, written pre-tiled for both stored-digit GEMM shapes (dig_ax, dig_atx: each
// oz_tiled_bytes(rows, cols)), row_ef, NaN/Inf flag. One read of A; r0, r1 multiples of 128
// except r1 = rows (the last chunk, which also zeroes the padding).
size_t oz_tiled_bytes(long rows, long cols);
// the same digit layouts from a scan's row exponents (row_ef input), coalesced tile writes;
// dig_ax may be null (atx blocks only)
cudaError_t launch_oz_convert_tiles(const double* A, long r0, long r1, long rows, long cols,
                                    long lda, uint8_t* dig_ax, uint8_t* dig_atx,
                                    const int* row_ef, cudaStream_t st);
// row exponents + NaN/Inf flag + the stored digits (atx blocks; ax tiles unless dig_ax is
// null) of rows [r0, r1) in one pass over A (row_ef output; no column maxima)
cudaError_t launch_oz_scan_convert(const double* A, long r0, long r1, long rows, long cols,
                                   long lda, uint8_t* dig_ax, uint8_t* dig_atx, int* row_ef,
                                   int* flag, cudaStream_t st);

// INT8 GEMM from stored digits (gemm_oz.cu gemm_ozd_kernel):
//   mn = false: out (M x NP) = A X, adig = dig_ax (a_inner = ceil(K / 32)), a_ef[M] (row_ef).
//   mn = true:  out = A^T W' with A (K x M) as stored, adig = dig_atx (a_inner = ceil(M / 128)),
//               W' digits from launch_oz_digits_cols(..., row_ef, nfirst); a_ef unused.
// B digits (bdig) in the tiled layout for oz_chunks(NP). out_t / splits as GemmOz.
struct GemmOzd {
    bool mn = false;
    const uint8_t* adig = nullptr;
    long a_inner = 0;
    long M = 0, K = 0;
    const int* a_ef = nullptr;
    const uint8_t* bdig = nullptr;
    const int* b_ef = nullptr;
    int NP = 0;
    double* out = nullptr;
    long ldo = 0;
    bool out_t = false;
    int splits = 1;
    long split_stride = 0;
    const int* abort = nullptr;
};
cudaError_t launch_gemm_ozd(const GemmOzd& p, cudaStream_t st);
// bytes of the stored atx blocks of A (rows x cols): 4 ceil(rows / 128) x ceil(cols / 128) blocks
size_t oz_atx_bytes(long rows, long cols);
// bytes of the stored ax tiles of A: ceil(rows / 128) x ceil(cols / 32) blocks
size_t oz_ax_bytes(long rows, long cols);  // rows rounded up to 128

cudaError_t launch_gemm_ax(const GemmAx& p, cudaStream_t st);
cudaError_t launch_gemm_atx(const GemmAtx& p, cudaStream_t st);
cudaError_t launch_reduce_partials(const double* part, long stride, int splits, double* out,
                                   long count, cudaStream_t st);
// Same over FP32 slabs (out FP64): the split-K partials of the 3xTF32 GEMMs, whose TMEM
// accumulators are FP32, so storing them as FP32 halves the slab traffic and loses nothing.
cudaError_t launch_reduce_partials_f32(const float* part, long stride, int splits, double* out,
                                       long count, cudaStream_t st);

// FP64 tensor-core (DMMA m16n8k16) issue-rate probe on the whole GPU, TFLOP/s.
cudaError_t measure_dmma_peak(cudaStream_t st, double* tflops);
// INT8 tensor-core (tcgen05 kind::i8, M 128 N 256 K 32) issue-rate probe, TOPS.
cudaError_t measure_imma_peak(cudaStream_t st, double* tops);

// A GaussianSampler state (rng.hpp:21-42): words drawn so far (`counter`) and the cached
// sine half of an unfinished pair, which the next normal() returns first. A fresh
// sampler is {0, 0, 0}; after drawing N normals from fresh, counter = 2 ceil(N/2) and
// has_cached = N odd.
struct StreamPos {
    uint64_t counter = 0;
    int has_cached = 0;
    double cached = 0.0;
};

// Omega^T (NP x n, ld) for the reference's SplitMix64 + Box-Muller stream:
// Omega(r, c) = the (r*s + c)-th normal a GaussianSampler(seed) in state `pos` returns
// (default: fresh); rows c >= s of Omega^T are zero.
cudaError_t launch_omega(uint64_t seed, long n, int s, int NP, double* omega_t, long ld,
                         cudaStream_t st, StreamPos pos = {});
// Raw stream pieces for the bit-exactness tests.
cudaError_t launch_splitmix_words(uint64_t seed, uint64_t first_counter, long count,
                                  uint64_t* out, cudaStream_t st);
cudaError_t launch_uniforms(uint64_t seed, uint64_t first_counter, long count, double* out,
                            cudaStream_t st);
cudaError_t launch_gaussian_rowmajor(uint64_t seed, long rows, long cols, double* out,
                                     cudaStream_t st, StreamPos pos = {});

// Small dense linear algebra, one CTA, matrices in shared memory.
// Cholesky of the s x s Gram G (ld ldg): writes R (upper, NP x NP, ld NP, zero padded)
// and Rinv^T (NP x NP, ld NP, zero padded: usable directly as the Xt operand of ax).
// status[0] = 0 ok, 1 breakdown (min pivot below tol * max diag); status is int[4].
// Gref/ldref/sref (optional): the breakdown threshold is tol * max diag of Gref's leading
// sref x sref block instead of G's (blocked Cholesky: the Schur complement is judged
// against the whole Gram). accumulate: status[0] is only ever set to 1 (OR semantics),
// never cleared. Widths up to cholesky_max_width() (shared memory).
cudaError_t launch_cholesky(const double* G, long ldg, int s, int NP, double* R, double* RinvT,
                            int* status, int* abort_flag, double tol, cudaStream_t st,
                            const double* Gref = nullptr, long ldref = 0, int sref = 0,
                            bool accumulate = false, int out_n = 0);  // out_n: written block (0: NP)
int cholesky_max_width();
// C (M x N, ldc) = alpha op(A) op(B) + beta Cin; ta/tb: operand stored transposed.
// Cin == nullptr means Cin = C.
cudaError_t launch_small_gemm(int M, int N, int K, double alpha, const double* A, long lda,
                              bool ta, const double* B, long ldb, bool tb, double beta,
                              const double* Cin, long ldcin, double* C, long ldc,
                              cudaStream_t st);
// Block one-sided Jacobi for s > 160 (cooperative launch, global scratch).
cudaError_t launch_block_jacobi_svd(const double* R, int s, int NP, double* sigma, double* U,
                                    double* W, int* status, double* scratch,
                                    const int* abort_flag, cudaStream_t st);
size_t block_jacobi_scratch_doubles(int s);
// out (NP x NP) = X (NP x NP) * Y (NP x NP), row-major, s-leading block only (rest zero).
cudaError_t launch_small_matmul(const double* X, const double* Y, int s, int NP, double* out,
                                bool transpose_out, cudaStream_t st);
// One-sided Jacobi SVD of the s x s matrix R (row-major, ld NP) with the reference's
// thresholds (svd.cpp:35-36): sigma (s, sorted non-increasing), U (s x s -> NP x NP ld NP,
// left vectors), W (right vectors, NP x NP ld NP).  status[0] = sweeps or -1 on no convergence.
// `scratch` must hold jacobi_global_scratch_doubles(s) doubles; the kernel returns at
// once (status 0) if *abort_flag is set.
cudaError_t launch_jacobi_svd(const double* R, int s, int NP, double* sigma, double* U,
                              double* W, int* status, double* scratch, const int* abort_flag,
                              cudaStream_t st);
size_t jacobi_max_width();
size_t jacobi_global_scratch_doubles(int s);

// Sign convention (svd.cpp:237-254): for each column c < s of V (rows x NP, ld ldv),
// if the largest-|.| entry (first index on ties) is negative, negate V[:, c] and
// column c of Ub (NP x NP, ld NP).
cudaError_t launch_sign_fix(double* V, long rows, long ldv, int s, double* Ub, int NP,
                            cudaStream_t st);

// out (cols x rows, ld ldo) = in^T (in: rows x cols, ld ldi).
cudaError_t launch_transpose(const double* in, long rows, long cols, long ldi, double* out,
                             long ldo, cudaStream_t st);
// Copy rows x cols block between strided buffers.
cudaError_t launch_copy2d(const double* in, long ldi, double* out, long ldo, long rows, long cols,
                          cudaStream_t st);
// out (rows_pad x ldo) = V diag(sigma) (first k columns, rows < rows), zero elsewhere.
cudaError_t launch_scale_cols(const double* V, long ldv, long rows, long rows_pad, int k,
                              const double* sigma, double* out, long ldo, cudaStream_t st);
// out = x - 1 mean^T with mean = colsum / rows (written to mean_out) or mean_in if given.
cudaError_t launch_center(const double* x, long ldx, long rows, long cols, const double* colsum,
                          const double* mean_in, double* out, long ldo, double* mean_out,
                          cudaStream_t st);
// Zero-fill.
cudaError_t launch_fill(double* p, long count, double v, cudaStream_t st);
// NaN/Inf scan: ORs 1 into *flag.
cudaError_t launch_nonfinite_scan(const double* A, long rows, long cols, long lda, int* flag,
                                  cudaStream_t st);

// Blocked (32-column panels, compact WY) Householder QR of a tall M x s matrix Y
// (row-major, ldy; s <= NP <= 288, M >= s) in one cooperative launch, the CholeskyQR2
// fallback: the reference's algorithm (qr.cpp:27-102; diag R >= 0, Q accumulated
// backwards) with fixed-order reductions. Q to Qout (M x NP, ldq; columns >= s zero),
// R to R (NP x NP, zero padded). Y is not modified. `work` holds
// householder_work_doubles(M, NP) doubles.
cudaError_t launch_householder_qr(const double* Y, long M, int s, long ldy, double* Qout,
                                  long ldq, double* R, int NP, double* work, cudaStream_t st);
size_t householder_work_doubles(long M, int NP);

// Deterministic orthonormal completion (svd.cpp:111-151) of the null columns of the
// small SVD: the first j with !(sigma[j] > sigma[0] * null_dim * eps) starts the null
// block [j, s) (svd.cpp:221-234, decided on the device); those columns of U (rows x ld,
// row-major) are filled by Gram-Schmidt of canonical vectors ordered by row load.
// status[0] = 1 if no candidate survived. Returns at once if *abort_flag is set.
cudaError_t launch_complete_basis(double* U, long rows, long ld, int s, const double* sigma,
                                  long null_dim, double* work, int* status,
                                  const int* abort_flag, cudaStream_t st);
size_t complete_basis_work_doubles(long rows);

}  // namespace rsvdb200
