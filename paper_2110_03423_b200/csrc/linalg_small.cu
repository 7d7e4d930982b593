// Small dense linear algebra on the (k+p) x (k+p) side of the rSVD, one CTA (or, for the
// Jacobi at 64 < s <= 112, one thread-block cluster) each, operands held in shared memory:
//   * Cholesky of a Gram matrix + the triangular inverse (CholeskyQR, replaces the
//     reference's Householder QR, qr.cpp:27-102, on the well-conditioned path),
//   * one-sided Jacobi SVD of the small triangular factor R_B of B^T (replaces the
//     reference's Jacobi on the full n x s B^T, svd.cpp:153-263, same thresholds),
//   * the reference's sign convention (svd.cpp:237-254),
// plus the elementwise helpers (transpose, copies, NaN/Inf scan).
#include <float.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace rsvdb200 {

// =================================================================== Cholesky
// G (s x s, ldg) symmetric positive definite -> G = R^T R with R upper and a positive
// diagonal, plus Rinv^T = (R^-1)^T. Breakdown when a pivot falls below tol * max_i G_ii
// (status[0] = 1 and, if `abort` is given, *abort |= 1).
// Single CTA (512 threads), blocked by 16-wide panels. The matrix is padded to sp = s
// rounded up to 16 with a decoupled diagonal (max_i G_ii) so every panel is full.
//  * factorisation (right-looking, two barriers per panel): warp 0 factors the 16 x 16
//    diagonal block in registers (lane c holds column c; pivot rows travel by shuffle;
//    the pivot chain is one shuffle, a Newton reciprocal and an FMA per step - the square
//    roots are off the chain). The panel row block is solved column-parallel against it
//    (forward substitution in registers with the block's multipliers), then the trailing
//    upper triangle gets the rank-16 update in 4 x 4 register tiles while warp 0 updates
//    and factors the next diagonal block (lookahead).
//  * R is written transposed into the strict lower triangle as it is produced, and the
//    upper triangle is reset to I panel by panel, so the inversion R X = I runs in place
//    bottom-up by panels: 16 rows of X column-parallel (back substitution with broadcast R
//    loads), then the rank-16 update of every row above in 4 x 4 tiles.
// Shared memory: sp x (sp + 2) doubles + diag(R) and its reciprocals.
#ifdef CHOL_TRACE  // tools/probe/small_probe.cu: per-phase clock64 stamps of thread 0
__device__ long long g_chol_trace[256];
__device__ int g_chol_ntrace;
#define CHOL_MARK(tag)                                                   \
    do {                                                                 \
        if (threadIdx.x == 0 && g_chol_ntrace < 128) {                   \
            g_chol_trace[2 * g_chol_ntrace] = (tag);                     \
            g_chol_trace[2 * g_chol_ntrace + 1] = clock64();             \
            ++g_chol_ntrace;                                             \
        }                                                                \
    } while (0)
#else
#define CHOL_MARK(tag) \
    do {               \
    } while (0)
#endif
constexpr int kCholThreads = 512;
constexpr int kCholPanel = 16;

__host__ __device__ inline int chol_pad(int s) { return (s + kCholPanel - 1) & ~(kCholPanel - 1); }

// flat index e of the upper triangle of a T x T tile grid (row-major) -> (tr, tc), tc >= tr
__device__ __forceinline__ void chol_tri_index(int e, int T, int& tr, int& tc) {
    const float b = 2.0f * T + 1.0f;
    int r = (int)((b - sqrtf(fmaxf(b * b - 8.0f * e, 0.0f))) * 0.5f);
    auto start = [T](int q) { return q * T - q * (q - 1) / 2; };
    while (r > 0 && start(r) > e) --r;
    while (r + 1 < T && start(r + 1) <= e) ++r;
    tr = r;
    tc = r + (e - start(r));
}

// 1/d to full precision off the MUFU seed: two Newton steps
__device__ __forceinline__ double rcp_nr(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

struct __align__(16) CholShared {
    double U[kCholPanel * kCholPanel];  // U[k][i] = u_k[i]: pivot row k of the diagonal block
    double L[kCholPanel * 17];          // L[k][i] = u_k[i] / d_k (pivot row k over its pivot)
    double rs[kCholPanel];              // pivots d_k, then 1 / sqrt(d_k)
    int bad;
};

// Pivot step K of the diagonal block (template recursion: fully unrolled, a[] in registers;
// lane c holds column c, entries below the diagonal are don't-care). The pivot d = u_K[K]
// comes by shuffle (the chain: shuffle, Newton reciprocal, multiply, FMA); the rest of
// pivot row K is published through shared memory and read back as broadcasts, off the chain.
template <int K>
__device__ __forceinline__ void chol_pivot_steps(double (&a)[kCholPanel], int c, int lane,
                                                 double thresh, CholShared& cs, bool& ok) {
    if constexpr (K < kCholPanel) {
        constexpr unsigned kFull = 0xffffffffu;
        const double d = __shfl_sync(kFull, a[K], K);
        if constexpr (K + 1 < kCholPanel) {
            if (lane < kCholPanel) cs.U[K * kCholPanel + c] = a[K];
        }
        __syncwarp();
        ok = ok && (d > thresh);  // also catches NaN
        const double m = a[K] * rcp_nr(d);
        if (lane < kCholPanel) cs.L[K * 17 + c] = m;
        if (lane == 0) cs.rs[K] = d;
#pragma unroll
        for (int i = K + 1; i < kCholPanel; ++i) a[i] = fma(-cs.U[K * kCholPanel + i], m, a[i]);
        chol_pivot_steps<K + 1>(a, c, lane, thresh, cs, ok);
    }
}

// Warp 0: the diagonal block at j0 (after the updates of the panels before it; with
// `update`, panel jp's rank-16 update is applied here first). Lane c < 16 holds column c.
// Leaves L / rs for the panel solve, rdiag / dinv, the block's R transposed in S's strict
// lower triangle and I in its upper triangle; cs.bad = 1 on breakdown.
__device__ __forceinline__ void chol_diag_factor(double* S, int ld, int j0, double thresh,
                                                 CholShared& cs, double* rdiag, double* dinv,
                                                 int lane, bool update, int jp) {
    const int c = lane & (kCholPanel - 1);
    double a[kCholPanel];
#pragma unroll
    for (int i = 0; i < kCholPanel; ++i) a[i] = S[(j0 + i) * ld + j0 + c];
    if (update) {
#pragma unroll
        for (int k = 0; k < kCholPanel; ++k) {
            const double* row = S + (jp + k) * ld + j0;
            const double2* row2 = reinterpret_cast<const double2*>(row);
            const double rc = row[c];
#pragma unroll
            for (int i = 0; i < kCholPanel / 2; ++i) {
                const double2 v = row2[i];
                a[2 * i] = fma(-v.x, rc, a[2 * i]);
                a[2 * i + 1] = fma(-v.y, rc, a[2 * i + 1]);
            }
        }
    }
    CHOL_MARK(8);
    bool ok = true;
    chol_pivot_steps<0>(a, c, lane, thresh, cs, ok);
    __syncwarp();
    CHOL_MARK(9);
    if (lane < kCholPanel) {  // square roots off the pivot chain, one pivot per lane
        const double sq = sqrt(cs.rs[lane]), is = 1.0 / sq;
        rdiag[j0 + lane] = sq;
        dinv[j0 + lane] = is;
        cs.rs[lane] = is;
    }
    __syncwarp();
    if (lane < kCholPanel) {
#pragma unroll
        for (int k = 0; k < kCholPanel; ++k) {
            if (k < c) S[(j0 + c) * ld + j0 + k] = a[k] * cs.rs[k];  // R[k][c], transposed
            if (k <= c) S[(j0 + k) * ld + j0 + c] = (k == c) ? 1.0 : 0.0;
        }
    }
    if (lane == 0 && !ok) cs.bad = 1;
    CHOL_MARK(10);
}

__global__ void __launch_bounds__(kCholThreads) cholesky_kernel(
    const double* __restrict__ G, long ldg, int s, int NP, double* __restrict__ R,
    double* __restrict__ RinvT, int* __restrict__ status, int* __restrict__ abort_flag,
    double tol, const double* __restrict__ Gref, long ldref, int sref, bool accumulate,
    int out_n) {
    extern __shared__ __align__(16) double S[];
    const int sp = chol_pad(s), ld = sp + 2;
    double* rdiag = S + (size_t)sp * ld;
    double* dinv = rdiag + sp;
    __shared__ double gmax;
    __shared__ CholShared cs;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31;
    constexpr unsigned kFull = 0xffffffffu;
    if (warp == 0) {  // breakdown threshold relative to the largest diagonal of Gref
        double m = 0.0;
        for (int i = lane; i < sref; i += 32) m = fmax(m, Gref[i * ldref + i]);
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
        if (lane == 0) {
            gmax = m;
            cs.bad = 0;
        }
    }
    __syncthreads();
    const double thresh = tol * gmax;
    for (int e = tid; e < sp * sp; e += nth) {
        const int r = e / sp, c = e - r * sp;
        S[r * ld + c] = (r < s && c < s) ? (c >= r ? G[r * ldg + c] : 0.0) : (r == c ? gmax : 0.0);
    }
    __syncthreads();
    CHOL_MARK(0);

    // ---------------------------------------------------------------- factorisation
    // Phase A: warp 0 updates (with panel jp's rows) and factors the diagonal block of
    // panel j0 while warps 1.. apply panel jp's trailing update elsewhere. Phase B: the
    // panel row block of j0 is solved column-parallel. One call site for the diagonal
    // factor keeps its pivot loop unrolled in registers.
    for (int j0 = 0; j0 < sp; j0 += kCholPanel) {
        const int jp = j0 - kCholPanel;
        if (warp == 0) {
            chol_diag_factor(S, ld, j0, thresh, cs, rdiag, dinv, lane, jp >= 0, jp);
        } else if (jp >= 0 && (warp & 3)) {
            // trailing update A[j0:sp, j0:sp] -= R[jp:j0, j0:sp]^T R[jp:j0, j0:sp] (upper 4 x 4
            // tiles) except the diagonal block (warp 0's). Warps 4, 8, 12 stay idle so warp 0
            // has its scheduler (warp % 4) to itself: it is the critical path.
            const int nt = (sp - j0) >> 2;
            const int wq = warp - 1 - (warp >> 2);  // 0 .. 11 over the warps with warp % 4 != 0
            const int nsy = (nth >> 5) * 3 / 4 * 32;
            for (int e = wq * 32 + lane; e < nt * (nt + 1) / 2; e += nsy) {
                int tr, tc;
                chol_tri_index(e, nt, tr, tc);
                if (tc < kCholPanel / 4) continue;
                const int r = j0 + 4 * tr, cl = j0 + 4 * tc;
                double acc[4][4] = {};
#pragma unroll 4
                for (int k = 0; k < kCholPanel; ++k) {
                    const double2* pr = reinterpret_cast<const double2*>(S + (jp + k) * ld + r);
                    const double2* pc = reinterpret_cast<const double2*>(S + (jp + k) * ld + cl);
                    const double2 r01 = pr[0], r23 = pr[1], c01 = pc[0], c23 = pc[1];
                    const double rv[4] = {r01.x, r01.y, r23.x, r23.y};
                    const double cv[4] = {c01.x, c01.y, c23.x, c23.y};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) acc[i][jj] = fma(rv[i], cv[jj], acc[i][jj]);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) S[(r + i) * ld + cl + jj] -= acc[i][jj];
            }
        }
        __syncthreads();
        CHOL_MARK(3);
        if (cs.bad) break;
        const int j1 = j0 + kCholPanel;
        if (jp >= 0)  // the previous panel's rows over this diagonal block -> I (0)
            for (int e = tid; e < kCholPanel * kCholPanel; e += nth)
                S[(jp + (e >> 4)) * ld + j0 + (e & 15)] = 0.0;
        // panel row block: R[j0:j1, j1:sp] = R_dd^-T A[j0:j1, j1:sp], one column per thread;
        // R goes to the upper rows (for the trailing update) and transposed below
        for (int cc = j1 + tid; cc < sp; cc += nth) {
            double x[kCholPanel];
#pragma unroll
            for (int i = 0; i < kCholPanel; ++i) x[i] = S[(j0 + i) * ld + cc];
            if (jp >= 0)
#pragma unroll
                for (int i = 0; i < kCholPanel; ++i) S[(jp + i) * ld + cc] = 0.0;
#pragma unroll
            for (int k = 0; k < kCholPanel; ++k) {
#pragma unroll
                for (int i = k + 1; i < kCholPanel; ++i) x[i] = fma(-cs.L[k * 17 + i], x[k], x[i]);
                asm volatile("" ::: "memory");  // one multiplier row in registers at a time
            }
#pragma unroll
            for (int k = 0; k < kCholPanel; ++k) {
                const double r = x[k] * cs.rs[k];
                S[(j0 + k) * ld + cc] = r;
                S[cc * ld + j0 + k] = r;
            }
        }
        __syncthreads();
        CHOL_MARK(2);
    }
    if (cs.bad) {
        if (tid == 0) {
            status[0] = 1;  // (accumulate: OR into a status a previous block may have set)
            if (abort_flag) atomicOr(abort_flag, 1);
        }
        return;
    }

    // ---------------------------------------------------------------- inversion
    // upper triangle = B (I, updated) -> X = R^-1; R[m][l] (m < l) at S[l][m]
    for (int i0 = sp - kCholPanel; i0 >= 0; i0 -= kCholPanel) {
        for (int c = i0 + tid; c < sp; c += nth) {  // rows i0..i0+16 of X, column c
            double b[kCholPanel];
#pragma unroll
            for (int l = 0; l < kCholPanel; ++l) b[l] = (c >= i0 + l) ? S[(i0 + l) * ld + c] : 0.0;
#pragma unroll
            for (int l = kCholPanel - 1; l >= 0; --l) {
                b[l] *= dinv[i0 + l];
#pragma unroll
                for (int m = 0; m < l; ++m) b[m] = fma(-S[(i0 + l) * ld + i0 + m], b[l], b[m]);
                asm volatile("" ::: "memory");
            }
#pragma unroll
            for (int l = 0; l < kCholPanel; ++l)
                if (c >= i0 + l) S[(i0 + l) * ld + c] = b[l];
        }
        __syncthreads();
        CHOL_MARK(5);
        if (i0 == 0) break;
        // B[0:i0, i0:sp] -= R[0:i0, i0:i0+16] X[i0:i0+16, i0:sp]
        const int nr = i0 >> 2, nc = (sp - i0) >> 2;
        for (int e = tid; e < nr * nc; e += nth) {
            const int tr = e / nc, tc = e - tr * nc;
            const int r = 4 * tr, cl = i0 + 4 * tc;
            double acc[4][4] = {};
#pragma unroll 4
            for (int l = 0; l < kCholPanel; ++l) {
                const double2* pr = reinterpret_cast<const double2*>(S + (i0 + l) * ld + r);
                const double2* px = reinterpret_cast<const double2*>(S + (i0 + l) * ld + cl);
                const double2 r01 = pr[0], r23 = pr[1], x01 = px[0], x23 = px[1];
                const double rv[4] = {r01.x, r01.y, r23.x, r23.y};
                double xv[4] = {x01.x, x01.y, x23.x, x23.y};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
                    if (cl + jj < i0 + l) xv[jj] = 0.0;  // X is upper: below it lives R^T
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) acc[i][jj] = fma(rv[i], xv[jj], acc[i][jj]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) S[(r + i) * ld + cl + jj] -= acc[i][jj];
        }
        __syncthreads();
        CHOL_MARK(6);
    }
    // R[r][c] (c > r) and Rinv^T[r][c] = X[c][r] (c < r) both live at S[c][r]; the output is
    // the out_n x out_n block at R / RinvT (leading dimension NP), zero outside s x s
    for (int e = tid; e < out_n * out_n; e += nth) {
        const int r = e / out_n, c = e - r * out_n;
        double rv = 0.0, xv = 0.0;
        if (r < s && c < s) {
            const double v = S[c * ld + r];
            if (c > r) rv = v;
            else if (c < r) xv = v;
            else {
                rv = rdiag[r];
                xv = v;
            }
        }
        R[(size_t)r * NP + c] = rv;
        RinvT[(size_t)r * NP + c] = xv;
    }
    if (tid == 0 && !accumulate) status[0] = 0;
    CHOL_MARK(7);
}

size_t cholesky_smem(int s) {
    const size_t sp = chol_pad(s), ld = sp + 2;
    return (sp * ld + 2 * sp) * sizeof(double);
}

int cholesky_max_width() {
    int s = 1;
    while (cholesky_smem(s + 1) <= 225 * 1024) ++s;
    return s;
}

cudaError_t launch_cholesky(const double* G, long ldg, int s, int NP, double* R, double* RinvT,
                            int* status, int* abort_flag, double tol, cudaStream_t st,
                            const double* Gref, long ldref, int sref, bool accumulate,
                            int out_n) {
    if (out_n <= 0) out_n = NP;
    if (!Gref) {
        Gref = G;
        ldref = ldg;
        sref = s;
    }
    const size_t smem = cholesky_smem(s);
    if (smem > 225 * 1024) return cudaErrorInvalidValue;
    cudaError_t e =
        cudaFuncSetAttribute(cholesky_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cholesky_kernel<<<1, kCholThreads, smem, st>>>(G, ldg, s, NP, R, RinvT, status, abort_flag, tol,
                                                   Gref, ldref, sref, accumulate, out_n);
    return cudaGetLastError();
}

// out = X * Y (NP x NP each, s-leading block), optionally stored transposed.
__global__ void small_matmul_kernel(const double* __restrict__ X, const double* __restrict__ Y,
                                    int s, int NP, double* __restrict__ out, bool tr) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < NP * NP; e += gridDim.x * blockDim.x) {
        const int r = e / NP, c = e % NP;
        double acc = 0.0;
        if (r < s && c < s)
            for (int k = 0; k < s; ++k) acc += X[r * NP + k] * Y[k * NP + c];
        out[tr ? c * NP + r : e] = acc;
    }
}

cudaError_t launch_small_matmul(const double* X, const double* Y, int s, int NP, double* out,
                                bool transpose_out, cudaStream_t st) {
    small_matmul_kernel<<<(NP * NP + 255) / 256, 256, 0, st>>>(X, Y, s, NP, out, transpose_out);
    return cudaGetLastError();
}

// ============================================================ one-sided Jacobi
// Hestenes one-sided Jacobi on the columns of R (s x s): R J = U diag(sigma).
// Rotation rule and skip thresholds restate svd.cpp:35-36,60-90:
//   skip the pair (i, j) iff |d| <= 1e-14 * ||R||_F^2  and  d^2 <= (1e-13)^2 ||r_i||^2 ||r_j||^2
// (the norms and d are recomputed from the columns for every pair). A sweep visits
// all pairs in round-robin (tournament) order so the s/2 pairs of a round run
// concurrently, one 8-lane group per pair: each lane holds NQ row pairs of both columns
// in registers (double2 shared-memory accesses; the column stride is padded to 16 doubles
// when it fits so every group reads whole 128-byte lines), the reduction is three
// shuffles, and the CTA has just the warps the round needs. A sweep without any rotation
// ends the iteration (svd.cpp:196-199); more than 30 sweeps is a convergence failure
// (svd.hpp:20). The columns and the rotation accumulator J live in shared memory.
#ifdef JAC_TRACE  // tools/probe/small_probe.cu: per-phase clock64 stamps of thread 0 of CTA 0
__device__ long long g_jac_trace[1024];
__device__ int g_jac_ntrace;
#define JAC_DECL int jac_n = 0
#define JAC_MARK(tag)                                                          \
    do {                                                                       \
        if (threadIdx.x == 0 && blockIdx.x == 0 && jac_n < 512) {              \
            g_jac_trace[2 * jac_n] = (tag);                                    \
            g_jac_trace[2 * jac_n + 1] = clock64();                            \
            g_jac_ntrace = ++jac_n;                                            \
        }                                                                      \
    } while (0)
#else
#define JAC_DECL \
    do {         \
    } while (0)
#define JAC_MARK(tag) \
    do {              \
    } while (0)
#endif
constexpr int kJacobiGroup = 8;
constexpr int kJacobiMaxNQ = 7;  // row pairs per lane: s <= 8 * 2 * 7 = 112
// widths beyond (columns + J over 200 KB of shared memory) run the multi-CTA block Jacobi
// (linalg_blocked.cu)
constexpr int kJacobiSmemMax = 112;
constexpr int kMaxSweeps = 30;

__device__ __forceinline__ int rr_index(int slot, int round, int sp) {
    return slot == 0 ? 0 : 1 + (slot - 1 + round) % (sp - 1);
}

__host__ __device__ inline int jacobi_ld(int s) {
    const int l16 = (s + 15) & ~15;
    return 2 * (size_t)s * l16 * sizeof(double) <= 200 * 1024 ? l16 : (s + 1) & ~1;
}

template <int NQ, int G>
__global__ void __launch_bounds__(G == 16 ? 1024 : 512) jacobi_kernel(
    const double* __restrict__ Rin, int s, int NP, double* __restrict__ sigma_out,
    double* __restrict__ Uout, double* __restrict__ Wout, int* __restrict__ status,
    const int* __restrict__ abort_flag) {
    extern __shared__ __align__(16) double sh[];
    const int ls = jacobi_ld(s);
    double* Rc = sh;            // s columns, stride ls (rows s..ls-1 zero)
    double* J = sh + s * ls;    // s columns, stride ls
    __shared__ double abs_thresh;
    __shared__ double norms[kJacobiSmemMax];
    __shared__ int order[kJacobiSmemMax];
    const int tid = threadIdx.x, nth = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;
    if (abort_flag && *abort_flag) {  // an earlier stage failed; the host reruns robustly
        if (tid == 0) status[0] = 0;
        return;
    }
    __shared__ double scale_sh;
    if (warp == 0) {  // exact power-of-two scale so that the largest entry is O(1)
        double mx = 0.0;
        for (int e = lane; e < s * s; e += 32) mx = fmax(mx, fabs(Rin[(e % s) * NP + e / s]));
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) {
            int ex = 0;
            frexp(mx, &ex);
            scale_sh = mx > 0.0 ? ldexp(1.0, -ex) : 1.0;
        }
    }
    __syncthreads();
    const double scale = scale_sh;
    for (int e = tid; e < s * ls; e += nth) {
        const int c = e / ls, r = e - c * ls;
        Rc[e] = r < s ? Rin[r * NP + c] * scale : 0.0;
        J[e] = (r == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
        double acc = 0.0;
        for (int e = lane; e < s * ls; e += 32) acc += Rc[e] * Rc[e];
        acc = warp_sum(acc);
        if (lane == 0) abs_thresh = 1e-14 * acc;
    }
    __syncthreads();
    const double athr = abs_thresh;

    const int sp = (s + 1) & ~1;  // even number of tournament slots (slot s is a bye)
    const int k = tid / G, gl = tid % G;  // this group's pair slot (one pass: k < sp / 2)
    int sweeps = 0;
    bool converged = false;
    while (sweeps < kMaxSweeps) {
        ++sweeps;
        int rotated = 0;
        // rr_index(slot, round) = slot == 0 ? 0 : 1 + (slot - 1 + round) % (sp - 1), stepped
        // incrementally (no integer division in the round loop)
        int ri = k == 0 ? -1 : k - 1, rj = sp - 2 - k;
        for (int round = 0; round < sp - 1; ++round) {
            int i = 0, j = 0;
            bool live = k < sp / 2;
            if (live) {
                i = ri < 0 ? 0 : 1 + ri;
                j = 1 + rj;
                if (i > j) { const int t = i; i = j; j = t; }
                live = j < s;
            }
            if (ri >= 0 && ++ri == sp - 1) ri = 0;
            if (++rj == sp - 1) rj = 0;
            double2* ci = reinterpret_cast<double2*>(Rc + i * ls) + gl;
            double2* cj = reinterpret_cast<double2*>(Rc + j * ls) + gl;
            double2 xi[NQ], xj[NQ];
            double aii = 0.0, ajj = 0.0, d = 0.0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const bool in = live && 2 * (gl + q * G) < ls;
                xi[q] = in ? ci[q * G] : make_double2(0.0, 0.0);
                xj[q] = in ? cj[q * G] : make_double2(0.0, 0.0);
                aii = fma(xi[q].x, xi[q].x, fma(xi[q].y, xi[q].y, aii));
                ajj = fma(xj[q].x, xj[q].x, fma(xj[q].y, xj[q].y, ajj));
                d = fma(xi[q].x, xj[q].x, fma(xi[q].y, xj[q].y, d));
            }
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) {  // xor offsets < G stay inside the group
                aii += __shfl_xor_sync(0xffffffffu, aii, o);
                ajj += __shfl_xor_sync(0xffffffffu, ajj, o);
                d += __shfl_xor_sync(0xffffffffu, d, o);
            }
            if (live && !(fabs(d) <= athr && d * d <= (1e-13 * 1e-13) * aii * ajj)) {
                // zeta = (ajj - aii) / (2d), t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2))
                //      = sign(zeta) 2|d| / (|ajj - aii| + sqrt((ajj - aii)^2 + 4 d^2))
                const double diff = ajj - aii;
                const double sgn = ((diff >= 0.0) == (d >= 0.0)) || diff == 0.0 ? 1.0 : -1.0;
                const double t =
                    sgn * 2.0 * fabs(d) / (fabs(diff) + sqrt(fma(diff, diff, 4.0 * d * d)));
                const double c = rsqrt(fma(t, t, 1.0));
                const double sn = c * t;
                double2* wi = reinterpret_cast<double2*>(J + i * ls) + gl;
                double2* wj = reinterpret_cast<double2*>(J + j * ls) + gl;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    if (2 * (gl + q * G) < ls) {
                        const double2 yi = wi[q * G], yj = wj[q * G];
                        ci[q * G] = make_double2(c * xi[q].x - sn * xj[q].x, c * xi[q].y - sn * xj[q].y);
                        cj[q * G] = make_double2(sn * xi[q].x + c * xj[q].x, sn * xi[q].y + c * xj[q].y);
                        wi[q * G] = make_double2(c * yi.x - sn * yj.x, c * yi.y - sn * yj.y);
                        wj[q * G] = make_double2(sn * yi.x + c * yj.x, sn * yi.y + c * yj.y);
                    }
                }
                rotated = 1;
            }
            __syncthreads();
        }
        if (!__syncthreads_or(rotated)) {
            converged = true;
            break;
        }
    }
    if (!converged) {
        if (tid == 0) status[0] = -1;
        return;
    }
    // singular values = column norms; stable descending order (svd.cpp:210-219)
    for (int c = warp; c < s; c += nwarps) {
        double acc = 0.0;
        for (int r = lane; r < s; r += 32) acc += Rc[c * ls + r] * Rc[c * ls + r];
        acc = warp_sum(acc);
        if (lane == 0) norms[c] = sqrt(acc);
    }
    __syncthreads();
    for (int c = tid; c < s; c += nth) {  // rank of column c in the stable descending order
        int rank = 0;
        for (int o = 0; o < s; ++o)
            rank += (norms[o] > norms[c]) || (norms[o] == norms[c] && o < c);
        order[rank] = c;
    }
    __syncthreads();
    for (int e = tid; e < NP * NP; e += nth) {
        const int r = e / NP, cc = e % NP;
        double u = 0.0, w = 0.0;
        if (r < s && cc < s) {
            const int src = order[cc];
            const double sg = norms[src];
            u = sg > 0.0 ? Rc[src * ls + r] / sg : 0.0;
            w = J[src * ls + r];
        }
        Uout[e] = u;
        Wout[e] = w;
    }
    for (int c = tid; c < NP; c += nth) sigma_out[c] = c < s ? norms[order[c]] / scale : 0.0;
    if (tid == 0) status[0] = sweeps;
}

// ------------------------------------------------- one-sided Jacobi over a thread-block cluster
// The single-CTA rounds above are bound by the SM's shared-memory pipe (every round reads and
// writes all of R and J: ~1.8k cycles of LDS/STS/SHFL per round at s = 74). Here the rows are
// split over a cluster: CTA r holds rows [RPC r, RPC r + RPC) of every column of R and J
// (RPC = 8 NQ), so each SM moves 1/NC of the bytes. A pair's group (4 lanes, NQ double2 each)
// reduces its rows' partial (|r_i|^2, |r_j|^2, r_i.r_j), lane 0 stores the partial into every
// CTA's shared memory, one cluster barrier, and every CTA adds the NC partials in rank order:
// all CTAs see bit-identical sums, so they take identical skip / rotation decisions (and agree
// on convergence) without further exchange. Same ordering, rotation formula and thresholds as
// jacobi_kernel (svd.cpp:35-36,60-90,196-199).
constexpr int kJcLanes = 4;

// 16 bytes into a cluster peer's shared memory, counted by the peer's mbarrier (complete_tx)
__device__ __forceinline__ void st_async_f64x2(uint32_t caddr, double a, double b, uint32_t cbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                 ::"r"(caddr), "d"(a), "d"(b), "r"(cbar) : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

template <int NQ>
__global__ void __launch_bounds__(1024) jacobi_cluster_kernel(
    const double* __restrict__ Rin, int s, int NP, double* __restrict__ sigma_out,
    double* __restrict__ Uout, double* __restrict__ Wout, int* __restrict__ status,
    const int* __restrict__ abort_flag) {
    constexpr int RPC = 8 * NQ;  // rows per CTA (column stride in shared memory)
    extern __shared__ __align__(16) double sh[];
    uint32_t nc, rank;
    asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(nc));
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int sp = (s + 1) & ~1, pairs = sp / 2;
    double* Rc = sh;                    // s columns x RPC rows
    double* J = Rc + (size_t)s * RPC;   // s columns x RPC rows
    double* part = J + (size_t)s * RPC; // [2][nc][pairs][4]: per-round partials of every CTA
    __shared__ double red_sh[2];
    const int tid = threadIdx.x, nth = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (abort_flag && *abort_flag) {  // every CTA reads the same flag: all leave together
        if (tid == 0 && rank == 0) status[0] = 0;
        return;
    }
    if (warp == 0) {  // scale and skip threshold from the whole matrix, identically in every CTA
        double mx = 0.0, f2 = 0.0;
        for (int e = lane; e < s * s; e += 32) {
            const double v = Rin[(e / s) * NP + e % s];
            mx = fmax(mx, fabs(v));
        }
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        int ex = 0;
        frexp(mx, &ex);
        const double scale = mx > 0.0 ? ldexp(1.0, -ex) : 1.0;
        for (int e = lane; e < s * s; e += 32) {
            const double v = Rin[(e / s) * NP + e % s] * scale;
            f2 = fma(v, v, f2);
        }
        f2 = warp_sum(f2);
        if (lane == 0) {
            red_sh[0] = scale;
            red_sh[1] = 1e-14 * f2;
        }
    }
    __syncthreads();
    const double scale = red_sh[0], athr = red_sh[1];
    const int r0 = (int)rank * RPC;
    for (int e = tid; e < s * RPC; e += nth) {
        const int c = e / RPC, rr = e - c * RPC, r = r0 + rr;
        Rc[e] = r < s ? Rin[(size_t)r * NP + c] * scale : 0.0;
        J[e] = (r == c) ? 1.0 : 0.0;
    }
    const uint32_t part_u32 = smem_u32(part);
    // full[slot]: round n's partials (slot n & 1) from every CTA have landed here (st.async
    // complete_tx; thread 0 arms the expected bytes once per round)
    __shared__ __align__(8) uint64_t full[2];
    const uint32_t round_bytes = (uint32_t)(nc * pairs * 4 * sizeof(double));
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_barrier_init();
    }
    cluster_sync_all();  // every CTA of the cluster is running, barriers initialised

    const int k = tid / kJcLanes, gl = tid % kJcLanes;
    const bool slot_ok = k < pairs;
    const int qx = k & 1;  // odd slots walk their double2s in swapped pairs: a quarter-warp's two
                           // groups touch opposite halves of the banks
    int sweeps = 0, nround = 0;
    bool converged = false;
    JAC_DECL;
    while (sweeps < kMaxSweeps) {
        ++sweeps;
        int rotated = 0;
        int ri = k == 0 ? -1 : k - 1, rj = sp - 2 - k;
        for (int round = 0; round < sp - 1; ++round, ++nround) {
            int i = 0, j = 0;
            bool live = slot_ok;
            if (live) {
                i = ri < 0 ? 0 : 1 + ri;
                j = 1 + rj;
                if (i > j) { const int t = i; i = j; j = t; }
                live = j < s;
            }
            if (ri >= 0 && ++ri == sp - 1) ri = 0;
            if (++rj == sp - 1) rj = 0;
            JAC_MARK(0);
            double2* ci = reinterpret_cast<double2*>(Rc + i * RPC);
            double2* cj = reinterpret_cast<double2*>(Rc + j * RPC);
            double2 xi[NQ], xj[NQ];
            double aii = 0.0, ajj = 0.0, d = 0.0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int e = gl + kJcLanes * (q ^ qx);
                xi[q] = live ? ci[e] : make_double2(0.0, 0.0);
                xj[q] = live ? cj[e] : make_double2(0.0, 0.0);
                aii = fma(xi[q].x, xi[q].x, fma(xi[q].y, xi[q].y, aii));
                ajj = fma(xj[q].x, xj[q].x, fma(xj[q].y, xj[q].y, ajj));
                d = fma(xi[q].x, xj[q].x, fma(xi[q].y, xj[q].y, d));
            }
            JAC_MARK(1);
#pragma unroll
            for (int o = kJcLanes / 2; o > 0; o >>= 1) {
                aii += __shfl_xor_sync(0xffffffffu, aii, o);
                ajj += __shfl_xor_sync(0xffffffffu, ajj, o);
                d += __shfl_xor_sync(0xffffffffu, d, o);
            }
            JAC_MARK(2);
            const int slot = nround & 1;
            if (tid == 0) mbar_arrive_expect_tx(&full[slot], round_bytes);
            if (slot_ok && gl < (int)nc) {  // lane gl (and gl + 4, ...) feeds CTA gl's copy
                const uint32_t off =
                    (uint32_t)((((slot * nc + rank) * pairs + k) * 4) * sizeof(double));
                const uint32_t bar = smem_u32(&full[slot]);
                for (uint32_t dst = gl; dst < nc; dst += kJcLanes) {
                    const uint32_t ca = mapa_rank(part_u32 + off, dst);
                    const uint32_t cb = mapa_rank(bar, dst);
                    st_async_f64x2(ca, aii, ajj, cb);
                    st_async_f64x2(ca + 16, d, 0.0, cb);
                }
            }
            mbar_wait_cluster(&full[slot], (uint32_t)(nround >> 1) & 1u);
            JAC_MARK(3);
            if (live) {
                aii = ajj = d = 0.0;
                for (uint32_t rk = 0; rk < nc; ++rk) {  // rank order: identical in every CTA
                    const double2* pp =
                        reinterpret_cast<const double2*>(part + ((slot * nc + rk) * pairs + k) * 4);
                    const double2 a = pp[0], b = pp[1];
                    aii += a.x;
                    ajj += a.y;
                    d += b.x;
                }
            }
            if (live && !(fabs(d) <= athr && d * d <= (1e-13 * 1e-13) * aii * ajj)) {
                const double diff = ajj - aii;
                const double sgn = ((diff >= 0.0) == (d >= 0.0)) || diff == 0.0 ? 1.0 : -1.0;
                const double t =
                    sgn * 2.0 * fabs(d) / (fabs(diff) + sqrt(fma(diff, diff, 4.0 * d * d)));
                const double c = rsqrt(fma(t, t, 1.0));
                const double sn = c * t;
                double2* wi = reinterpret_cast<double2*>(J + i * RPC);
                double2* wj = reinterpret_cast<double2*>(J + j * RPC);
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const int e = gl + kJcLanes * (q ^ qx);
                    const double2 yi = wi[e], yj = wj[e];
                    ci[e] = make_double2(c * xi[q].x - sn * xj[q].x, c * xi[q].y - sn * xj[q].y);
                    cj[e] = make_double2(sn * xi[q].x + c * xj[q].x, sn * xi[q].y + c * xj[q].y);
                    wi[e] = make_double2(c * yi.x - sn * yj.x, c * yi.y - sn * yj.y);
                    wj[e] = make_double2(sn * yi.x + c * yj.x, sn * yi.y + c * yj.y);
                }
                rotated = 1;
            }
            JAC_MARK(4);
            // the next round's groups read columns this round rotated; a peer's round-(n+2)
            // partials reuse slot n & 1 only after it has seen ours of round n + 1, which we
            // send after these reads
            __syncthreads();
            JAC_MARK(5);
        }
        if (!__syncthreads_or(rotated)) {  // identical in every CTA (identical decisions)
            converged = true;
            break;
        }
    }
    if (!converged) {
        if (tid == 0 && rank == 0) status[0] = -1;
        cluster_sync_all();
        return;
    }
    // singular values = column norms (partials of every CTA, added in rank order); stable
    // descending order (svd.cpp:210-219)
    double* npart = part;  // [nc][s], reusing the partial buffers: once every CTA has read
    cluster_sync_all();    // the last round's partials
    for (int c = tid; c < s; c += nth) {
        double acc = 0.0;
        for (int rr = 0; rr < RPC; ++rr) acc = fma(Rc[c * RPC + rr], Rc[c * RPC + rr], acc);
        for (uint32_t dst = 0; dst < nc; ++dst) {
            const uint32_t ca =
                mapa_rank(part_u32 + (uint32_t)((rank * s + c) * sizeof(double)), dst);
            asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ca), "d"(acc) : "memory");
        }
    }
    cluster_sync_all();
    __shared__ double norms[kJacobiSmemMax];
    __shared__ int order[kJacobiSmemMax];
    for (int c = tid; c < s; c += nth) {
        double acc = 0.0;
        for (uint32_t rk = 0; rk < nc; ++rk) acc += npart[rk * s + c];
        norms[c] = sqrt(acc);
    }
    __syncthreads();
    for (int c = tid; c < s; c += nth) {
        int rnk = 0;
        for (int o = 0; o < s; ++o) rnk += (norms[o] > norms[c]) || (norms[o] == norms[c] && o < c);
        order[rnk] = c;
    }
    __syncthreads();
    const int rend = rank + 1 == nc ? NP : r0 + RPC;  // the last CTA also zero-fills rows >= nc RPC
    for (int e = tid; e < (rend - r0) * NP; e += nth) {
        const int r = r0 + e / NP, cc = e % NP;
        double u = 0.0, w = 0.0;
        if (r < s && cc < s) {
            const int src = order[cc];
            const double sg = norms[src];
            u = sg > 0.0 ? Rc[src * RPC + (r - r0)] / sg : 0.0;
            w = J[src * RPC + (r - r0)];
        }
        Uout[(size_t)r * NP + cc] = u;
        Wout[(size_t)r * NP + cc] = w;
    }
    if (rank == 0) {
        for (int c = tid; c < NP; c += nth) sigma_out[c] = c < s ? norms[order[c]] / scale : 0.0;
        if (tid == 0) status[0] = sweeps;
    }
}

template <int NQ>
static size_t jacobi_cluster_smem(int s, int nc) {
    const int pairs = ((s + 1) & ~1) / 2;
    const size_t cols = 2 * (size_t)s * 8 * NQ;
    const size_t part = std::max((size_t)2 * nc * pairs * 4, (size_t)nc * s);
    return (cols + part) * sizeof(double);
}

template <int NQ>
static cudaError_t launch_jacobi_cluster(const double* R, int s, int NP, double* sigma, double* U,
                                         double* W, int* status, const int* abort_flag,
                                         cudaStream_t st) {
    const int nc = (s + 8 * NQ - 1) / (8 * NQ);
    const int pairs = ((s + 1) & ~1) / 2;
    const size_t smem = jacobi_cluster_smem<NQ>(s, nc);
    if (nc > 8 || smem > 200 * 1024 || pairs * kJcLanes > 1024) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(jacobi_cluster_kernel<NQ>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nc);
    cfg.blockDim = dim3((pairs * kJcLanes + 31) & ~31);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = nc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, jacobi_cluster_kernel<NQ>, R, s, NP, sigma, U, W, status,
                              abort_flag);
}

size_t jacobi_max_width() { return 320; }

size_t jacobi_global_scratch_doubles(int s) {
    return block_jacobi_scratch_doubles(s);  // the block Jacobi's scratch
}

template <int NQ, int G>
static cudaError_t launch_jacobi_g(const double* R, int s, int NP, double* sigma, double* U,
                                   double* W, int* status, const int* abort_flag,
                                   cudaStream_t st) {
    const size_t smem = 2 * (size_t)s * jacobi_ld(s) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(jacobi_kernel<NQ, G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int pairs = ((s + 1) & ~1) / 2;
    const int threads = std::max(128, (pairs * G + 31) & ~31);
    jacobi_kernel<NQ, G><<<1, threads, smem, st>>>(R, s, NP, sigma, U, W, status, abort_flag);
    return cudaGetLastError();
}

// 16 lanes per column pair when the pairs fit 1024 threads (s <= 128): half the per-lane rows
// (shorter dependent chains per round) at one more shuffle level; 8 lanes otherwise
template <int NQ>
static cudaError_t launch_jacobi_nq(const double* R, int s, int NP, double* sigma, double* U,
                                    double* W, int* status, const int* abort_flag,
                                    cudaStream_t st) {
    static const bool g16 = getenv("RSVD_B200_JACOBI_G16") != nullptr;  // measured equal (0.59 ms)
    const int pairs = ((s + 1) & ~1) / 2;
    if (g16 && pairs * 16 <= 1024)
        return launch_jacobi_g<(NQ + 1) / 2, 16>(R, s, NP, sigma, U, W, status, abort_flag, st);
    return launch_jacobi_g<NQ, kJacobiGroup>(R, s, NP, sigma, U, W, status, abort_flag, st);
}

cudaError_t launch_jacobi_svd(const double* R, int s, int NP, double* sigma, double* U, double* W,
                              int* status, double* scratch, const int* abort_flag,
                              cudaStream_t st) {
    if (s > (int)jacobi_max_width()) return cudaErrorInvalidValue;
    static const int smem_max = getenv("RSVD_B200_JACOBI_SMEM_MAX")
                                    ? atoi(getenv("RSVD_B200_JACOBI_SMEM_MAX"))
                                    : kJacobiSmemMax;
    if (s > std::min(smem_max, kJacobiSmemMax))
        return launch_block_jacobi_svd(R, s, NP, sigma, U, W, status, scratch, abort_flag, st);
    // the cluster variant pays ~0.5k cycles of DSMEM exchange per round and saves shared-memory
    // pipe cycles in proportion to s: measured (tools/probe/small_probe.cu, cycles per round)
    // s = 48: 1686 vs 1438 single-CTA, s = 74: 2209 vs 2318, s = 112: 2925 vs 3634
    static const int cl_min = getenv("RSVD_B200_JACOBI_CLUSTER_MIN")
                                  ? atoi(getenv("RSVD_B200_JACOBI_CLUSTER_MIN"))
                                  : 64;
    if (s > std::max(cl_min, 16))
        return launch_jacobi_cluster<2>(R, s, NP, sigma, U, W, status, abort_flag, st);
    switch ((jacobi_ld(s) + 15) / 16) {  // row pairs per lane
        case 1: return launch_jacobi_nq<1>(R, s, NP, sigma, U, W, status, abort_flag, st);
        case 2: return launch_jacobi_nq<2>(R, s, NP, sigma, U, W, status, abort_flag, st);
        case 3: return launch_jacobi_nq<3>(R, s, NP, sigma, U, W, status, abort_flag, st);
        case 4: return launch_jacobi_nq<4>(R, s, NP, sigma, U, W, status, abort_flag, st);
        case 5: return launch_jacobi_nq<5>(R, s, NP, sigma, U, W, status, abort_flag, st);
        case 6: return launch_jacobi_nq<6>(R, s, NP, sigma, U, W, status, abort_flag, st);
        default: return launch_jacobi_nq<7>(R, s, NP, sigma, U, W, status, abort_flag, st);
    }
}

// ============================================================== sign convention
__global__ void sign_fix_kernel(double* __restrict__ V, long rows, long ldv, int s,
                                double* __restrict__ Ub, int NP) {
    const int c = blockIdx.x;
    if (c >= s) return;
    double best = -1.0;
    long arg = 0;
    for (long r = threadIdx.x; r < rows; r += blockDim.x) {
        const double a = fabs(V[r * ldv + c]);
        if (a > best) {  // strictly greater keeps the first index per thread
            best = a;
            arg = r;
        }
    }
    __shared__ double sb[32];
    __shared__ long sa[32];
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, o);
        const long oa = __shfl_down_sync(0xffffffffu, arg, o);
        if (ob > best || (ob == best && oa < arg)) {
            best = ob;
            arg = oa;
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sb[warp] = best;
        sa[warp] = arg;
    }
    __syncthreads();
    __shared__ int flip;
    if (threadIdx.x == 0) {
        double b = sb[0];
        long a = sa[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (sb[w] > b || (sb[w] == b && sa[w] < a)) {
                b = sb[w];
                a = sa[w];
            }
        flip = V[a * ldv + c] < 0.0;
    }
    __syncthreads();
    if (flip) {
        for (long r = threadIdx.x; r < rows; r += blockDim.x) V[r * ldv + c] = -V[r * ldv + c];
        for (int r = threadIdx.x; r < NP; r += blockDim.x) Ub[r * NP + c] = -Ub[r * NP + c];
    }
}

cudaError_t launch_sign_fix(double* V, long rows, long ldv, int s, double* Ub, int NP,
                            cudaStream_t st) {
    sign_fix_kernel<<<s, 256, 0, st>>>(V, rows, ldv, s, Ub, NP);
    return cudaGetLastError();
}

// ============================================================ elementwise helpers
__global__ void transpose_kernel(const double* __restrict__ in, long rows, long cols, long ldi,
                                 double* __restrict__ out, long ldo) {
    __shared__ double tile[32][33];
    const long r0 = (long)blockIdx.y * 32, c0 = (long)blockIdx.x * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const long r = r0 + y, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[y][threadIdx.x] = in[r * ldi + c];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const long c = c0 + y, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[c * ldo + r] = tile[threadIdx.x][y];
    }
}

cudaError_t launch_transpose(const double* in, long rows, long cols, long ldi, double* out,
                             long ldo, cudaStream_t st) {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(in, rows, cols, ldi, out, ldo);
    return cudaGetLastError();
}

__global__ void copy2d_kernel(const double* __restrict__ in, long ldi, double* __restrict__ out,
                              long ldo, long rows, long cols) {
    const long total = rows * cols;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const long r = e / cols, c = e % cols;
        out[r * ldo + c] = in[r * ldi + c];
    }
}

static unsigned grid_for(long work, int threads) {
    long b = (work + threads - 1) / threads;
    if (b > 148L * 32) b = 148L * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

cudaError_t launch_copy2d(const double* in, long ldi, double* out, long ldo, long rows, long cols,
                          cudaStream_t st) {
    copy2d_kernel<<<grid_for(rows * cols, 256), 256, 0, st>>>(in, ldi, out, ldo, rows, cols);
    return cudaGetLastError();
}

// out (rows_pad x k, ldo) = V diag(sigma) for rows < rows, zero below (residual operand).
__global__ void scale_cols_kernel(const double* __restrict__ V, long ldv, long rows, long rows_pad,
                                  int k, const double* __restrict__ sigma, double* __restrict__ out,
                                  long ldo) {
    const long total = rows_pad * ldo;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const long r = e / ldo, t = e % ldo;
        out[e] = (r < rows && t < k) ? V[r * ldv + t] * sigma[t] : 0.0;
    }
}

cudaError_t launch_scale_cols(const double* V, long ldv, long rows, long rows_pad, int k,
                              const double* sigma, double* out, long ldo, cudaStream_t st) {
    scale_cols_kernel<<<grid_for(rows_pad * ldo, 256), 256, 0, st>>>(V, ldv, rows, rows_pad, k,
                                                                     sigma, out, ldo);
    return cudaGetLastError();
}

// PCA centering (pca.cpp:10-26): mean[j] = colsum[j] / n (when mean_out is given) and
// out[i][j] = x[i][j] - mean[j]; `mean_in` supplies a fixed mean instead (transform).
__global__ void center_kernel(const double* __restrict__ x, long ldx, long rows, long cols,
                              const double* __restrict__ colsum, const double* __restrict__ mean_in,
                              double inv_rows, double* __restrict__ out, long ldo,
                              double* __restrict__ mean_out) {
    const long total = rows * cols;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const long i = e / cols, j = e % cols;
        const double mu = mean_in ? mean_in[j] : colsum[j] * inv_rows;
        out[i * ldo + j] = x[i * ldx + j] - mu;
        if (mean_out && i == 0) mean_out[j] = mu;
    }
}

cudaError_t launch_center(const double* x, long ldx, long rows, long cols, const double* colsum,
                          const double* mean_in, double* out, long ldo, double* mean_out,
                          cudaStream_t st) {
    center_kernel<<<grid_for(rows * cols, 256), 256, 0, st>>>(
        x, ldx, rows, cols, colsum, mean_in, 1.0 / (double)rows, out, ldo, mean_out);
    return cudaGetLastError();
}

__global__ void fill_kernel(double* p, long count, double v) {
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < count;
         e += (long)gridDim.x * blockDim.x)
        p[e] = v;
}

cudaError_t launch_fill(double* p, long count, double v, cudaStream_t st) {
    fill_kernel<<<grid_for(count, 256), 256, 0, st>>>(p, count, v);
    return cudaGetLastError();
}

__global__ void nonfinite_kernel(const double* __restrict__ A, long rows, long cols, long lda,
                                 int* flag) {
    bool bad = false;
    const long total = rows * cols;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const double x = A[(e / cols) * lda + e % cols];
        bad |= ((__double_as_longlong(x) >> 52) & 0x7ff) == 0x7ff;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

cudaError_t launch_nonfinite_scan(const double* A, long rows, long cols, long lda, int* flag,
                                  cudaStream_t st) {
    nonfinite_kernel<<<grid_for(rows * cols, 256), 256, 0, st>>>(A, rows, cols, lda, flag);
    return cudaGetLastError();
}

}  // namespace rsvdb200
