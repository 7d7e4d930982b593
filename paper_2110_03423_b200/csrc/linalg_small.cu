// Small dense linear algebra on the (k+p) x (k+p) side of the rSVD, one CTA each,
// operands held in shared memory:
//   * Cholesky of a Gram matrix + the triangular inverse (CholeskyQR, replaces the
//     reference's Householder QR, qr.cpp:27-102, on the well-conditioned path),
//   * one-sided Jacobi SVD of the small triangular factor R_B of B^T (replaces the
//     reference's Jacobi on the full n x s B^T, svd.cpp:153-263, same thresholds),
//   * the reference's sign convention (svd.cpp:237-254),
// plus the elementwise helpers (transpose, copies, NaN/Inf scan).
#include <float.h>

#include "common.cuh"
#include "kernels.h"

namespace rsvdb200 {

// =================================================================== Cholesky
// G (s x s, ldg) symmetric positive definite -> G = R^T R, R upper with positive
// diagonal.  Breakdown (status[0] = 1) when a pivot falls below tol * max_i G_ii.
// Writes R (NP x NP, zero padded) and Rinv^T (NP x NP, zero padded).  Only R is
// staged in shared memory (s <= 168); each thread back-substitutes one column of
// R^-1 straight into its row of Rinv^T.
__global__ void __launch_bounds__(512) cholesky_kernel(const double* __restrict__ G, long ldg,
                                                       int s, int NP, double* __restrict__ R,
                                                       double* __restrict__ RinvT,
                                                       int* __restrict__ status, double tol) {
    extern __shared__ double a[];  // s x s row-major, upper triangle used
    __shared__ double gmax;
    __shared__ int broke;
    const int tid = threadIdx.x, nth = blockDim.x;
    for (int e = tid; e < s * s; e += nth) a[e] = G[(e / s) * ldg + e % s];
    if (tid == 0) {
        broke = 0;
        double m = 0.0;
        for (int i = 0; i < s; ++i) m = fmax(m, G[i * ldg + i]);
        gmax = m;
    }
    __syncthreads();
    const double thresh = tol * gmax;
    for (int j = 0; j < s; ++j) {
        const double d = a[j * s + j];
        if (!(d > thresh)) {  // also catches NaN
            if (tid == 0) broke = 1;
            break;
        }
        const double rjj = sqrt(d);
        __syncthreads();
        for (int c = j + tid; c < s; c += nth) a[j * s + c] = (c == j) ? rjj : a[j * s + c] / rjj;
        __syncthreads();
        const int rem = s - j - 1;
        for (int e = tid; e < rem * rem; e += nth) {
            const int r = j + 1 + e / rem, c = j + 1 + e % rem;
            if (c >= r) a[r * s + c] -= a[j * s + r] * a[j * s + c];
        }
        __syncthreads();
    }
    __syncthreads();
    if (broke) {
        if (tid == 0) status[0] = 1;
        return;
    }
    for (int e = tid; e < NP * NP; e += nth) {
        const int r = e / NP, c = e % NP;
        R[e] = (r < s && c < s && c >= r) ? a[r * s + c] : 0.0;
    }
    // Rinv column c -> RinvT row c: x_i = (delta_ic - sum_{k=i+1..c} R_ik x_k) / R_ii
    for (int c = tid; c < NP; c += nth) {
        double* x = RinvT + (long)c * NP;
        for (int i = c + 1; i < NP; ++i) x[i] = 0.0;
        if (c >= s) {
            for (int i = 0; i <= c; ++i) x[i] = 0.0;
            continue;
        }
        for (int i = c; i >= 0; --i) {
            double acc = (i == c) ? 1.0 : 0.0;
            for (int k = i + 1; k <= c; ++k) acc -= a[i * s + k] * x[k];
            x[i] = acc / a[i * s + i];
        }
    }
    if (tid == 0) status[0] = 0;
}

cudaError_t launch_cholesky(const double* G, long ldg, int s, int NP, double* R, double* RinvT,
                            int* status, double tol, cudaStream_t st) {
    const size_t smem = (size_t)s * s * sizeof(double);
    if (smem > 225 * 1024) return cudaErrorInvalidValue;
    cudaError_t e =
        cudaFuncSetAttribute(cholesky_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cholesky_kernel<<<1, 512, smem, st>>>(G, ldg, s, NP, R, RinvT, status, tol);
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
// The sweep visits all pairs in round-robin (tournament) order so that the s/2
// pairs of a round run concurrently, one warp per pair; a sweep with no rotation
// ends the iteration (svd.cpp:196-199); more than 30 sweeps is a convergence
// failure (svd.hpp:20).  Columns are stored contiguously (column-major) in smem;
// the rotation accumulator J lives in smem when it fits, else in global scratch.
constexpr int kJacobiThreads = 512;
constexpr int kMaxSweeps = 30;

__device__ __forceinline__ int rr_index(int slot, int round, int sp) {
    return slot == 0 ? 0 : 1 + (slot - 1 + round) % (sp - 1);
}

__global__ void __launch_bounds__(kJacobiThreads) jacobi_kernel(
    const double* __restrict__ Rin, int s, int NP, double* __restrict__ sigma_out,
    double* __restrict__ Uout, double* __restrict__ Wout, int* __restrict__ status,
    double* __restrict__ Jglobal) {
    extern __shared__ double sh[];
    double* Rc = sh;                                  // s columns of length s
    double* J = Jglobal ? Jglobal : sh + s * s;       // s columns of length s
    __shared__ int rotations;
    __shared__ double abs_thresh;
    __shared__ double norms[288];
    __shared__ int order[288];
    const int tid = threadIdx.x, nth = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;

    for (int e = tid; e < s * s; e += nth) {
        const int c = e / s, r = e % s;
        Rc[e] = Rin[r * NP + c];
        J[e] = (r == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
        double acc = 0.0;
        for (int e = lane; e < s * s; e += 32) acc += Rc[e] * Rc[e];
        acc = warp_sum(acc);
        if (lane == 0) abs_thresh = 1e-14 * acc;
    }
    __syncthreads();

    const int sp = (s + 1) & ~1;  // even number of tournament slots (slot s is a bye)
    int sweeps = 0;
    bool converged = false;
    while (sweeps < kMaxSweeps) {
        ++sweeps;
        if (tid == 0) rotations = 0;
        __syncthreads();
        for (int round = 0; round < sp - 1; ++round) {
            for (int k = warp; k < sp / 2; k += nwarps) {
                int i = rr_index(k, round, sp), j = rr_index(sp - 1 - k, round, sp);
                if (i > j) { const int tmp = i; i = j; j = tmp; }
                if (j >= s) continue;
                double* ci = Rc + i * s;
                double* cj = Rc + j * s;
                double aii = 0.0, ajj = 0.0, d = 0.0;
                for (int r = lane; r < s; r += 32) {
                    const double x = ci[r], y = cj[r];
                    aii += x * x;
                    ajj += y * y;
                    d += x * y;
                }
                aii = warp_sum(aii);
                ajj = warp_sum(ajj);
                d = warp_sum(d);
                if (fabs(d) <= abs_thresh && d * d <= (1e-13 * 1e-13) * aii * ajj) continue;
                const double zeta = (ajj - aii) / (2.0 * d);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double sn = c * t;
                for (int r = lane; r < s; r += 32) {
                    const double x = ci[r], y = cj[r];
                    ci[r] = c * x - sn * y;
                    cj[r] = sn * x + c * y;
                }
                double* ji = J + i * s;
                double* jj = J + j * s;
                for (int r = lane; r < s; r += 32) {
                    const double x = ji[r], y = jj[r];
                    ji[r] = c * x - sn * y;
                    jj[r] = sn * x + c * y;
                }
                if (lane == 0) atomicAdd(&rotations, 1);
            }
            __syncthreads();
        }
        const int rot = rotations;
        __syncthreads();
        if (rot == 0) {
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
        for (int r = lane; r < s; r += 32) acc += Rc[c * s + r] * Rc[c * s + r];
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
            u = sg > 0.0 ? Rc[src * s + r] / sg : 0.0;
            w = J[src * s + r];
        }
        Uout[e] = u;
        Wout[e] = w;
    }
    for (int c = tid; c < s; c += nth) sigma_out[c] = norms[order[c]];
    if (tid == 0) status[0] = sweeps;
}

size_t jacobi_max_width() { return 288; }

cudaError_t launch_jacobi_svd(const double* R, int s, int NP, double* sigma, double* U, double* W,
                              int* status, cudaStream_t st) {
    if (s > (int)jacobi_max_width()) return cudaErrorInvalidValue;
    const size_t one = (size_t)s * s * sizeof(double);
    double* jglobal = nullptr;
    size_t smem = 2 * one;
    if (smem > 200 * 1024) {  // keep J in global memory (L2 resident)
        smem = one;
        if (smem > 200 * 1024) return cudaErrorInvalidValue;
        cudaError_t e = cudaMallocAsync(&jglobal, one, st);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e =
        cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    jacobi_kernel<<<1, kJacobiThreads, smem, st>>>(R, s, NP, sigma, U, W, status, jglobal);
    e = cudaGetLastError();
    if (jglobal) cudaFreeAsync(jglobal, st);
    return e;
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
