// Small dense linear algebra beyond one CTA: the blocked Cholesky's pieces for s > ~150 (an
// s x s FP64 matrix no longer fits one CTA's shared memory: s = 272 is 592 KB) and the
// multi-CTA block Jacobi, used for every s > 64 (more SMs, 8 warps each, beat one CTA's
// 32 IPC-bound warps):
//   * small_gemm_kernel — generic C = alpha op(A) op(B) + beta Cin on s-sized
//     operands (tiles of 16 x 16 per CTA), the building block of the blocked Cholesky
//     that rsvd_b200.cpp assembles from two in-smem Cholesky factorisations;
//   * block_jacobi_kernel — one-sided block Jacobi SVD of the s x s triangular factor
//     R_B, the wide-sketch twin of jacobi_kernel (linalg_small.cu). Columns live in
//     global memory (L2 resident); the s/8 column blocks are paired in round-robin
//     (tournament) order, each block pair is one CTA that loads its 16 columns into
//     shared memory (cp.async) and rotates the 64 cross-block pairs (the first round of a
//     sweep also every within-block pair) with the
//     reference's rotation rule and skip thresholds (svd.cpp:35-36, 60-90); a grid-wide
//     barrier (cooperative launch) separates rounds. A sweep without any rotation ends
//     the iteration, more than 30 sweeps is a convergence failure (svd.hpp:20), and the
//     final sort / U / W extraction matches jacobi_kernel.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace rsvdb200 {

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)),
                 "l"(gmem_src)
                 : "memory");
}

// ============================================================== small GEMM
// C (M x N, ldc) = alpha * op(A) op(B) + beta * Cin (ldcin); op(A) is M x K,
// op(B) K x N; ta / tb: the operand is stored transposed (row-major K x M / N x K).
// Cin may alias C (each element is read before it is written by the same thread).
// 16 x 16 output tiles (one output per thread, so an s = 136 block spans 81 CTAs), K in chunks
// of up to 144; both operand tiles are loaded along their contiguous dimension whatever the
// transposition (coalesced), and transposed on the way into shared memory.
__global__ void __launch_bounds__(256) small_gemm_kernel(int M, int N, int K, double alpha,
                                                         const double* __restrict__ A, long lda,
                                                         bool ta, const double* __restrict__ B,
                                                         long ldb, bool tb, double beta,
                                                         const double* Cin, long ldcin,
                                                         double* C, long ldc) {
    // K in chunks of up to 144 (the blocked Cholesky's 136-wide products in one chunk: one
    // load phase and one barrier instead of five 32-wide rounds), two accumulators
    constexpr int KC = 144;
    __shared__ double As[16][KC + 1];  // As[r][k] = op(A)[i0 + r][k0 + k]
    __shared__ double Bs[KC][17];      // Bs[k][c] = op(B)[k0 + k][j0 + c]
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int i0 = blockIdx.y * 16, j0 = blockIdx.x * 16;
    double acc0 = 0.0, acc1 = 0.0;
    for (int k0 = 0; k0 < K; k0 += KC) {
        const int kc = min(KC, K - k0);
        // both operands loaded along their contiguous dimension (coalesced)
        for (int e = tid; e < 16 * kc; e += 256) {
            int r, k;
            if (ta) { k = e >> 4; r = e & 15; } else { r = e / kc; k = e - r * kc; }
            const int i = i0 + r, kk = k0 + k;
            As[r][k] = i < M ? (ta ? A[(long)kk * lda + i] : A[(long)i * lda + kk]) : 0.0;
            int c, kb;
            if (tb) { c = e / kc; kb = e - c * kc; } else { kb = e >> 4; c = e & 15; }
            const int j = j0 + c, kj = k0 + kb;
            Bs[kb][c] = j < N ? (tb ? B[(long)j * ldb + kj] : B[(long)kj * ldb + j]) : 0.0;
        }
        __syncthreads();
        int kk = 0;
        for (; kk + 1 < kc; kk += 2) {
            acc0 = fma(As[ty][kk], Bs[kk][tx], acc0);
            acc1 = fma(As[ty][kk + 1], Bs[kk + 1][tx], acc1);
        }
        if (kk < kc) acc0 = fma(As[ty][kk], Bs[kk][tx], acc0);
        __syncthreads();
    }
    const int i = i0 + ty, j = j0 + tx;
    if (i < M && j < N) {
        double v = alpha * (acc0 + acc1);
        if (beta != 0.0) v += beta * Cin[(long)i * ldcin + j];
        C[(long)i * ldc + j] = v;
    }
}

cudaError_t launch_small_gemm(int M, int N, int K, double alpha, const double* A, long lda,
                              bool ta, const double* B, long ldb, bool tb, double beta,
                              const double* Cin, long ldcin, double* C, long ldc,
                              cudaStream_t st) {
    if (M <= 0 || N <= 0) return cudaSuccess;
    dim3 grid((unsigned)((N + 15) / 16), (unsigned)((M + 15) / 16));
    small_gemm_kernel<<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, ta, B, ldb, tb, beta,
                                            Cin ? Cin : C, Cin ? ldcin : ldc, C, ldc);
    return cudaGetLastError();
}

// ========================================================= block Jacobi SVD
constexpr int kBJW = 8;           // columns per block
constexpr int kBJThreads = 256;   // 8 warps: one per column pair of an inner round
constexpr int kBJMaxSweeps = 30;

__device__ __forceinline__ int bj_rr(int slot, int round, int sp) {
    return slot == 0 ? 0 : 1 + (slot - 1 + round) % (sp - 1);
}

__host__ __device__ inline int bj_ld(int s) { return (s + 1) & ~1; }  // column stride

// scratch: Rc (s columns, stride bj_ld(s)), J (same), sweep flags (32 ints), norms (s)
template <int NQ>
__global__ void __launch_bounds__(kBJThreads, 1) block_jacobi_kernel(
    const double* __restrict__ Rin, int s, int NP, double* __restrict__ sigma_out,
    double* __restrict__ Uout, double* __restrict__ Wout, int* __restrict__ status,
    double* __restrict__ scratch, const int* __restrict__ abort_flag) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double sh[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nb = (s + kBJW - 1) / kBJW;
    const int sp = (nb + 1) & ~1;
    const int ls = bj_ld(s), l2 = ls / 2;  // column stride in doubles / double2
    double* Rc = scratch;
    double* J = Rc + (size_t)s * ls;
    int* sweep_flag = reinterpret_cast<int*>(J + (size_t)s * ls);
    double* norms = J + (size_t)s * ls + 16;
    __shared__ double red[32];
    __shared__ double scale_sh, athr_sh;
    __shared__ int order_sh[320];
    if (abort_flag && *abort_flag) {  // uniform over the grid
        if (blockIdx.x == 0 && tid == 0) status[0] = 0;
        return;
    }
    // power-of-two scale and the absolute threshold, computed redundantly per CTA (same
    // order everywhere, so every CTA holds identical values)
    {
        double mx = 0.0;
        for (int e = tid; e < s * s; e += kBJThreads) mx = fmax(mx, fabs(Rin[(e / s) * NP + e % s]));
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) red[warp] = mx;
        __syncthreads();
        if (tid == 0) {
            double m = 0.0;
            for (int w = 0; w < kBJThreads / 32; ++w) m = fmax(m, red[w]);
            int ex = 0;
            frexp(m, &ex);
            scale_sh = m > 0.0 ? ldexp(1.0, -ex) : 1.0;
        }
        __syncthreads();
        const double sc = scale_sh;
        double acc = 0.0;
        for (int e = tid; e < s * s; e += kBJThreads) {
            const double x = Rin[(e / s) * NP + e % s] * sc;
            acc = fma(x, x, acc);
        }
        acc = warp_sum(acc);
        __syncthreads();
        if (lane == 0) red[warp] = acc;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < kBJThreads / 32; ++w) t += red[w];
            athr_sh = 1e-14 * t;
        }
        __syncthreads();
    }
    const double scale = scale_sh, athr = athr_sh;
    for (long e = blockIdx.x * (long)kBJThreads + tid; e < (long)s * ls;
         e += (long)gridDim.x * kBJThreads) {
        const int c = (int)(e / ls), r = (int)(e % ls);
        Rc[e] = r < s ? Rin[(long)r * NP + c] * scale : 0.0;
        J[e] = (r == c) ? 1.0 : 0.0;
    }
    if (blockIdx.x == 0 && tid < 32) sweep_flag[tid] = 0;
    grid.sync();

    double2* C = reinterpret_cast<double2*>(sh);          // 2*kBJW columns, stride l2
    double2* Jl = C + 2 * kBJW * l2;                       // their rotation accumulators
    const double2* Rc2 = reinterpret_cast<const double2*>(Rc);
    const double2* J2 = reinterpret_cast<const double2*>(J);
    __shared__ int cols[2 * kBJW];
    int sweeps = 0;
    bool converged = false;
    while (sweeps < kBJMaxSweeps) {
        ++sweeps;
        for (int round = 0; round < sp - 1; ++round) {
            const int k = blockIdx.x;
            int bi = bj_rr(k, round, sp), bj = bj_rr(sp - 1 - k, round, sp);
            if (bi > bj) { const int t = bi; bi = bj; bj = t; }
            int cnt = 0;
            // a block paired with the bye slot (bj == nb, odd block count) still sweeps its
            // own pairs — with a single block that is the whole matrix
            if (k < sp / 2 && bi < nb) {
                const int e0 = min(s, (bi + 1) * kBJW);
                const int e1 = bj < nb ? min(s, (bj + 1) * kBJW) : bj * kBJW;
                cnt = (e0 - bi * kBJW) + (e1 - bj * kBJW);
                if (tid < cnt) {
                    const int n0 = e0 - bi * kBJW;
                    cols[tid] = tid < n0 ? bi * kBJW + tid : bj * kBJW + (tid - n0);
                }
            }
            __syncthreads();
            int rotated = 0;
            if (cnt > 0) {
                // columns in: every 16-byte piece as its own cp.async (L2 -> shared, no register
                // staging), all in flight at once; the scratch was written by other CTAs before
                // the last grid barrier, and .cg reads it from L2
                for (int l = warp; l < cnt; l += kBJThreads / 32) {
                    const long src = (long)cols[l] * l2;
                    for (int r = lane; r < l2; r += 32) {
                        cp_async16(C + l * l2 + r, Rc2 + src + r);
                        cp_async16(Jl + l * l2 + r, J2 + src + r);
                    }
                }
                asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
                __syncthreads();
                // The first round of a sweep visits every pair of the CTA's 16 columns (so each
                // block's own pairs are covered once per sweep); later rounds only the 8 x 8
                // pairs across the two blocks: 8 inner rounds instead of 15, warp w pairs
                // column w of the first block with column (w + ir) mod 8 of the second.
                const int spl = (cnt + 1) & ~1;
                const bool full = round == 0;
                const int n0 = min(s, (bi + 1) * kBJW) - bi * kBJW;
                const int inner = full ? spl - 1 : kBJW;
                for (int ir = 0; ir < inner; ++ir) {
                    const int pk = warp;
                    bool live;
                    int i = 0, j = 0;
                    if (full) {
                        live = pk < spl / 2;
                        if (live) {
                            i = bj_rr(pk, ir, spl);
                            j = bj_rr(spl - 1 - pk, ir, spl);
                            if (i > j) { const int t = i; i = j; j = t; }
                            live = j < cnt;
                        }
                    } else {
                        i = pk;
                        j = n0 + (pk + ir) % kBJW;
                        live = i < n0 && j < cnt;
                    }
                    if (live) {  // warp-uniform
                        double2* ci = C + i * l2;
                        double2* cj = C + j * l2;
                        double2 xi[NQ], xj[NQ];
                        double aii = 0.0, ajj = 0.0, d = 0.0;
#pragma unroll
                        for (int q = 0; q < NQ; ++q) {
                            const int r = lane + 32 * q;
                            xi[q] = r < l2 ? ci[r] : make_double2(0.0, 0.0);
                            xj[q] = r < l2 ? cj[r] : make_double2(0.0, 0.0);
                            aii = fma(xi[q].x, xi[q].x, fma(xi[q].y, xi[q].y, aii));
                            ajj = fma(xj[q].x, xj[q].x, fma(xj[q].y, xj[q].y, ajj));
                            d = fma(xi[q].x, xj[q].x, fma(xi[q].y, xj[q].y, d));
                        }
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            aii += __shfl_xor_sync(0xffffffffu, aii, o);
                            ajj += __shfl_xor_sync(0xffffffffu, ajj, o);
                            d += __shfl_xor_sync(0xffffffffu, d, o);
                        }
                        if (!(fabs(d) <= athr && d * d <= (1e-13 * 1e-13) * aii * ajj)) {
                            const double diff = ajj - aii;
                            const double sgn =
                                ((diff >= 0.0) == (d >= 0.0)) || diff == 0.0 ? 1.0 : -1.0;
                            const double t = sgn * 2.0 * fabs(d) /
                                             (fabs(diff) + sqrt(fma(diff, diff, 4.0 * d * d)));
                            const double c = rsqrt(fma(t, t, 1.0));
                            const double sn = c * t;
                            double2* wi = Jl + i * l2;
                            double2* wj = Jl + j * l2;
#pragma unroll
                            for (int q = 0; q < NQ; ++q) {
                                const int r = lane + 32 * q;
                                if (r < l2) {
                                    const double2 yi = wi[r], yj = wj[r];
                                    ci[r] = make_double2(c * xi[q].x - sn * xj[q].x,
                                                         c * xi[q].y - sn * xj[q].y);
                                    cj[r] = make_double2(sn * xi[q].x + c * xj[q].x,
                                                         sn * xi[q].y + c * xj[q].y);
                                    wi[r] = make_double2(c * yi.x - sn * yj.x, c * yi.y - sn * yj.y);
                                    wj[r] = make_double2(sn * yi.x + c * yj.x, sn * yi.y + c * yj.y);
                                }
                            }
                            rotated = 1;
                        }
                    }
                    __syncthreads();
                }
                double2* Rcw = reinterpret_cast<double2*>(Rc);
                double2* Jw = reinterpret_cast<double2*>(J);
                for (int l = warp; l < cnt; l += kBJThreads / 32) {
                    const long dst = (long)cols[l] * l2;
                    for (int r = lane; r < l2; r += 32) {
                        Rcw[dst + r] = C[l * l2 + r];
                        Jw[dst + r] = Jl[l * l2 + r];
                    }
                }
            }
            if (__syncthreads_or(rotated) && tid == 0) atomicOr(&sweep_flag[sweeps - 1], 1);
            grid.sync();
        }
        if (*((volatile int*)&sweep_flag[sweeps - 1]) == 0) {
            converged = true;
            break;
        }
    }
    if (!converged) {
        if (blockIdx.x == 0 && tid == 0) status[0] = -1;
        return;
    }
    // column norms (grid-stride), then every CTA derives the same stable descending order
    for (int c = blockIdx.x * (kBJThreads / 32) + warp; c < s; c += gridDim.x * (kBJThreads / 32)) {
        double acc = 0.0;
        for (int r = lane; r < s; r += 32) acc = fma(Rc[(long)c * ls + r], Rc[(long)c * ls + r], acc);
        acc = warp_sum(acc);
        if (lane == 0) norms[c] = sqrt(acc);
    }
    grid.sync();
    for (int c = tid; c < s; c += kBJThreads) {
        const double nc = norms[c];
        int rank = 0;
        for (int o = 0; o < s; ++o) {
            const double no = norms[o];
            rank += (no > nc) || (no == nc && o < c);
        }
        order_sh[rank] = c;
    }
    __syncthreads();
    for (long e = blockIdx.x * (long)kBJThreads + tid; e < (long)NP * NP;
         e += (long)gridDim.x * kBJThreads) {
        const int r = (int)(e / NP), cc = (int)(e % NP);
        double u = 0.0, w = 0.0;
        if (r < s && cc < s) {
            const int src = order_sh[cc];
            const double sg = norms[src];
            u = sg > 0.0 ? Rc[(long)src * ls + r] / sg : 0.0;
            w = J[(long)src * ls + r];
        }
        Uout[e] = u;
        Wout[e] = w;
    }
    if (blockIdx.x == 0) {
        for (int c = tid; c < NP; c += kBJThreads)
            sigma_out[c] = c < s ? norms[order_sh[c]] / scale : 0.0;
        if (tid == 0) status[0] = sweeps;
    }
}

size_t block_jacobi_scratch_doubles(int s) {
    return 2 * (size_t)s * bj_ld(s) + 16 + (size_t)s + 16;
}

template <int NQ>
static cudaError_t launch_bj(const double* R, int s, int NP, double* sigma, double* U, double* W,
                             int* status, double* scratch, const int* abort_flag, cudaStream_t st) {
    const size_t smem = 2 * (size_t)(2 * kBJW) * bj_ld(s) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(block_jacobi_kernel<NQ>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int nb = (s + kBJW - 1) / kBJW;
    const int sp = (nb + 1) & ~1;
    void* args[] = {(void*)&R, (void*)&s, (void*)&NP, (void*)&sigma, (void*)&U, (void*)&W,
                    (void*)&status, (void*)&scratch, (void*)&abort_flag};
    e = cudaLaunchCooperativeKernel((void*)block_jacobi_kernel<NQ>, dim3(sp / 2), dim3(kBJThreads),
                                    args, smem, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_block_jacobi_svd(const double* R, int s, int NP, double* sigma, double* U,
                                    double* W, int* status, double* scratch,
                                    const int* abort_flag, cudaStream_t st) {
    if (s > 320) return cudaErrorInvalidValue;
    // row pairs per lane (one warp per column pair)
    switch ((bj_ld(s) / 2 + 31) / 32) {
        case 1: return launch_bj<1>(R, s, NP, sigma, U, W, status, scratch, abort_flag, st);
        case 2: return launch_bj<2>(R, s, NP, sigma, U, W, status, scratch, abort_flag, st);
        case 3: return launch_bj<3>(R, s, NP, sigma, U, W, status, scratch, abort_flag, st);
        case 4: return launch_bj<4>(R, s, NP, sigma, U, W, status, scratch, abort_flag, st);
        default: return launch_bj<5>(R, s, NP, sigma, U, W, status, scratch, abort_flag, st);
    }
}

}  // namespace rsvdb200
