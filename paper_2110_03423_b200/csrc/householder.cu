// Robust paths of the rSVD on B200:
//
//  * the Householder QR fallback of CholeskyQR2 — a restatement of the reference's
//    unblocked Householder QR (qr.cpp:27-102): reflector v ~ x + sign(x_1)||x|| e_1
//    per column, applied to the trailing columns, thin Q accumulated backwards from
//    the identity, then diag(R) >= 0 by flipping R rows / Q columns. Each CTA owns a
//    contiguous row slab; every reduction is a fixed-order sum over per-CTA partials,
//    so the result is deterministic. Two launches per column (factorisation) and two
//    per column (Q accumulation); it only runs on ill-conditioned input.
//
//  * complete_basis_kernel — the reference's deterministic orthonormal completion
//    (svd.cpp:111-151): for each missing column, canonical vectors e_t are tried in
//    ascending order of row load (sum of squares of the row over the valid columns,
//    ties by index, i.e. the stable sort of svd.cpp:126-130), orthogonalised by two
//    modified Gram-Schmidt passes and accepted when the remaining norm >= 1e-4.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace rsvdb200 {

constexpr int kHHThreads = 256;
constexpr int kHHWarps = kHHThreads / 32;
constexpr int kMaxCh = 9;  // up to 288 columns, 32 per lane-chunk
constexpr int kMaxCols = 32 * kMaxCh;

// Block-wide partial sums of sum_{rows i in [lo,hi)} x_i * w[i][j] for j in [j0, s),
// x_i given by a functor; written to out[j].
template <typename XF>
__device__ void block_col_dots(const double* __restrict__ w, long ld, long lo, long hi, int j0,
                               int s, XF xval, double* __restrict__ out /* [s] */,
                               double* __restrict__ red /* smem kHHWarps x kMaxCols */) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double acc[kMaxCh];
#pragma unroll
    for (int c = 0; c < kMaxCh; ++c) acc[c] = 0.0;
    for (long i = lo + warp; i < hi; i += kHHWarps) {
        const double x = xval(i);
        const double* row = w + i * ld;
#pragma unroll
        for (int c = 0; c < kMaxCh; ++c) {
            const int j = j0 + lane + 32 * c;
            if (j < s) acc[c] += x * row[j];
        }
    }
#pragma unroll
    for (int c = 0; c < kMaxCh; ++c) {
        const int j = j0 + lane + 32 * c;
        if (j < s) red[warp * kMaxCols + j] = acc[c];
    }
    __syncthreads();
    for (int j = j0 + threadIdx.x; j < s; j += blockDim.x) {
        double t = 0.0;
        for (int q = 0; q < kHHWarps; ++q) t += red[q * kMaxCols + j];
        out[j] = t;
    }
    __syncthreads();
}

// The factorisation is a sequence of ordinary launches (two per column, one grid-wide
// reduction each), so no grid-wide barrier or co-residency assumption is needed.
// Partial sums live in part[block][0..NP-1] (column dots) and part[block][NP] (tail
// norm^2); every block re-reduces the partials in the same fixed order, so all blocks
// derive bit-identical reflectors.
struct HH {
    const double* Y;
    long M;
    int s;
    long ldy;
    double* Q;
    long ldq;
    double* R;
    int NP;
    double* work;  // M x NP row-major working copy
    double* refl;  // M x NP reflector columns
    double* part;  // nb x (NP + 2)
    int* act;      // NP
};

__device__ __forceinline__ void hh_rows(const HH& h, long& lo, long& hi) {
    const long rpb = (h.M + gridDim.x - 1) / gridDim.x;
    lo = blockIdx.x * rpb;
    hi = min(h.M, lo + rpb);
}

// tail norm^2 of column k (rows > k) into slot NP + (k & 1): consecutive columns use
// different slots, so a launch never overwrites a value another block may still read.
__device__ void hh_tail_norm(const HH& h, int k, long lo, long hi, double* red) {
    double acc = 0.0;
    for (long i = max(lo, (long)k + 1) + threadIdx.x; i < hi; i += blockDim.x) {
        const double x = h.work[i * h.NP + k];
        acc += x * x;
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < kHHWarps; ++q) t += red[q];
        h.part[blockIdx.x * (h.NP + 2) + h.NP + (k & 1)] = t;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kHHThreads) hh_init_kernel(HH h) {
    __shared__ double red[kHHWarps];
    long lo, hi;
    hh_rows(h, lo, hi);
    for (long i = lo; i < hi; ++i)
        for (int j = threadIdx.x; j < h.NP; j += blockDim.x) {
            h.work[i * h.NP + j] = j < h.s ? h.Y[i * h.ldy + j] : 0.0;
            h.refl[i * h.NP + j] = 0.0;
        }
    __syncthreads();
    hh_tail_norm(h, 0, lo, hi, red);
}

// column k, phase A: reflector v_k (qr.cpp:44-58) and partial dots v_k . w_j, j > k
__global__ void __launch_bounds__(kHHThreads) hh_col_a_kernel(HH h, int k) {
    __shared__ double red[kHHWarps * kMaxCols];
    long lo, hi;
    hh_rows(h, lo, hi);
    const int NP = h.NP;
    double tail2 = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) tail2 += h.part[b * (NP + 2) + NP + (k & 1)];
    const double x0 = h.work[(long)k * NP + k];
    const double norm_x = sqrt(tail2 + x0 * x0);
    if (norm_x == 0.0) {  // zero column: H_k = I, r_kk = 0 (qr.cpp:47)
        if (blockIdx.x == 0 && threadIdx.x == 0) h.act[k] = 0;
        return;
    }
    const double sign = x0 >= 0.0 ? 1.0 : -1.0;
    const double alpha = x0 + sign * norm_x;
    const double inv_nv = 1.0 / sqrt(tail2 + alpha * alpha);
    if (blockIdx.x == 0 && threadIdx.x == 0) h.act[k] = 1;
    for (long i = max(lo, (long)k) + threadIdx.x; i < hi; i += blockDim.x)
        h.refl[i * NP + k] = (i == k ? alpha : h.work[i * NP + k]) * inv_nv;
    __syncthreads();
    block_col_dots(h.work, NP, max(lo, (long)k), hi, k + 1, h.s,
                   [&](long i) { return h.refl[i * NP + k]; }, h.part + blockIdx.x * (NP + 2), red);
}

// column k, phase B: w_j -= 2 (v.w_j) v for j > k, r_kk, tail norm of column k + 1
__global__ void __launch_bounds__(kHHThreads) hh_col_b_kernel(HH h, int k) {
    __shared__ double dj[kMaxCols];
    __shared__ double red[kHHWarps];
    long lo, hi;
    hh_rows(h, lo, hi);
    const int NP = h.NP;
    const bool active = h.act[k] != 0;
    if (active) {
        for (int j = k + 1 + threadIdx.x; j < h.s; j += blockDim.x) {
            double t = 0.0;
            for (unsigned b = 0; b < gridDim.x; ++b) t += h.part[b * (NP + 2) + j];
            dj[j] = 2.0 * t;
        }
        double tail2 = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) tail2 += h.part[b * (NP + 2) + NP + (k & 1)];
        __syncthreads();
        for (long i = max(lo, (long)k); i < hi; ++i) {
            const double vi = h.refl[i * NP + k];
            for (int j = k + 1 + threadIdx.x; j < h.s; j += blockDim.x)
                h.work[i * NP + j] -= dj[j] * vi;
        }
        if (k >= lo && k < hi && threadIdx.x == 0) {
            const double x0 = h.work[(long)k * NP + k];
            const double norm_x = sqrt(tail2 + x0 * x0);
            h.work[(long)k * NP + k] = -(x0 >= 0.0 ? 1.0 : -1.0) * norm_x;
        }
        __syncthreads();
    }
    if (k + 1 < h.s) hh_tail_norm(h, k + 1, lo, hi, red);
}

__global__ void __launch_bounds__(kHHThreads) hh_q_init_kernel(HH h) {
    long lo, hi;
    hh_rows(h, lo, hi);
    for (long i = lo; i < hi; ++i)
        for (int j = threadIdx.x; j < h.NP; j += blockDim.x)
            h.Q[i * h.ldq + j] = (i == j && j < h.s) ? 1.0 : 0.0;
}

// backward accumulation (qr.cpp:71-84), reflector kk: partial dots, then the update
__global__ void __launch_bounds__(kHHThreads) hh_q_a_kernel(HH h, int kk) {
    __shared__ double red[kHHWarps * kMaxCols];
    if (!h.act[kk]) return;
    long lo, hi;
    hh_rows(h, lo, hi);
    block_col_dots(h.Q, h.ldq, max(lo, (long)kk), hi, kk, h.s,
                   [&](long i) { return h.refl[i * h.NP + kk]; },
                   h.part + blockIdx.x * (h.NP + 2), red);
}

__global__ void __launch_bounds__(kHHThreads) hh_q_b_kernel(HH h, int kk) {
    __shared__ double dj[kMaxCols];
    if (!h.act[kk]) return;
    long lo, hi;
    hh_rows(h, lo, hi);
    const int NP = h.NP;
    for (int j = kk + threadIdx.x; j < h.s; j += blockDim.x) {
        double t = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) t += h.part[b * (NP + 2) + j];
        dj[j] = 2.0 * t;
    }
    __syncthreads();
    for (long i = max(lo, (long)kk); i < hi; ++i) {
        const double vi = h.refl[i * NP + kk];
        for (int j = kk + threadIdx.x; j < h.s; j += blockDim.x) h.Q[i * h.ldq + j] -= dj[j] * vi;
    }
}

// diag(R) >= 0 (qr.cpp:86-93): flip R rows / Q columns; R written from the owned rows
__global__ void __launch_bounds__(kHHThreads) hh_finish_kernel(HH h) {
    long lo, hi;
    hh_rows(h, lo, hi);
    const int NP = h.NP;
    for (long i = lo; i < hi && i < NP; ++i)
        for (int j = threadIdx.x; j < NP; j += blockDim.x) {
            double r = (i < h.s && j < h.s && j >= i) ? h.work[i * NP + j] : 0.0;
            if (i < h.s && h.work[i * NP + i] < 0.0) r = -r;
            h.R[i * NP + j] = r;
        }
    for (long i = lo; i < hi; ++i)
        for (int j = threadIdx.x; j < h.s; j += blockDim.x)
            if (h.work[(long)j * NP + j] < 0.0) h.Q[i * h.ldq + j] = -h.Q[i * h.ldq + j];
}

size_t householder_work_doubles(long M, int s) {
    const int NP = kMaxCols;
    (void)s;
    return 2 * (size_t)M * NP + 2 * 296 * (size_t)(NP + 2) + NP + 64;
}

cudaError_t launch_householder_qr(const double* Y, long M, int s, long ldy, double* Qout, long ldq,
                                  double* R, int NP, double* work, cudaStream_t st) {
    if (s > kMaxCols || NP > kMaxCols) return cudaErrorInvalidValue;
    const unsigned nb = (unsigned)std::max(1L, std::min(296L, M));
    HH h;
    h.Y = Y;
    h.M = M;
    h.s = s;
    h.ldy = ldy;
    h.Q = Qout;
    h.ldq = ldq;
    h.R = R;
    h.NP = NP;
    h.work = work;
    h.refl = work + (size_t)M * NP;
    h.part = h.refl + (size_t)M * NP;
    h.act = reinterpret_cast<int*>(h.part + (size_t)nb * (NP + 2));
    cudaError_t e = cudaMemsetAsync(R, 0, (size_t)NP * NP * sizeof(double), st);
    if (e != cudaSuccess) return e;
    hh_init_kernel<<<nb, kHHThreads, 0, st>>>(h);
    for (int k = 0; k < s; ++k) {
        hh_col_a_kernel<<<nb, kHHThreads, 0, st>>>(h, k);
        hh_col_b_kernel<<<nb, kHHThreads, 0, st>>>(h, k);
    }
    hh_q_init_kernel<<<nb, kHHThreads, 0, st>>>(h);
    for (int kk = s - 1; kk >= 0; --kk) {
        hh_q_a_kernel<<<nb, kHHThreads, 0, st>>>(h, kk);
        hh_q_b_kernel<<<nb, kHHThreads, 0, st>>>(h, kk);
    }
    hh_finish_kernel<<<nb, kHHThreads, 0, st>>>(h);
    return cudaGetLastError();
}

// ========================================================= orthonormal completion
__global__ void __launch_bounds__(1024) complete_basis_kernel(
    double* __restrict__ U, long rows, long ld, int s, const double* __restrict__ sigma,
    long null_dim, double* __restrict__ work, int* __restrict__ status,
    const int* __restrict__ abort_flag) {
    double* load = work;         // rows
    double* cand = work + rows;  // rows
    unsigned char* tried = reinterpret_cast<unsigned char*>(work + 2 * rows);
    __shared__ double sv[32];
    __shared__ long si[32];
    __shared__ double bcast;
    __shared__ long bidx;
    const int tid = threadIdx.x, nth = blockDim.x, warp = tid >> 5, lane = tid & 31;
    if (abort_flag && *abort_flag) return;
    // null block of the small SVD (svd.cpp:221-234)
    const double null_thresh = sigma[0] * (double)null_dim * 2.220446049250313e-16;
    int r0 = s;
    for (int j = 0; j < s; ++j)
        if (!(sigma[j] > null_thresh)) {
            r0 = j;
            break;
        }
    const int r1 = s;
    if (r0 >= r1) {
        if (tid == 0) status[0] = 0;
        return;
    }
    auto block_sum = [&](double v) {
        v = warp_sum(v);
        if (lane == 0) sv[warp] = v;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int q = 0; q < nth / 32; ++q) t += sv[q];
            bcast = t;
        }
        __syncthreads();
        const double r = bcast;
        __syncthreads();
        return r;
    };
    for (int slot = r0; slot < r1; ++slot) {
        for (long r = tid; r < rows; r += nth) {
            double acc = 0.0;
            for (int c = 0; c < slot; ++c) acc += U[r * ld + c] * U[r * ld + c];
            load[r] = acc;
            tried[r] = 0;
        }
        __syncthreads();
        bool placed = false;
        for (long attempt = 0; attempt < rows && !placed; ++attempt) {
            // next untried row with the smallest load (first index on ties)
            double best = 1e308;
            long arg = -1;
            for (long r = tid; r < rows; r += nth)
                if (!tried[r] && (load[r] < best || (load[r] == best && r < arg))) {
                    best = load[r];
                    arg = r;
                }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_down_sync(0xffffffffu, best, o);
                const long oa = __shfl_down_sync(0xffffffffu, arg, o);
                if (oa >= 0 && (arg < 0 || ob < best || (ob == best && oa < arg))) {
                    best = ob;
                    arg = oa;
                }
            }
            if (lane == 0) {
                sv[warp] = best;
                si[warp] = arg;
            }
            __syncthreads();
            if (tid == 0) {
                double b = sv[0];
                long a = si[0];
                for (int q = 1; q < nth / 32; ++q)
                    if (si[q] >= 0 && (a < 0 || sv[q] < b || (sv[q] == b && si[q] < a))) {
                        b = sv[q];
                        a = si[q];
                    }
                bidx = a;
                if (a >= 0) tried[a] = 1;
            }
            __syncthreads();
            const long t = bidx;
            if (t < 0) break;
            for (long r = tid; r < rows; r += nth) cand[r] = (r == t) ? 1.0 : 0.0;
            __syncthreads();
            for (int pass = 0; pass < 2; ++pass)
                for (int c = 0; c < slot; ++c) {
                    double acc = 0.0;
                    for (long r = tid; r < rows; r += nth) acc += cand[r] * U[r * ld + c];
                    const double d = block_sum(acc);
                    for (long r = tid; r < rows; r += nth) cand[r] -= d * U[r * ld + c];
                    __syncthreads();
                }
            double acc = 0.0;
            for (long r = tid; r < rows; r += nth) acc += cand[r] * cand[r];
            const double nrm = sqrt(block_sum(acc));
            if (nrm >= 1e-4) {
                for (long r = tid; r < rows; r += nth) U[r * ld + slot] = cand[r] / nrm;
                placed = true;
            }
            __syncthreads();
        }
        if (!placed) {
            if (tid == 0) status[0] = 1;
            return;
        }
    }
    if (tid == 0) status[0] = 0;
}

size_t complete_basis_work_doubles(long rows) { return 2 * (size_t)rows + (size_t)rows / 8 + 8; }

cudaError_t launch_complete_basis(double* U, long rows, long ld, int s, const double* sigma,
                                  long null_dim, double* work, int* status,
                                  const int* abort_flag, cudaStream_t st) {
    complete_basis_kernel<<<1, 1024, 0, st>>>(U, rows, ld, s, sigma, null_dim, work, status,
                                              abort_flag);
    return cudaGetLastError();
}

}  // namespace rsvdb200
