// Robust paths of the rSVD on B200:
//
//  * householder_qr_kernel — the CholeskyQR2 fallback. A cooperative (grid-
//    synchronised) restatement of the reference's unblocked Householder QR
//    (qr.cpp:27-102): reflector v ~ x + sign(x_1)||x|| e_1 per column, applied to
//    the trailing columns, thin Q accumulated backwards from the identity, then
//    diag(R) >= 0 by flipping R rows / Q columns. One CTA per SM owns a contiguous
//    row slab; every reduction is a fixed-order sum over per-CTA partials, so the
//    result is deterministic. Two grid barriers per column in the factorisation and
//    one per column in the Q accumulation.
//
//  * complete_basis_kernel — the reference's deterministic orthonormal completion
//    (svd.cpp:111-151): for each missing column, canonical vectors e_t are tried in
//    ascending order of row load (sum of squares of the row over the valid columns,
//    ties by index, i.e. the stable sort of svd.cpp:126-130), orthogonalised by two
//    modified Gram-Schmidt passes and accepted when the remaining norm >= 1e-4.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace rsvdb200 {

constexpr int kHHThreads = 256;
constexpr int kHHWarps = kHHThreads / 32;
constexpr int kMaxCh = 6;  // up to 192 columns, 32 per lane-chunk

// Sense-reversing grid barrier for a cooperative launch.
__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen,
                                             unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned my = *gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicAdd((unsigned*)gen, 1u);
        } else {
            while (*gen == my) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// Block-wide partial sums of sum_{rows i in [lo,hi)} x_i * w[i][j] for j in [j0, s):
// x_i = xcol ? w[i][xcol_idx] * xscale : vbuf[i]... generalised through a functor.
template <typename XF>
__device__ void block_col_dots(const double* __restrict__ w, long ld, long lo, long hi, int j0,
                               int s, XF xval, double* __restrict__ out /* [s] */,
                               double* __restrict__ red /* smem kHHWarps x 192 */) {
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
        if (j < s) red[warp * 192 + j] = acc[c];
    }
    __syncthreads();
    for (int j = j0 + threadIdx.x; j < s; j += blockDim.x) {
        double t = 0.0;
        for (int q = 0; q < kHHWarps; ++q) t += red[q * 192 + j];
        out[j] = t;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kHHThreads) householder_qr_kernel(
    const double* __restrict__ Y, long M, int s, long ldy, double* __restrict__ Q, long ldq,
    double* __restrict__ R, int NP, double* __restrict__ work /* M x NP */,
    double* __restrict__ refl /* M x NP */, double* __restrict__ part /* 2 x nb x (NP+2) */,
    int* __restrict__ act /* NP */, unsigned* __restrict__ bar) {
    __shared__ double red[kHHWarps * 192];
    __shared__ double dj[192];
    const unsigned nb = gridDim.x;
    const long rpb = (M + nb - 1) / nb;
    const long lo = blockIdx.x * rpb, hi = min(M, lo + rpb);
    const long pstride = (long)nb * (NP + 2);
    unsigned* count = bar;
    volatile unsigned* gen = bar + 1;

    // working copy (row-major, ld NP) and zeroed reflectors
    for (long i = lo; i < hi; ++i)
        for (int j = threadIdx.x; j < NP; j += blockDim.x) {
            work[i * NP + j] = j < s ? Y[i * ldy + j] : 0.0;
            refl[i * NP + j] = 0.0;
        }
    // Partial-sum layout: part[buf][block][0..NP-1] = column dots, [NP] = tail norm^2.
    // Buffers alternate per step; every reader of a buffer is separated from its next
    // writer by at least one grid barrier.
    auto tail_norm = [&](int k, double* dst) {
        double acc = 0.0;
        for (long i = max(lo, (long)k + 1) + threadIdx.x; i < hi; i += blockDim.x) {
            const double x = work[i * NP + k];
            acc += x * x;
        }
        acc = warp_sum(acc);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int q = 0; q < kHHWarps; ++q) t += red[q];
            dst[blockIdx.x * (NP + 2) + NP] = t;
        }
        __syncthreads();
    };
    __syncthreads();
    tail_norm(0, part);
    grid_barrier(count, gen, nb);

    for (int k = 0; k < s; ++k) {
        double* pk = part + (k & 1) * pstride;        // norms of column k, dots of step k
        double* pn = part + ((k + 1) & 1) * pstride;  // norms of column k + 1
        double tail2 = 0.0;
        for (unsigned b = 0; b < nb; ++b) tail2 += pk[b * (NP + 2) + NP];
        const double x0 = work[(long)k * NP + k];
        const double norm_x = sqrt(tail2 + x0 * x0);
        if (norm_x == 0.0) {  // zero column: H_k = I, r_kk = 0 (qr.cpp:47)
            if (blockIdx.x == 0 && threadIdx.x == 0) act[k] = 0;
            if (k + 1 < s) {
                tail_norm(k + 1, pn);
                grid_barrier(count, gen, nb);
            }
            continue;
        }
        const double sign = x0 >= 0.0 ? 1.0 : -1.0;
        const double alpha = x0 + sign * norm_x;
        const double inv_nv = 1.0 / sqrt(tail2 + alpha * alpha);
        if (blockIdx.x == 0 && threadIdx.x == 0) act[k] = 1;
        for (long i = max(lo, (long)k) + threadIdx.x; i < hi; i += blockDim.x)
            refl[i * NP + k] = (i == k ? alpha : work[i * NP + k]) * inv_nv;
        __syncthreads();
        block_col_dots(work, NP, max(lo, (long)k), hi, k + 1, s,
                       [&](long i) { return refl[i * NP + k]; }, pk + blockIdx.x * (NP + 2), red);
        grid_barrier(count, gen, nb);
        for (int j = k + 1 + threadIdx.x; j < s; j += blockDim.x) {
            double t = 0.0;
            for (unsigned b = 0; b < nb; ++b) t += pk[b * (NP + 2) + j];
            dj[j] = 2.0 * t;
        }
        __syncthreads();
        for (long i = max(lo, (long)k); i < hi; ++i) {
            const double vi = refl[i * NP + k];
            for (int j = k + 1 + threadIdx.x; j < s; j += blockDim.x) work[i * NP + j] -= dj[j] * vi;
        }
        if (k >= lo && k < hi && threadIdx.x == 0) work[(long)k * NP + k] = -sign * norm_x;
        __syncthreads();
        if (k + 1 < s) tail_norm(k + 1, pn);
        grid_barrier(count, gen, nb);
    }

    // ---- thin Q by backward accumulation (qr.cpp:71-84), Q rows owned per block
    for (long i = lo; i < hi; ++i)
        for (int j = threadIdx.x; j < NP; j += blockDim.x)
            Q[i * ldq + j] = (i == j && j < s) ? 1.0 : 0.0;
    __syncthreads();
    int phase = 0;
    for (int kk = s - 1; kk >= 0; --kk) {
        if (!act[kk]) continue;
        double* pd = part + (phase & 1) * pstride;
        ++phase;
        block_col_dots(Q, ldq, max(lo, (long)kk), hi, kk, s,
                       [&](long i) { return refl[i * NP + kk]; }, pd + blockIdx.x * (NP + 2), red);
        grid_barrier(count, gen, nb);
        for (int j = kk + threadIdx.x; j < s; j += blockDim.x) {
            double t = 0.0;
            for (unsigned b = 0; b < nb; ++b) t += pd[b * (NP + 2) + j];
            dj[j] = 2.0 * t;
        }
        __syncthreads();
        for (long i = max(lo, (long)kk); i < hi; ++i) {
            const double vi = refl[i * NP + kk];
            for (int j = kk + threadIdx.x; j < s; j += blockDim.x) Q[i * ldq + j] -= dj[j] * vi;
        }
        __syncthreads();
    }
    grid_barrier(count, gen, nb);

    // ---- diag(R) >= 0 (qr.cpp:86-93); R written from the rows each block owns
    for (long i = lo; i < hi && i < NP; ++i)
        for (int j = threadIdx.x; j < NP; j += blockDim.x) {
            double r = (i < s && j < s && j >= i) ? work[i * NP + j] : 0.0;
            if (i < s && work[i * NP + i] < 0.0) r = -r;
            R[i * NP + j] = r;
        }
    for (long i = lo; i < hi; ++i)
        for (int j = threadIdx.x; j < s; j += blockDim.x)
            if (work[(long)j * NP + j] < 0.0) Q[i * ldq + j] = -Q[i * ldq + j];
}

size_t householder_work_doubles(long M, int s) {
    const int NP = 192;
    (void)s;
    return 2 * (size_t)M * NP + 2 * 148 * 8 * (size_t)(NP + 2) + NP + 64;
}

cudaError_t launch_householder_qr(const double* Y, long M, int s, long ldy, double* Qout, long ldq,
                                  double* R, int NP, double* work, cudaStream_t st) {
    if (s > 192 || NP > 192) return cudaErrorInvalidValue;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, householder_qr_kernel, kHHThreads, 0);
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    unsigned nb = (unsigned)sms;
    if ((long)nb > M) nb = (unsigned)(M < 1 ? 1 : M);
    double* w = work;
    double* refl = work + (size_t)M * NP;
    double* part = refl + (size_t)M * NP;
    int* act = reinterpret_cast<int*>(part + 2 * (size_t)nb * (NP + 2));
    unsigned* bar = reinterpret_cast<unsigned*>(act + NP);
    cudaError_t e = cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(R, 0, (size_t)NP * NP * sizeof(double), st);
    if (e != cudaSuccess) return e;
    void* args[] = {(void*)&Y, (void*)&M, (void*)&s, (void*)&ldy, (void*)&Qout, (void*)&ldq,
                    (void*)&R, (void*)&NP, (void*)&w, (void*)&refl, (void*)&part, (void*)&act,
                    (void*)&bar};
    e = cudaLaunchCooperativeKernel((const void*)householder_qr_kernel, dim3(nb), dim3(kHHThreads),
                                    args, 0, st);
    return e;
}

// ========================================================= orthonormal completion
__global__ void __launch_bounds__(1024) complete_basis_kernel(double* __restrict__ U, long rows,
                                                              long ld, int r0, int r1,
                                                              double* __restrict__ work,
                                                              int* __restrict__ status) {
    double* load = work;         // rows
    double* cand = work + rows;  // rows
    unsigned char* tried = reinterpret_cast<unsigned char*>(work + 2 * rows);
    __shared__ double sv[32];
    __shared__ long si[32];
    __shared__ double bcast;
    __shared__ long bidx;
    const int tid = threadIdx.x, nth = blockDim.x, warp = tid >> 5, lane = tid & 31;
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

cudaError_t launch_complete_basis(double* U, long rows, long ld, int r0, int r1, double* work,
                                  int* status, cudaStream_t st) {
    complete_basis_kernel<<<1, 1024, 0, st>>>(U, rows, ld, r0, r1, work, status);
    return cudaGetLastError();
}

}  // namespace rsvdb200
