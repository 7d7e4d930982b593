// Robust paths of the rSVD on B200:
//
//  * the Householder QR fallback of CholeskyQR2 — the reference's Householder QR
//    (qr.cpp:27-102: reflector v ~ x + sign(x_1)||x|| e_1 per column, thin Q accumulated
//    backwards from the identity, diag(R) >= 0 by flipping R rows / Q columns) blocked
//    into 32-column panels with the compact WY form, in one cooperative launch (below);
//    it only runs on ill-conditioned input.
//
//  * complete_basis_kernel — the reference's deterministic orthonormal completion
//    (svd.cpp:111-151): for each missing column, canonical vectors e_t are tried in
//    ascending order of row load (sum of squares of the row over the valid columns,
//    ties by index, i.e. the stable sort of svd.cpp:126-130), orthogonalised by two
//    modified Gram-Schmidt passes and accepted when the remaining norm >= 1e-4.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace rsvdb200 {

// =============================================== blocked Householder QR (compact WY)
// One cooperative launch per QR. CTA b owns the contiguous rows [lo, hi) of the M x NP
// working copy A of Y. Columns are factored in panels of up to 32 (one warp lane per
// panel column):
//  * column step k (one grid barrier each): every CTA re-reduces, in a fixed order, the
//    partials p_l = sum_{i > k} A[i][k] A[i][j0 + l] the previous step left behind
//    (p_k is the tail norm^2 of column k, p_j its dots with the later panel columns) and
//    reads row k from a broadcast buffer; that gives the reflector v = (x + sign(x_k)
//    ||x|| e_k) / ||.|| of qr.cpp:44-58 and v.w_j = (p_j + alpha A[k][j]) / ||v|| without a
//    second reduction; the CTA then updates its rows of the panel (w_j -= 2 (v.w_j) v) and
//    accumulates the partials of column k + 1 in the same pass. The panel slice lives in
//    shared memory when it fits (rows_per * 32 doubles), else it is updated in place in HBM.
//  * panel end (two barriers): V^T V and W = V^T A_trail partials per CTA, a distributed
//    fixed-order reduction, then T of the compact WY form H_j0 ... H_j0+jb-1 = I - V T V^T
//    (T(1:i-1, i) = -tau_i T(1:i-1, 1:i-1) V^T v_i, tau = 2 for the unit reflectors) and
//    A_trail -= V (T^T W) on every CTA's rows (DFMA; the first column of the next panel
//    gets its partials from the same pass).
//  * Q: backward over the panels from [I; 0] (qr.cpp:71-84 accumulates reflectors
//    backwards the same way), Q[:, j0:] -= V (T (V^T Q[:, j0:])), two barriers per panel.
//  * diag(R) >= 0 by flipping R rows / Q columns (qr.cpp:86-93).
// Every cross-CTA sum is a fixed-order sum, so the result is deterministic. Barriers: s
// column steps plus two per panel for the factorisation and two per panel for Q (s = 74:
// 86), instead of the unblocked version's 4s + 3 launches that each re-read the m x s
// working matrix.
constexpr int kPW = 32;           // panel width = warp lanes
constexpr int kHHThreads = 512;
constexpr int kHHWarps = kHHThreads / 32;
constexpr int kUnroll = 4;  // independent row loads in flight per warp
constexpr int kMaxCols = 288;
constexpr int kPartStride = kPW * kPW + kPW * kMaxCols;  // V^T V, then W (kPW x kMaxCols)
// shared memory: per-warp reduction buffer (kHHWarps x kPW x kPW) + M2 (kPW x kMaxCols) +
// T (kPW x (kPW + 1)); the panel slice of the column steps aliases the first two
constexpr int kSmRed = kHHWarps * kPW * kPW;
constexpr int kSmM2 = kPW * kMaxCols;
constexpr int kSmT = kPW * (kPW + 1);
constexpr size_t kHHSmem = (size_t)(kSmRed + kSmM2 + kSmT) * sizeof(double);
constexpr long kSlabRows = (kSmRed + kSmM2) / kPW;  // rows of a panel slice that fit

struct HH {
    const double* Y;
    long ldy;
    long M;
    int s, NP, G;
    long rows_per;
    double* A;        // M x NP working copy, R in its upper triangle at the end
    double* V;        // M x NP reflectors (column k: rows >= k, unit norm)
    double* Q;        // output M x ldq
    long ldq;
    double* R;        // output NP x NP
    double* colpart;  // [2][G][kPW] column-step partials (double-buffered by k parity)
    double* rowbuf;   // [2][kPW] row k of the panel (double-buffered)
    double* part;     // [G][kPartStride] panel-pass partials
    double* red;      // [2][kPartStride] reduced panel-pass sums (double-buffered)
    double* T;        // [panels][kPW][kPW]
};

// Deterministic sum over the CTAs of the 32-lane column-step partials of parity `par`
// into out[32]: warp w sums the CTAs g = w (mod 16) in order, then lane l adds the 16
// warp sums in order. Cross-CTA data is read with ld.global.cg (L2), never a stale L1 line.
__device__ __forceinline__ void sum_colpart(const HH& h, int par, double* wred, double* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* p = h.colpart + (size_t)par * h.G * kPW;
    double t = 0.0;
    for (int g = warp; g < h.G; g += kHHWarps) t += __ldcg(p + g * kPW + lane);
    wred[warp * kPW + lane] = t;
    __syncthreads();
    if (threadIdx.x < kPW) {
        double u = 0.0;
        for (int w = 0; w < kHHWarps; ++w) u += wred[w * kPW + threadIdx.x];
        out[threadIdx.x] = u;
    }
}

// Warp partials acc (one per lane) of all warps -> CTA partial written to out[lane].
__device__ __forceinline__ void cta_lane_sum(double acc, double* wred, double* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    wred[warp * kPW + lane] = acc;
    __syncthreads();
    if (threadIdx.x < kPW) {
        double t = 0.0;
        for (int w = 0; w < kHHWarps; ++w) t += wred[w * kPW + threadIdx.x];
        out[threadIdx.x] = t;
    }
    __syncthreads();
}

// Pass over rows [r0, hi) of this CTA accumulating, per job, acc[a] (a < jb) at lane l:
// job 0 (if with_vtv): sum v_a v_{j0+l};  job 1 + c: sum v_a X[i][c0 + 32 c + l].
// Per-CTA sums go to part[cta][a * kPW + l] (V^T V) and part[cta][kPW*kPW + a*kMaxCols + j]
// (W, j = column offset from c0).
__device__ void panel_dots(const HH& h, const double* X, long ldx, long r0, long hi, int j0,
                           int jb, int c0, int ncols, bool with_vtv, double* sred) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nch = (ncols + kPW - 1) / kPW;
    const int jobs = nch + (with_vtv ? 1 : 0);
    double* out = h.part + (size_t)blockIdx.x * kPartStride;
    if (jobs == 0) return;
    const int groups = kHHWarps / jobs;
    const int job = warp % jobs, grp = warp / jobs;
    double acc[kPW];
#pragma unroll
    for (int a = 0; a < kPW; ++a) acc[a] = 0.0;
    if (grp < groups) {
        const bool vtv = with_vtv && job == 0;
        const int c = with_vtv ? job - 1 : job;
        const int col = c0 + c * kPW + lane;
        const bool colok = vtv ? lane < jb : (c * kPW + lane) < ncols;
        // rows in groups of kUnroll independent loads (the loop is L2/HBM-latency bound)
        for (long i0 = r0 + grp; i0 < hi; i0 += (long)kUnroll * groups) {
            double vl[kUnroll], x[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const long i = i0 + (long)u * groups;
                const bool ok = i < hi;
                vl[u] = ok && lane < jb ? h.V[i * h.NP + j0 + lane] : 0.0;
                x[u] = ok && !vtv && colok ? X[i * ldx + col] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const double xv = vtv ? vl[u] : x[u];
#pragma unroll
                for (int a = 0; a < kPW; ++a)
                    acc[a] = fma(__shfl_sync(0xffffffffu, vl[u], a), xv, acc[a]);
            }
        }
    }
    // cross-warp (same job) reduction in a fixed order
#pragma unroll
    for (int a = 0; a < kPW; ++a) sred[(warp * kPW + a) * kPW + lane] = acc[a];
    __syncthreads();
    for (int e = threadIdx.x; e < jobs * kPW * kPW; e += kHHThreads) {
        const int jj = e / (kPW * kPW), a = (e / kPW) % kPW, l = e % kPW;
        if (a >= jb) continue;
        double t = 0.0;
        for (int g = 0; g < groups; ++g) t += sred[((g * jobs + jj) * kPW + a) * kPW + l];
        const bool vtv = with_vtv && jj == 0;
        const int c = with_vtv ? jj - 1 : jj;
        if (vtv) {
            out[a * kPW + l] = t;
        } else if (c * kPW + l < ncols) {
            out[kPW * kPW + a * kMaxCols + c * kPW + l] = t;
        }
    }
    __syncthreads();
}

// Distributed fixed-order reduction of entries [0, n) of every CTA's part into red.
__device__ void reduce_part(const HH& h, double* red, int n_vtv, int jb, int ncols) {
    const long nw = (long)jb * kMaxCols;
    const long total = kPW * kPW + nw;
    for (long e = (long)blockIdx.x * kHHThreads + threadIdx.x; e < total;
         e += (long)h.G * kHHThreads) {
        bool ok;
        if (e < kPW * kPW) ok = n_vtv && (e / kPW) < jb && (e % kPW) < jb;
        else ok = ((e - kPW * kPW) % kMaxCols) < ncols;
        if (!ok) continue;
        double t = 0.0;
        for (int g = 0; g < h.G; ++g) t += __ldcg(h.part + (size_t)g * kPartStride + e);
        red[e] = t;
    }
}

// X[i][c0 + j] -= sum_a v_a[i] M2[a][j] for the CTA's rows [r0, hi), j < ncols. With
// `next_k` >= 0 the warps on the first chunk also accumulate the column-step partials of
// column next_k = c0 (lanes < next_jb) and the owner of row next_k broadcasts it.
__device__ void panel_update(const HH& h, double* X, long ldx, long r0, long hi, int j0, int jb,
                             int c0, int ncols, const double* M2, long next_k, int next_jb,
                             double* wred) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nch = (ncols + kPW - 1) / kPW;
    double acc = 0.0;
    if (nch > 0) {
        const int groups = kHHWarps / nch;
        const int c = warp % nch, grp = warp / nch;
        if (grp < groups) {
            const int j = c * kPW + lane;
            const bool colok = j < ncols;
            for (long i0 = r0 + grp; i0 < hi; i0 += (long)kUnroll * groups) {
                double vl[kUnroll], x[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const long i = i0 + (long)u * groups;
                    const bool ok = i < hi;
                    vl[u] = ok && lane < jb ? h.V[i * h.NP + j0 + lane] : 0.0;
                    x[u] = ok && colok ? X[i * ldx + c0 + j] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const long i = i0 + (long)u * groups;
                    double upd = 0.0;
#pragma unroll
                    for (int a = 0; a < kPW; ++a)
                        upd = fma(__shfl_sync(0xffffffffu, vl[u], a), M2[a * kMaxCols + j], upd);
                    const double xv = x[u] - upd;
                    if (i < hi && colok) X[i * ldx + c0 + j] = xv;
                    if (next_k >= 0 && c == 0) {
                        const double xk = __shfl_sync(0xffffffffu, xv, 0);
                        if (i < hi && i > next_k && lane < next_jb) acc = fma(xk, xv, acc);
                        if (i == next_k && i < hi && lane < next_jb)
                            h.rowbuf[(next_k & 1) * kPW + lane] = xv;
                    }
                }
            }
        }
    }
    if (next_k >= 0)
        cta_lane_sum(acc, wred, h.colpart + ((size_t)(next_k & 1) * h.G + blockIdx.x) * kPW);
}

__global__ void __launch_bounds__(kHHThreads, 1) hh_blocked_kernel(HH h) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double sm[];
    double* sred = sm;                  // kSmRed
    double* M2 = sm + kSmRed;           // kSmM2
    double* Ts = M2 + kSmM2;            // kSmT
    __shared__ double cs[kPW], rowk[kPW], dd[kPW], wred[kHHWarps * kPW], diag[kMaxCols];
    __shared__ int taus[kPW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = h.s, NP = h.NP;
    const long lo = (long)blockIdx.x * h.rows_per, hi = min(h.M, lo + h.rows_per);
    const int panels = (s + kPW - 1) / kPW;

    // ---- init: A = Y (pad columns zero), V = 0, partials of column 0
    {
        double acc = 0.0;
        const int jb0 = min(kPW, s);
        for (long i = lo + warp; i < hi; i += kHHWarps) {
            double a0 = 0.0;
            for (int c = lane; c < NP; c += kPW) {
                const double y = c < s ? h.Y[i * h.ldy + c] : 0.0;
                h.A[i * NP + c] = y;
                h.V[i * NP + c] = 0.0;
                if (c == lane) a0 = y;
            }
            const double x0 = __shfl_sync(0xffffffffu, a0, 0);
            if (i > 0 && lane < jb0) acc = fma(x0, a0, acc);
            if (i == 0 && lane < jb0) h.rowbuf[lane] = a0;
        }
        cta_lane_sum(acc, wred, h.colpart + (size_t)blockIdx.x * kPW);
    }
    grid.sync();

    for (int p = 0; p < panels; ++p) {
        const int j0 = p * kPW, jb = min(kPW, s - j0);
        // the panel slice [max(lo, j0), hi) x jb in shared memory when it fits
        const long r0 = max(lo, (long)j0);
        const bool in_smem = hi - r0 <= kSlabRows;
        double* P;
        long ldp;
        long base;
        if (in_smem) {
            P = sm;
            ldp = kPW;
            base = r0;
            for (long i = r0 + warp; i < hi; i += kHHWarps)
                if (lane < jb) P[(i - base) * kPW + lane] = h.A[i * NP + j0 + lane];
            __syncthreads();
        } else {
            P = h.A + j0;
            ldp = NP;
            base = 0;
        }
        for (int kl = 0; kl < jb; ++kl) {
            const long k = j0 + kl;
            const int par = (int)(k & 1);
            sum_colpart(h, par, wred, cs);
            if (threadIdx.x < kPW) rowk[threadIdx.x] = __ldcg(h.rowbuf + par * kPW + threadIdx.x);
            __syncthreads();
            const double tail2 = cs[kl], x0 = rowk[kl];
            const double norm_x = sqrt(tail2 + x0 * x0);
            const bool active = norm_x != 0.0;  // zero column: H_k = I, r_kk = 0
            const double sign = x0 >= 0.0 ? 1.0 : -1.0;
            const double alpha = x0 + sign * norm_x;
            const double inv_nv = active ? 1.0 / sqrt(tail2 + alpha * alpha) : 0.0;
            if (threadIdx.x < kPW) {
                const int l = threadIdx.x;
                dd[l] = (l > kl && l < jb) ? 2.0 * (inv_nv * (cs[l] + alpha * rowk[l])) : 0.0;
                if (l == 0) taus[kl] = active ? 1 : 0;
            }
            __syncthreads();
            const bool more = kl + 1 < jb;
            double acc = 0.0;
            for (long i0 = max(lo, k) + warp; i0 < hi; i0 += (long)kUnroll * kHHWarps) {
                double av[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const long i = i0 + (long)u * kHHWarps;
                    av[u] = i < hi && lane < jb ? P[(i - base) * ldp + lane] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const long i = i0 + (long)u * kHHWarps;
                    double a = av[u];
                    const double xk = __shfl_sync(0xffffffffu, a, kl);
                    const double v = (i == k ? alpha : xk) * inv_nv;
                    if (i < hi) {
                        if (lane == kl) {
                            h.V[i * NP + k] = v;
                            if (i == k && active) a = -sign * norm_x;
                        } else if (lane > kl && lane < jb && active) {
                            a = fma(-dd[lane], v, a);
                        }
                        if (lane < jb && (lane > kl || i == k)) P[(i - base) * ldp + lane] = a;
                    }
                    if (more) {
                        const double xn = __shfl_sync(0xffffffffu, a, kl + 1);
                        if (i < hi && i > k + 1 && lane < jb) acc = fma(xn, a, acc);
                        if (i == k + 1 && i < hi && lane < jb)
                            h.rowbuf[(par ^ 1) * kPW + lane] = a;
                    }
                }
            }
            if (more) {
                cta_lane_sum(acc, wred, h.colpart + ((size_t)(par ^ 1) * h.G + blockIdx.x) * kPW);
                grid.sync();
            }
        }
        if (in_smem) {
            __syncthreads();
            for (long i = r0 + warp; i < hi; i += kHHWarps)
                if (lane < jb) h.A[i * NP + j0 + lane] = P[(i - base) * kPW + lane];
            __syncthreads();
        }
        // ---- panel end: V^T V and W = V^T A_trail (trailing columns in blocks of
        // kMaxCols), reduced over the grid; T; A_trail -= V (T^T W)
        const int c0 = j0 + jb, ntrail = s - c0;
        double* red = h.red + (size_t)(p & 1) * kPartStride;
        const bool next = p + 1 < panels;
        for (int cb = 0; cb == 0 || cb < ntrail; cb += kMaxCols) {
            const int nc = max(0, min(kMaxCols, ntrail - cb));
            panel_dots(h, h.A, NP, r0, hi, j0, jb, c0 + cb, nc, cb == 0, sred);
            grid.sync();
            reduce_part(h, red, cb == 0, jb, nc);
            grid.sync();
            // the reduced V^T V and W blocks into shared memory (sred is free here)
            double* vtv_s = sred;              // kPW x kPW
            double* w_s = sred + kPW * kPW;    // kPW x kMaxCols
            for (int e = threadIdx.x; e < kPW * kPW; e += kHHThreads)
                if (cb == 0) vtv_s[e] = (e / kPW < jb && e % kPW < jb) ? __ldcg(red + e) : 0.0;
            for (int e = threadIdx.x; e < jb * kMaxCols; e += kHHThreads)
                w_s[e] = (e % kMaxCols < nc) ? __ldcg(red + kPW * kPW + e) : 0.0;
            __syncthreads();
            if (cb == 0) {
                // T (every CTA the same; CTA 0 keeps it for the Q pass)
                if (warp == 0) {
                    for (int i = 0; i < kPW; ++i) Ts[lane * (kPW + 1) + i] = 0.0;
                    __syncwarp();
                    for (int i = 0; i < jb; ++i) {
                        const double ti = taus[i] ? 2.0 : 0.0;
                        double w = 0.0;
                        if (lane < i)
                            for (int c = lane; c < i; ++c)
                                w = fma(Ts[lane * (kPW + 1) + c], vtv_s[c * kPW + i], w);
                        __syncwarp();
                        if (lane < i) Ts[lane * (kPW + 1) + i] = -ti * w;
                        if (lane == i) Ts[i * (kPW + 1) + i] = ti;
                        __syncwarp();
                    }
                }
                __syncthreads();
                if (blockIdx.x == 0)
                    for (int e = threadIdx.x; e < kPW * kPW; e += kHHThreads)
                        h.T[(size_t)p * kPW * kPW + e] = Ts[(e / kPW) * (kPW + 1) + e % kPW];
            }
            // M2 = T^T W (jb x nc)
            for (int e = threadIdx.x; e < kPW * kMaxCols; e += kHHThreads) {
                const int a = e / kMaxCols, j = e % kMaxCols;
                double t = 0.0;
                if (a < jb && j < nc)
                    for (int c = 0; c <= a; ++c)
                        t = fma(Ts[c * (kPW + 1) + a], w_s[c * kMaxCols + j], t);
                M2[e] = t;
            }
            __syncthreads();
            const bool first = next && cb == 0;
            panel_update(h, h.A, NP, r0, hi, j0, jb, c0 + cb, nc, M2, first ? c0 : -1,
                         first ? min(kPW, s - c0) : 0, wred);
            __syncthreads();
        }
        grid.sync();
    }

    // ---- Q = H_0 ... H_{s-1} [I; 0], backward over the panels
    for (long i = lo + warp; i < hi; i += kHHWarps)
        for (int c = lane; c < NP; c += kPW) h.Q[i * h.ldq + c] = (i == c && c < s) ? 1.0 : 0.0;
    __syncthreads();
    for (int p = panels - 1; p >= 0; --p) {
        const int j0 = p * kPW, jb = min(kPW, s - j0), ntot = s - j0;
        const long r0 = max(lo, (long)j0);
        double* red = h.red + (size_t)(p & 1) * kPartStride;
        for (int e = threadIdx.x; e < kPW * kPW; e += kHHThreads)
            Ts[(e / kPW) * (kPW + 1) + e % kPW] = __ldcg(h.T + (size_t)p * kPW * kPW + e);
        __syncthreads();
        for (int cb = 0; cb < ntot; cb += kMaxCols) {
            const int nc = min(kMaxCols, ntot - cb);
            panel_dots(h, h.Q, h.ldq, r0, hi, j0, jb, j0 + cb, nc, false, sred);
            grid.sync();
            reduce_part(h, red, 0, jb, nc);
            grid.sync();
            double* w_s = sred;  // the reduced W block (kPW x kMaxCols) in shared memory
            for (int e = threadIdx.x; e < jb * kMaxCols; e += kHHThreads)
                w_s[e] = (e % kMaxCols < nc) ? __ldcg(red + kPW * kPW + e) : 0.0;
            __syncthreads();
            // M2 = T W
            for (int e = threadIdx.x; e < kPW * kMaxCols; e += kHHThreads) {
                const int a = e / kMaxCols, j = e % kMaxCols;
                double t = 0.0;
                if (a < jb && j < nc)
                    for (int c = a; c < jb; ++c)
                        t = fma(Ts[a * (kPW + 1) + c], w_s[c * kMaxCols + j], t);
                M2[e] = t;
            }
            __syncthreads();
            panel_update(h, h.Q, h.ldq, r0, hi, j0, jb, j0 + cb, nc, M2, -1, 0, wred);
            __syncthreads();
        }
    }
    // ---- diag(R) >= 0 (qr.cpp:86-93): the factorisation is final (grid.sync above)
    for (int cb = 0; cb < s; cb += kMaxCols) {
        const int nc = min(kMaxCols, s - cb);
        for (int j = threadIdx.x; j < nc; j += kHHThreads)
            diag[j] = __ldcg(h.A + (long)(cb + j) * NP + cb + j);
        __syncthreads();
        for (long i = lo + warp; i < hi; i += kHHWarps)
            for (int c = lane; c < nc; c += kPW)
                if (diag[c] < 0.0) h.Q[i * h.ldq + cb + c] = -h.Q[i * h.ldq + cb + c];
        __syncthreads();
    }
    for (long i = blockIdx.x; i < NP; i += h.G) {
        const bool flip = i < s && __ldcg(h.A + i * NP + i) < 0.0;
        for (int j = threadIdx.x; j < NP; j += kHHThreads) {
            double r = (i < s && j < s && j >= i) ? __ldcg(h.A + i * NP + j) : 0.0;
            h.R[i * NP + j] = flip ? -r : r;
        }
    }
}

static int hh_grid(long M) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return (int)std::max(1L, std::min((long)sms, (M + 63) / 64));
}

size_t householder_work_doubles(long M, int NP) {
    const int G = hh_grid(M);
    const int panels = (NP + kPW - 1) / kPW;
    return 2 * (size_t)M * NP + 2 * (size_t)G * kPW + 2 * kPW + (size_t)G * kPartStride +
           2 * (size_t)kPartStride + (size_t)panels * kPW * kPW + NP + 64;
}

cudaError_t launch_householder_qr(const double* Y, long M, int s, long ldy, double* Qout, long ldq,
                                  double* R, int NP, double* work, cudaStream_t st) {
    if (s > NP || M < s || s < 1) return cudaErrorInvalidValue;
    HH h;
    h.Y = Y;
    h.ldy = ldy;
    h.M = M;
    h.s = s;
    h.NP = NP;
    h.G = hh_grid(M);
    h.rows_per = (M + h.G - 1) / h.G;
    h.Q = Qout;
    h.ldq = ldq;
    h.R = R;
    h.A = work;
    h.V = h.A + (size_t)M * NP;
    h.colpart = h.V + (size_t)M * NP;
    h.rowbuf = h.colpart + 2 * (size_t)h.G * kPW;
    h.part = h.rowbuf + 2 * kPW;
    h.red = h.part + (size_t)h.G * kPartStride;
    h.T = h.red + 2 * (size_t)kPartStride;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(hh_blocked_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kHHSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    void* args[] = {&h};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)hh_blocked_kernel, dim3(h.G),
                                                dim3(kHHThreads), args, kHHSmem, st);
    if (e != cudaSuccess) return e;
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
