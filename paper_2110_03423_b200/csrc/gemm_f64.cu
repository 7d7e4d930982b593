// FP64 tensor-core GEMMs for the rSVD hot path on B200 (sm_100a).
//
// The reference does every product of Algorithm 1 with one blocked CPU GEMM
// that materialises transposed operands (gemm.cpp:48-100). Here the two
// shapes that occur are separate kernels, both fed by TMA (128-byte swizzled
// boxes, 4-stage mbarrier pipeline, one producer warp) and computed on the FP64
// tensor cores with mma.sync m16n8k16 (DMMA; tcgen05 has no f64 kind):
//
//   ax  : Y = A * X      A row-major (M x K, lda), X given as Xt (NP x K, ldx),
//                        Y row-major (M x NP, ldy).  Contraction over A's rows'
//                        contiguous dimension.  Used for Y = A*Omega, Y = A*Z
//                        (rsvd.cpp:58,70), U = Q*U_B (rsvd.cpp:105), the TRSM
//                        Q = Y*R^-1 of CholeskyQR and the Gram B*B^T.
//   atx : Z = A^T * W    A row-major (K x N, lda) read in place (no transpose
//                        copy, cf. gemm.cpp:75-78), W row-major (K x NP, ldw);
//                        output either Z^T (NP x N) or Z (N x NP).  Used for
//                        A^T*W (rsvd.cpp:69), B = Q^T*A (rsvd.cpp:100) and the
//                        tall Gram Y^T*Y of CholeskyQR.
//
// Both support split-K into fixed partial slabs that rsvd_reduce_partials
// sums in a fixed order, so every result is deterministic run to run.
//
// The passes over A with a sketch width s whose last s % 8 <= 4 columns would fill a padded
// n8 MMA tile (s = 74, 42, ...) run those columns as DFMA partial dot products instead
// (ax only, TAIL / SKIP variants): DMMA and DFMA share the FP64 datapath at the same rate
// per flop, so the pipe then does s columns of work instead of round_up(s, 8). (The atx
// shape was measured slower with the one-warp-column layout the tail needs: its scalar
// fragment loads make it shared-memory-issue bound.)
//
// Bank-conflict-free fragment loads from the 128B-swizzled boxes come from
// permuting which physical k each MMA k-slot reads (the same permutation on
// both operands, so the product is unchanged):
//   ax : k = 4*t + q                     (K-major A and K-major Xt: a thread's k-slot
//                                          pairs are adjacent doubles, one 16-byte load)
//   atx: k = 2*t + (q&1) + 8*(q>>1)      (M-major A and N-major W)
// with t = lane&3 and q the 4-wide k-slot group.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace rsvdb200 {

constexpr int kBK = 32;           // k extent of one pipeline stage (two 16-wide boxes)
constexpr int kBoxBytesRow = 128; // 16 doubles

__device__ __forceinline__ int k_ax(int t, int q) { return 4 * t + q; }

__device__ __forceinline__ double2 lds_f64x2(const char* smem_base, uint32_t byte_off) {
    return *reinterpret_cast<const double2*>(smem_base + byte_off);
}
__device__ __forceinline__ int k_atx(int t, int q) { return 2 * t + (q & 1) + 8 * (q >> 1); }

// Exponent field all ones (Inf/NaN) from the high word with integer ops: the compiler turns
// the obvious form into DSETP |x| == Inf / NaN tests, which occupy the FP64 pipe the DMMAs need.
__device__ __forceinline__ uint32_t exp_bits(double x) {
    uint32_t hi;
    asm("mov.b64 {_, %0}, %1;" : "=r"(hi) : "d"(x));
    return hi & 0x7ff00000u;
}

// Fused Gram epilogue of the ax kernel: G_tile = Y_tile^T Y_tile (NP x NP, upper
// triangle) for the BM x NP output tile still held in the consumer warps' accumulators,
// so the CholeskyQR Gram of a freshly produced Y needs no extra pass over it. The tile
// is staged in the (now idle) pipeline buffers in the same 128B-swizzled box layout TMA
// produces and multiplied with the atx fragment maps (contraction over the BM rows).
// Only the 16x8 tiles that touch the upper triangle are computed, spread evenly over
// the warps; the rest of the partial is zero. Rows beyond M were zero-filled by TMA.
// One partial per CTA; the host reduces the partials in a fixed order.
template <int BM, int NT, int WM, int WN>
__device__ __forceinline__ void gram_epilogue(char* smem, const double (&acc)[BM / WM / 16][NT / WN][4],
                                              double* __restrict__ gpart) {
    constexpr int NP = NT * 8;
    constexpr int MI = BM / WM / 16;
    constexpr int NI = NT / WN;
    constexpr uint32_t kBox = BM * 128;  // BM rows x 16 doubles
    constexpr int MT = NP / 16;          // m16 tiles of G
    constexpr int NW = WM * WN;
    // upper-triangle tiles (a, b): b*8 + 7 >= a*16
    constexpr int kTiles = [] {
        int n = 0;
        for (int a = 0; a < MT; ++a)
            for (int b = 0; b < NT; ++b) n += (b * 8 + 7 >= a * 16);
        return n;
    }();
    constexpr int TPW = (kTiles + NW - 1) / NW;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp / WN, wn = warp % WN;
    const int g = lane >> 2, t = lane & 3;
    // all consumers are done reading the pipeline stages before they are overwritten
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int row = wm * (BM / WM) + mi * 16 + g + 8 * h;
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
                const int col = (wn * NI + ni) * 8 + 2 * t;
                *reinterpret_cast<double2*>(smem + (col >> 4) * kBox + swz128(row, col & 15)) =
                    make_double2(acc[mi][ni][2 * h], acc[mi][ni][2 * h + 1]);
            }
        }
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
    // tile idx -> (a, b): row a of the upper triangle holds tiles b = 2a .. NT-1
    auto tile_of = [](int idx, int& a, int& b) {
        a = 0;
        while (a < MT && idx >= NT - 2 * a) {
            idx -= NT - 2 * a;
            ++a;
        }
        b = 2 * a + idx;
    };
    double gacc[TPW][4];
#pragma unroll
    for (int i = 0; i < TPW; ++i)
#pragma unroll
        for (int v = 0; v < 4; ++v) gacc[i][v] = 0.0;
#pragma unroll 1
    for (int ks = 0; ks < BM / 16; ++ks) {
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
            const int idx = warp + i * NW;
            if (idx >= kTiles) continue;
            int a, b;
            tile_of(idx, a, b);
            const int c = b * 8 + g;
            double bf[4], af[8];
#pragma unroll
            for (int v = 0; v < 4; ++v)
                bf[v] = lds_f64(smem + (c >> 4) * kBox, swz128(ks * 16 + k_atx(t, v), c & 15));
#pragma unroll
            for (int v = 0; v < 8; ++v)
                af[v] = lds_f64(smem + a * kBox, swz128(ks * 16 + k_atx(t, v >> 1), g + 8 * (v & 1)));
            dmma_16x8x16(gacc[i], af, bf);
        }
    }
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
        const int idx = warp + i * NW;
        if (idx >= kTiles) continue;
        int a, b;
        tile_of(idx, a, b);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = a * 16 + g + 8 * h, c = b * 8 + 2 * t;
            *reinterpret_cast<double2*>(gpart + r * NP + c) =
                make_double2(gacc[i][2 * h], gacc[i][2 * h + 1]);
        }
    }
    // zero the tiles strictly below the diagonal (never read, kept finite for the reduce)
    for (int e = threadIdx.x; e < NP * NP; e += NW * 32) {
        const int r = e / NP, c = e % NP;
        if ((c >> 3) * 8 + 7 < (r >> 4) * 16) gpart[e] = 0.0;
    }
}

// ============================================================================ ax
// RESID: instead of storing Y, the epilogue accumulates sum (R[row][col] - Y[row][col])^2
// over the tile's rows < M and columns < resid_cols (R = resid, ld resid_ld) and writes
// the CTA's partial to resid_out[blockIdx.x] — the fused ||A - U S V^T||_F of
// RsvdResult::residual_fro (rsvd.cpp:37-49), one column chunk per launch.
// TAIL (> 0, WN == 1 only): X has nonzero rows only below 8 * nd + TAIL, nd = NT - SKIP.
// Column tiles [0, nd) run on DMMA, the TAIL columns after them as DFMA partial dot
// products over each thread's own k-slots (reduced across the 4 k-lanes once, after the main loop), and the
// tiles beyond are zero. DMMA and DFMA share the FP64 datapath at the same rate per flop
// (tools/probe/mixed_fp64.cu), so this removes the padding of s up to the MMA's n8 granule
// from the pipe: s = 74 costs 74 columns of FP64 work instead of 80.
template <int BM, int NT, int WM, int WN, int STAGES, bool CHECK, bool RESID = false, int TAIL = 0,
          int SKIP = 0>
__global__ void __launch_bounds__((WM * WN + 1) * 32, 1)
    gemm_ax_kernel(const __grid_constant__ CUtensorMap mapA,  // dims {K, M}, box {16, BM}
                   const __grid_constant__ CUtensorMap mapX,  // dims {K, NP}, box {16, NP}
                   double* __restrict__ Y, long ldy, long split_stride, int M, int k_tiles,
                   int k_tiles_per_split, int* __restrict__ flag, double* __restrict__ gram,
                   const double* __restrict__ resid, long resid_ld, int resid_cols,
                   double* __restrict__ resid_out, const int* __restrict__ abort_flag) {
    // a Cholesky breakdown earlier in an optimistic pipeline: the run is discarded and
    // repeated robustly, so skip the pass (all threads of the CTA return together)
    if (abort_flag && *(const volatile int*)abort_flag) return;
    constexpr int NP = NT * 8;
    constexpr int MI = BM / WM / 16;
    constexpr int NI = NT / WN;
    constexpr int kConsumers = WM * WN;
    constexpr uint32_t kABox = BM * kBoxBytesRow;
    constexpr uint32_t kXBox = NP * kBoxBytesRow;
    constexpr uint32_t kStage = 2 * kABox + 2 * kXBox;
    static_assert(MI >= 1 && NI >= 1 && BM % (16 * WM) == 0 && NT % WN == 0, "tiling");
    static_assert(kABox % 1024 == 0 && kXBox % 1024 == 0, "swizzle alignment");
    static_assert(TAIL == 0 || (WN == 1 && TAIL <= 4), "tail columns need WN == 1");

    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = align_smem_1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStage);
    uint64_t* empty = full + STAGES;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BM;
    constexpr int nd = NT - SKIP;  // DMMA column tiles (compile-time: acc stays in registers)
    static_assert(TAIL == 0 ? SKIP == 0 : (SKIP >= 1 && SKIP <= 2), "tail layout");
    const int kt0 = blockIdx.y * k_tiles_per_split;
    const int kt1 = min(k_tiles, kt0 + k_tiles_per_split);
    const int n_iter = max(0, kt1 - kt0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumers);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kConsumers) {
        // ----------------------------------------------------------- producer
        if (lane == 0) {
            tma_prefetch_desc(&mapA);
            tma_prefetch_desc(&mapX);
            for (int it = 0; it < n_iter; ++it) {
                const int s = it % STAGES;
                if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
                char* st = smem + s * kStage;
                mbar_arrive_expect_tx(&full[s], kStage);
                const int k = (kt0 + it) * kBK;
                tma_load_2d(st, &mapA, &full[s], k, m0);
                tma_load_2d(st + kABox, &mapA, &full[s], k + 16, m0);
                // TMA boxes hold at most 256 rows: wide sketches load Xt in two halves
                // (NP/2 is a multiple of 8 rows, so the 128B swizzle atoms line up)
                constexpr int kXParts = NP > 256 ? 2 : 1;
#pragma unroll
                for (int part = 0; part < kXParts; ++part) {
                    const uint32_t off = part * (kXBox / kXParts);
                    const int r0 = part * (NP / kXParts);
                    tma_load_2d(st + 2 * kABox + off, &mapX, &full[s], k, r0);
                    tma_load_2d(st + 2 * kABox + kXBox + off, &mapX, &full[s], k + 16, r0);
                }
            }
        }
        return;
    }

    // --------------------------------------------------------------- consumers
    const int wm = warp / WN, wn = warp % WN;
    const int g = lane >> 2, t = lane & 3;
    double acc[MI][NI][4];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;
    double tl[MI][2][TAIL > 0 ? TAIL : 1];  // tail partial sums: rows g, g + 8
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < (TAIL > 0 ? TAIL : 1); ++j) tl[i][h][j] = 0.0;
    uint32_t bad_exp = 0;  // max exponent field seen (CHECK): 0x7ff00000 = Inf/NaN

    for (int it = 0; it < n_iter; ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        const char* st = smem + s * kStage;
#pragma unroll 1
        for (int ks = 0; ks < 2; ++ks) {
            const char* boxA = st + ks * kABox;
            const char* boxX = st + 2 * kABox + ks * kXBox;
            double a[MI][8];
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) {
                const int r0 = wm * (BM / WM) + mi * 16 + g;
#pragma unroll
                for (int h = 0; h < 2; ++h)      // rows r0, r0 + 8
#pragma unroll
                    for (int qq = 0; qq < 2; ++qq) {  // k-slot groups (2qq, 2qq + 1)
                        const double2 p = lds_f64x2(boxA, swz128(r0 + 8 * h, k_ax(t, 2 * qq)));
                        a[mi][h + 4 * qq] = p.x;      // v = h + 2 * (2 qq)
                        a[mi][h + 4 * qq + 2] = p.y;  // v = h + 2 * (2 qq + 1)
                    }
            }
            if (CHECK && wn == 0) {
#pragma unroll
                for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                    for (int v = 0; v < 8; ++v) bad_exp = max(bad_exp, exp_bits(a[mi][v]));
            }
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
                if (TAIL == 0 || ni < nd) {  // warp-uniform
                    const int n = (wn * NI + ni) * 8 + g;
                    double b[4];
#pragma unroll
                    for (int qq = 0; qq < 2; ++qq) {
                        const double2 p = lds_f64x2(boxX, swz128(n, k_ax(t, 2 * qq)));
                        b[2 * qq] = p.x;
                        b[2 * qq + 1] = p.y;
                    }
#pragma unroll
                    for (int mi = 0; mi < MI; ++mi) dmma_16x8x16(acc[mi][ni], a[mi], b);
                }
            }
            if constexpr (TAIL > 0) {
                // a[mi][h + 2 q] holds A[row g + 8h][k = 4t + q]; X row c, k = 4t .. 4t + 3
#pragma unroll
                for (int j = 0; j < TAIL; ++j) {
                    const int c = nd * 8 + j;
                    const double2 x0 = lds_f64x2(boxX, swz128(c, k_ax(t, 0)));
                    const double2 x1 = lds_f64x2(boxX, swz128(c, k_ax(t, 2)));
#pragma unroll
                    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            tl[mi][h][j] = fma(a[mi][h + 6], x1.y, fma(a[mi][h + 4], x1.x,
                                           fma(a[mi][h + 2], x0.y, fma(a[mi][h], x0.x,
                                                                       tl[mi][h][j]))));
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (CHECK && __any_sync(0xffffffffu, bad_exp == 0x7ff00000u) && lane == 0) atomicOr(flag, 1);
    if constexpr (TAIL > 0) {
        // sum the tail over the 4 k-lanes, then place it in tile nd's accumulator layout
        // (lane t holds columns 8 nd + 2t, 2t + 1)
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int j = 0; j < TAIL; ++j) {
                    double v = tl[mi][h][j];
                    v += __shfl_xor_sync(0xffffffffu, v, 1);
                    v += __shfl_xor_sync(0xffffffffu, v, 2);
                    tl[mi][h][j] = v;
                }
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
            if (ni == nd)
#pragma unroll
                for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int v = 0; v < 2; ++v)  // explicit selects: no dynamic index
                            acc[mi][ni][2 * h + v] =
                                t == 0 ? tl[mi][h][v]
                                       : (TAIL > 2 && t == 1 ? tl[mi][h][TAIL > 2 ? 2 + v : 0] : 0.0);
    }

    // --------------------------------------------------------------- epilogue
    if constexpr (RESID) {
        double sq = 0.0;
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int row = m0 + wm * (BM / WM) + mi * 16 + g + 8 * h;
                if (row < M) {
#pragma unroll
                    for (int ni = 0; ni < NI; ++ni) {
                        const int col = (wn * NI + ni) * 8 + 2 * t;
#pragma unroll
                        for (int v = 0; v < 2; ++v)
                            if (col + v < resid_cols) {
                                const double d = resid[(long)row * resid_ld + col + v] -
                                                 acc[mi][ni][2 * h + v];
                                sq = fma(d, d, sq);
                            }
                    }
                }
            }
        sq = warp_sum(sq);
        __shared__ double red[WM * WN];
        if (lane == 0) red[warp] = sq;
        asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
        if (threadIdx.x == 0) {
            double tot = 0.0;
            for (int w = 0; w < kConsumers; ++w) tot += red[w];
            resid_out[blockIdx.x] = tot;
        }
        return;
    }
    double* out = Y + blockIdx.y * split_stride;
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int row = m0 + wm * (BM / WM) + mi * 16 + g + 8 * h;
            if (row < M) {
                double* yrow = out + row * ldy;
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) {
                    const int col = (wn * NI + ni) * 8 + 2 * t;
                    *reinterpret_cast<double2*>(yrow + col) =
                        make_double2(acc[mi][ni][2 * h], acc[mi][ni][2 * h + 1]);
                }
            }
        }
    }
    if constexpr (NT <= 12) {
        if (gram != nullptr) gram_epilogue<BM, NT, WM, WN>(smem, acc, gram + (long)blockIdx.x * NP * NP);
    }
}

// =========================================================================== atx
// ACC (OUT_T only): start from the Z^T already in Z instead of zero, so that a K range
// processed by consecutive launches accumulates exactly like one launch over it.
// TAIL (2, WN == 2, MI == 2): W has nonzero columns only below 8 * (NT - 1) + 2, i.e. the
// last column tile holds at most two sketch columns (s = 74 in NP = 80). Those two columns
// run as DFMA instead of a padded DMMA tile: warp column 1 does tiles NI .. NT - 2 on DMMA
// plus the tail, warp column 0 tiles 0 .. NI - 1; the warp columns are laid out so that every
// SMSP holds one warp of each (warp w and w + 4 share a scheduler), so the FP64 pipe of every
// SMSP does 2 NI - 1 tiles + a quarter tile of work instead of 2 NI tiles. Each stage's tail
// partial sums (over a thread's own k-slots) are reduced across the 4 k-lanes by a butterfly
// that leaves lane t owning (mi = t & 1, row half h = t >> 1, both columns), and added to a
// running sum: the accumulation order is per stage, so a K range split at stage boundaries
// (ACC launches) sums exactly like one launch.
template <int BJ, int NT, int WM, int WN, int STAGES, bool OUT_T, bool ACC = false, int TAIL = 0>
__global__ void __launch_bounds__((WM * WN + 1) * 32, 1)
    gemm_atx_kernel(const __grid_constant__ CUtensorMap mapA,  // dims {N, K}, box {16, 32}
                    const __grid_constant__ CUtensorMap mapW,  // dims {NP, K}, box {16, 32}
                    double* __restrict__ Z, long ldz, long split_stride, int N, int k_tiles,
                    int k_tiles_per_split, const int* __restrict__ abort_flag) {
    if (abort_flag && *(const volatile int*)abort_flag) return;  // see gemm_ax_kernel
    constexpr int NP = NT * 8;
    constexpr int MI = BJ / WM / 16;
    constexpr int NI = NT / WN;
    constexpr int kConsumers = WM * WN;
    constexpr int kABoxes = BJ / 16;
    constexpr int kWBoxes = NP / 16;
    constexpr uint32_t kBox = kBK * kBoxBytesRow;  // 4 KB: 32 rows x 16 doubles
    constexpr uint32_t kStage = (kABoxes + kWBoxes) * kBox;
    static_assert(NP % 16 == 0 && BJ % (16 * WM) == 0 && NT % WN == 0, "tiling");
    static_assert(TAIL == 0 || (TAIL == 2 && WN == 2 && MI == 2), "tail layout");

    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = align_smem_1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStage);
    uint64_t* empty = full + STAGES;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j0 = blockIdx.x * BJ;
    const int kt0 = blockIdx.y * k_tiles_per_split;
    const int kt1 = min(k_tiles, kt0 + k_tiles_per_split);
    const int n_iter = max(0, kt1 - kt0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumers);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kConsumers) {
        if (lane == 0) {
            tma_prefetch_desc(&mapA);
            tma_prefetch_desc(&mapW);
            for (int it = 0; it < n_iter; ++it) {
                const int s = it % STAGES;
                if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
                char* st = smem + s * kStage;
                mbar_arrive_expect_tx(&full[s], kStage);
                const int k = (kt0 + it) * kBK;
#pragma unroll
                for (int bx = 0; bx < kABoxes; ++bx)
                    tma_load_2d(st + bx * kBox, &mapA, &full[s], j0 + 16 * bx, k);
#pragma unroll
                for (int bx = 0; bx < kWBoxes; ++bx)
                    tma_load_2d(st + (kABoxes + bx) * kBox, &mapW, &full[s], 16 * bx, k);
            }
        }
        return;
    }

    // TAIL: warps w and w + 4 (one scheduler) get different warp columns
    const int wm = TAIL ? warp % WM : warp / WN, wn = TAIL ? warp / WM : warp % WN;
    const int g = lane >> 2, t = lane & 3;
    double* out = Z + blockIdx.y * split_stride;
    // the tail tile (warp column 1's last, ni = NI - 1): its accumulator slots hold the
    // current stage's partial sums p[mi][h][c] at acc[mi][NI - 1][2 h + c]
    const bool tail_warp = TAIL > 0 && wn == WN - 1;
    constexpr int c_tail = (NT - 1) * 8;
    double run[2] = {0.0, 0.0};  // lane t's reduced tail sums: mi = t & 1, h = t >> 1
    const int j_run = j0 + wm * (BJ / WM) + (t & 1) * 16 + g + 8 * (t >> 1);
    double acc[MI][NI][4];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;
    if constexpr (OUT_T && ACC) {
        // continue the partial sum a previous launch over the preceding K rows stored
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = j0 + wm * (BJ / WM) + mi * 16 + g + 8 * h;
                if (j < N)
#pragma unroll
                    for (int ni = 0; ni < NI; ++ni) {
                        if (tail_warp && ni == NI - 1) continue;
                        const int c = (wn * NI + ni) * 8 + 2 * t;
                        acc[mi][ni][2 * h] = out[(long)c * ldz + j];
                        acc[mi][ni][2 * h + 1] = out[(long)(c + 1) * ldz + j];
                    }
            }
        if (tail_warp && j_run < N) {
            run[0] = out[(long)c_tail * ldz + j_run];
            run[1] = out[(long)(c_tail + 1) * ldz + j_run];
        }
    }

    for (int it = 0; it < n_iter; ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        const char* st = smem + s * kStage;
#pragma unroll 1
        for (int ks = 0; ks < 2; ++ks) {
            double a[MI][8];
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) {
                const char* boxA = st + (wm * (BJ / WM / 16) + mi) * kBox;
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    const int col = g + 8 * (v & 1);
                    const int row = ks * 16 + k_atx(t, v >> 1);
                    a[mi][v] = lds_f64(boxA, swz128(row, col));
                }
            }
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
                if (tail_warp && ni == NI - 1) {  // warp-uniform
                    // W[k][c_tail .. c_tail + 1] for the thread's 4 k-slots (one 16-byte pair)
                    const char* boxW = st + (kABoxes + (c_tail >> 4)) * kBox;
                    if (ks == 0)
#pragma unroll
                        for (int v = 0; v < 4; ++v) acc[0][ni][v] = acc[1][ni][v] = 0.0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double2 w =
                            lds_f64x2(boxW, swz128(ks * 16 + k_atx(t, q), c_tail & 15));
#pragma unroll
                        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                acc[mi][ni][2 * h] = fma(a[mi][h + 2 * q], w.x, acc[mi][ni][2 * h]);
                                acc[mi][ni][2 * h + 1] =
                                    fma(a[mi][h + 2 * q], w.y, acc[mi][ni][2 * h + 1]);
                            }
                    }
                    continue;
                }
                const int c = (wn * NI + ni) * 8 + g;
                const char* boxW = st + (kABoxes + (c >> 4)) * kBox;
                double b[4];
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int row = ks * 16 + k_atx(t, v);
                    b[v] = lds_f64(boxW, swz128(row, c & 15));
                }
#pragma unroll
                for (int mi = 0; mi < MI; ++mi) dmma_16x8x16(acc[mi][ni], a[mi], b);
            }
        }
        if (tail_warp) {
            // butterfly over the 4 k-lanes: xor 1 keeps mi = t & 1, xor 2 keeps h = t >> 1
            double (&p0)[4] = acc[0][NI - 1];
            double (&p1)[4] = acc[1][NI - 1];
            const bool b0 = t & 1, b1 = t & 2;
            double r1[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const double mine = b0 ? p1[v] : p0[v];
                const double other = b0 ? p0[v] : p1[v];
                r1[v] = mine + __shfl_xor_sync(0xffffffffu, other, 1);
            }
#pragma unroll
            for (int c = 0; c < 2; ++c) {  // r1[2 h + c]
                const double mine = b1 ? r1[2 + c] : r1[c];
                const double other = b1 ? r1[c] : r1[2 + c];
                run[c] += mine + __shfl_xor_sync(0xffffffffu, other, 2);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (tail_warp) {
        // lane t = 0 of each quad takes the tile's columns 0, 1 for (mi, h) from lane mi + 2 h
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const double v = __shfl_sync(0xffffffffu, run[c], (lane & ~3) | (mi + 2 * h));
                    acc[mi][NI - 1][2 * h + c] = t == 0 ? v : 0.0;
                }
    }

#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = j0 + wm * (BJ / WM) + mi * 16 + g + 8 * h;
            if (j < N) {
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) {
                    const int c = (wn * NI + ni) * 8 + 2 * t;
                    if (OUT_T) {
                        out[(long)c * ldz + j] = acc[mi][ni][2 * h];
                        out[(long)(c + 1) * ldz + j] = acc[mi][ni][2 * h + 1];
                    } else {
                        *reinterpret_cast<double2*>(out + (long)j * ldz + c) =
                            make_double2(acc[mi][ni][2 * h], acc[mi][ni][2 * h + 1]);
                    }
                }
            }
        }
    }
}

// Fixed-order sum of split-K slabs: out[e] = sum_s part[s * stride + e]. Threads are
// laid out 32 elements x 8 split-groups; group g sums splits g, g+8, ... and the 8 group
// sums are added in a fixed order, so the result is deterministic.
// (T = float: the FP32 split-K slabs of the 3xTF32 GEMMs, summed in FP64.)
template <typename T>
__global__ void __launch_bounds__(256) reduce_partials_kernel(const T* __restrict__ part,
                                                              long stride, int splits,
                                                              double* __restrict__ out,
                                                              long count) {
    __shared__ double red[8][33];
    const int lx = threadIdx.x & 31, gy = threadIdx.x >> 5;
    for (long base = blockIdx.x * 32L; base < count; base += gridDim.x * 32L) {
        const long e = base + lx;
        double acc = 0.0;
        if (e < count)
            for (int sp = gy; sp < splits; sp += 8) acc += (double)part[sp * stride + e];
        red[gy][lx] = acc;
        __syncthreads();
        if (gy == 0 && e < count) {
            double t = red[0][lx];
#pragma unroll
            for (int q = 1; q < 8; ++q) t += red[q][lx];
            out[e] = t;
        }
        __syncthreads();
    }
}

// The same for many slabs of few elements (the fused-Gram partials: 1583 slabs of 80 x 80
// at C2): 32 elements x 32 split-groups per CTA, four independent loads in flight per
// thread, group sums combined in a fixed order.
template <typename T>
__global__ void __launch_bounds__(1024) reduce_partials_wide_kernel(const T* __restrict__ part,
                                                                    long stride, int splits,
                                                                    double* __restrict__ out,
                                                                    long count) {
    __shared__ double red[32][33];
    const int lx = threadIdx.x & 31, gy = threadIdx.x >> 5;
    for (long base = blockIdx.x * 32L; base < count; base += gridDim.x * 32L) {
        const long e = base + lx;
        double acc = 0.0;
        if (e < count) {
            int sp = gy;
            for (; sp + 96 < splits; sp += 128) {
                const double v0 = (double)part[sp * stride + e];
                const double v1 = (double)part[(sp + 32) * stride + e];
                const double v2 = (double)part[(sp + 64) * stride + e];
                const double v3 = (double)part[(sp + 96) * stride + e];
                acc += v0;
                acc += v1;
                acc += v2;
                acc += v3;
            }
            for (; sp < splits; sp += 32) acc += (double)part[sp * stride + e];
        }
        red[gy][lx] = acc;
        __syncthreads();
        if (gy == 0 && e < count) {
            double t = red[0][lx];
            for (int q = 1; q < 32; ++q) t += red[q][lx];
            out[e] = t;
        }
        __syncthreads();
    }
}

// ================================================================ host launchers
namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// Row-major (rows x cols, ld elements) FP64 matrix, box {16 cols, box_rows rows}, 128B swizzle.
int make_map(CUtensorMap* map, const double* base, long rows, long cols, long ld, int box_rows) {
    auto encode = get_encode();
    if (!encode) return -1;
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * 8) & 15)) return -2;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
    cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -3;
}

template <int BM, int NT, int WM, int WN, int STAGES, bool CHECK, bool RESID = false, int TAIL = 0,
          int SKIP = 0>
cudaError_t launch_ax_t(const GemmAx& p, cudaStream_t st) {
    constexpr int NP = NT * 8;
    constexpr size_t kStage = 2 * BM * 128 + 2 * NP * 128;
    constexpr size_t smem = STAGES * kStage + 2 * STAGES * 8 + 1024;
    auto kern = gemm_ax_kernel<BM, NT, WM, WN, STAGES, CHECK, RESID, TAIL, SKIP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    CUtensorMap mA, mX;
    if (make_map(&mA, p.A, p.M, p.K, p.lda, BM) ||
        make_map(&mX, p.Xt, NP, p.K, p.ldx, NP > 256 ? NP / 2 : NP))
        return cudaErrorInvalidValue;
    const int k_tiles = (int)((p.K + kBK - 1) / kBK);
    const int splits = p.splits < 1 ? 1 : p.splits;
    const int per = (k_tiles + splits - 1) / splits;
    dim3 grid((unsigned)((p.M + BM - 1) / BM), (unsigned)splits);
    if (p.gram && (splits != 1 || NT > 12)) return cudaErrorInvalidValue;
    kern<<<grid, (WM * WN + 1) * 32, smem, st>>>(mA, mX, p.Y, p.ldy, p.split_stride, (int)p.M,
                                                 k_tiles, per, p.flag, p.gram, p.resid,
                                                 p.resid_ld, p.resid_cols, p.resid_out, p.abort);
    return cudaGetLastError();
}

template <int BJ, int NT, int WM, int WN, int STAGES, bool OUT_T, bool ACC = false, int TAIL = 0>
cudaError_t launch_atx_t(const GemmAtx& p, cudaStream_t st) {
    constexpr int NP = NT * 8;
    constexpr size_t kStage = (BJ / 16 + NP / 16) * kBK * 128;
    constexpr size_t smem = STAGES * kStage + 2 * STAGES * 8 + 1024;
    auto kern = gemm_atx_kernel<BJ, NT, WM, WN, STAGES, OUT_T, ACC, TAIL>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    CUtensorMap mA, mW;
    if (make_map(&mA, p.A, p.K, p.N, p.lda, kBK) || make_map(&mW, p.W, p.K, NP, p.ldw, kBK))
        return cudaErrorInvalidValue;
    const int k_tiles = (int)((p.K + kBK - 1) / kBK);
    const int splits = p.splits < 1 ? 1 : p.splits;
    const int per = (k_tiles + splits - 1) / splits;
    dim3 grid((unsigned)((p.N + BJ - 1) / BJ), (unsigned)splits);
    if (ACC && splits != 1) return cudaErrorInvalidValue;
    kern<<<grid, (WM * WN + 1) * 32, smem, st>>>(mA, mW, p.Z, p.ldz, p.split_stride, (int)p.N,
                                                 k_tiles, per, p.abort);
    return cudaGetLastError();
}

}  // namespace

// NP (padded sketch width) dispatch. Widths up to 96 use 128-row tiles with a
// 4x2 warp grid and 4 stages; wider sketches use 64-row tiles, 2x4 warps, 3 stages.
// Tail split for a product whose Xt has nonzero rows only below `cols`: 0 = plain
// DMMA tiles, else 4 * (NT - nd) + tail with nd = cols / 8 DMMA tiles and a DFMA tail of
// 2 or 4 columns (cols % 8 in [1, 4]; NT - nd is 1 or 2 for NP = cols rounded up to 16).
inline int tail_code(int cols, int NT) {
    if (cols <= 0 || cols >= NT * 8) return 0;
    const int r = cols % 8, skip = NT - cols / 8;
    if (r == 0 || r > 4 || skip < 1 || skip > 2) return 0;
    return 4 * skip + (r <= 2 ? 2 : 4);
}

template <int NT, bool CHECK>
cudaError_t launch_ax_tail(const GemmAx& p, cudaStream_t st, int code) {
    switch (code) {
        case 6: return launch_ax_t<128, NT, 8, 1, 4, CHECK, false, 2, 1>(p, st);
        case 8: return launch_ax_t<128, NT, 8, 1, 4, CHECK, false, 4, 1>(p, st);
        case 10: return launch_ax_t<128, NT, 8, 1, 4, CHECK, false, 2, 2>(p, st);
        default: return launch_ax_t<128, NT, 8, 1, 4, CHECK, false, 4, 2>(p, st);
    }
}

template <int NT>
cudaError_t dispatch_ax(const GemmAx& p, cudaStream_t st) {
    if constexpr (NT <= 12) {
        if (const int code = tail_code(p.cols, NT))
            return p.flag ? launch_ax_tail<NT, true>(p, st, code)
                          : launch_ax_tail<NT, false>(p, st, code);
        return p.flag ? launch_ax_t<128, NT, 4, 2, 4, true>(p, st)
                      : launch_ax_t<128, NT, 4, 2, 4, false>(p, st);
    } else if constexpr (NT > 24) {  // sketches wider than 192: 2 stages fit in smem
        return p.flag ? launch_ax_t<64, NT, 4, 4, 2, true>(p, st)
                      : launch_ax_t<64, NT, 4, 4, 2, false>(p, st);
    } else {
        return p.flag ? launch_ax_t<64, NT, 2, 4, 3, true>(p, st)
                      : launch_ax_t<64, NT, 2, 4, 3, false>(p, st);
    }
}

// atx: the last column tile holds at most 2 of the cols nonzero W columns (s % 8 in {1, 2}
// with NP = round_up(s, 16) - 8 < s): DFMA tail variant.
inline bool atx_tail(int cols, int NT) {
    return NT <= 12 && cols > (NT - 1) * 8 && cols <= (NT - 1) * 8 + 2;
}

template <int NT>
cudaError_t dispatch_atx(const GemmAtx& p, cudaStream_t st) {
    if constexpr (NT <= 12) {
        if (atx_tail(p.cols, NT)) {
            if (p.accumulate || p.out_transposed) {
                if (!p.out_transposed) return cudaErrorInvalidValue;
                return p.accumulate ? launch_atx_t<128, NT, 4, 2, 4, true, true, 2>(p, st)
                                    : launch_atx_t<128, NT, 4, 2, 4, true, false, 2>(p, st);
            }
            return launch_atx_t<128, NT, 4, 2, 4, false, false, 2>(p, st);
        }
    }
    if (p.accumulate) {  // upload segments (rsvd_b200.cpp gemm_ax_chunked): Z^T only
        if (!p.out_transposed) return cudaErrorInvalidValue;
        if constexpr (NT <= 12)
            return launch_atx_t<128, NT, 4, 2, 4, true, true>(p, st);
        else if constexpr (NT > 24)
            return launch_atx_t<64, NT, 4, 4, 2, true, true>(p, st);
        else
            return launch_atx_t<64, NT, 2, 4, 3, true, true>(p, st);
    }
    if constexpr (NT <= 12) {
        return p.out_transposed ? launch_atx_t<128, NT, 4, 2, 4, true>(p, st)
                                : launch_atx_t<128, NT, 4, 2, 4, false>(p, st);
    } else if constexpr (NT > 24) {
        return p.out_transposed ? launch_atx_t<64, NT, 4, 4, 2, true>(p, st)
                                : launch_atx_t<64, NT, 4, 4, 2, false>(p, st);
    } else {
        return p.out_transposed ? launch_atx_t<64, NT, 2, 4, 3, true>(p, st)
                                : launch_atx_t<64, NT, 2, 4, 3, false>(p, st);
    }
}

cudaError_t launch_gemm_ax(const GemmAx& p, cudaStream_t st) {
    if (p.resid) {  // fused residual chunk: NP = 96 tiles, no split, no flag / Gram
        if (p.NP != 96 || p.splits > 1 || p.gram || p.flag) return cudaErrorInvalidValue;
        return launch_ax_t<128, 12, 4, 2, 4, false, true>(p, st);
    }
    switch (p.NP / 8) {
        case 2: return dispatch_ax<2>(p, st);
        case 4: return dispatch_ax<4>(p, st);
        case 6: return dispatch_ax<6>(p, st);
        case 8: return dispatch_ax<8>(p, st);
        case 10: return dispatch_ax<10>(p, st);
        case 12: return dispatch_ax<12>(p, st);
        case 16: return dispatch_ax<16>(p, st);
        case 20: return dispatch_ax<20>(p, st);
        case 24: return dispatch_ax<24>(p, st);
        case 28: return dispatch_ax<28>(p, st);
        case 32: return dispatch_ax<32>(p, st);
        case 36: return dispatch_ax<36>(p, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_gemm_atx(const GemmAtx& p, cudaStream_t st) {
    switch (p.NP / 8) {
        case 2: return dispatch_atx<2>(p, st);
        case 4: return dispatch_atx<4>(p, st);
        case 6: return dispatch_atx<6>(p, st);
        case 8: return dispatch_atx<8>(p, st);
        case 10: return dispatch_atx<10>(p, st);
        case 12: return dispatch_atx<12>(p, st);
        case 16: return dispatch_atx<16>(p, st);
        case 20: return dispatch_atx<20>(p, st);
        case 24: return dispatch_atx<24>(p, st);
        case 28: return dispatch_atx<28>(p, st);
        case 32: return dispatch_atx<32>(p, st);
        case 36: return dispatch_atx<36>(p, st);
        default: return cudaErrorInvalidValue;
    }
}

template <typename T>
static cudaError_t launch_reduce_t(const T* part, long stride, int splits, double* out, long count,
                                   cudaStream_t st) {
    long blocks = (count + 31) / 32;
    if (splits >= 128 && blocks <= 148 * 4) {  // few elements, many slabs
        reduce_partials_wide_kernel<T><<<(unsigned)std::max(1L, blocks), 1024, 0, st>>>(
            part, stride, splits, out, count);
        return cudaGetLastError();
    }
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    reduce_partials_kernel<T><<<(unsigned)blocks, 256, 0, st>>>(part, stride, splits, out, count);
    return cudaGetLastError();
}

cudaError_t launch_reduce_partials(const double* part, long stride, int splits, double* out,
                                   long count, cudaStream_t st) {
    return launch_reduce_t(part, stride, splits, out, count, st);
}

cudaError_t launch_reduce_partials_f32(const float* part, long stride, int splits, double* out,
                                       long count, cudaStream_t st) {
    return launch_reduce_t(part, stride, splits, out, count, st);
}

}  // namespace rsvdb200

// ===================================================================== peak probe
namespace rsvdb200 {

// FP64 tensor-pipe issue rate: every warp runs independent m16n8k16 DMMA chains on
// register operands (no memory traffic), 2 CTAs x 8 warps per SM. The roofline
// denominator for the passes over A (MEASURED_PEAKS.json has no FP64 entry).
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
    double acc[4][4];
    double a[8], b[4];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[t][r] = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = (threadIdx.x + i) * 1e-3;
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = (threadIdx.x - i) * 1e-3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 4; ++t) dmma_16x8x16(acc[t], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int r = 0; r < 4; ++r) s += acc[t][r];
    if (s == 1234.5) out[0] = s;  // keep the chains alive
}

cudaError_t measure_dmma_peak(cudaStream_t st, double* tflops) {
    double* out = nullptr;
    cudaError_t e = cudaMalloc(&out, sizeof(double));
    if (e != cudaSuccess) return e;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = 148 * 2, iters = 4096;
    dmma_peak_kernel<<<grid, 256, 0, st>>>(out, iters);  // warm-up (clocks up)
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0, st);
        dmma_peak_kernel<<<grid, 256, 0, st>>>(out, iters);
        cudaEventRecord(e1, st);
        e = cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flop = 2.0 * 16 * 8 * 16 * 4.0 * iters * grid * (256 / 32);
    *tflops = flop / (best * 1e-3) / 1e12;
    return e;
}

}  // namespace rsvdb200
