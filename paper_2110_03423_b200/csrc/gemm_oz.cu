// FP64 GEMMs of the rSVD passes over A on the INT8 tensor cores (tcgen05 kind::i8), by the
// Ozaki scheme: exact integer products of fixed-point digit slices, accumulated exactly in
// int32 in TMEM, recombined in FP64 once per output tile.
//
// Why: B200's FP64 tensor path (DMMA, gemm_f64.cu) peaks at ~37 TFLOP/s, and every pass over A
// of Algorithm 1 is bound by it (arithmetic intensity s/4 flop/B against a ridge of ~5.6). The
// INT8 tensor cores run 4.5 POPS dense. Splitting each FP64 operand into S = 7 signed 8-bit
// digits of a common per-row (per-column) fixed-point scale,
//     x = 2^(E - 53) * sum_{i<7} d_i 256^i,   d_i in [-128, 127],  |x| < 2^(E + 1),
// turns a row of A times a column of B into sum_{i,j} (d_i . e_j) 256^(i+j) 2^(E_a + E_b - 106)
// with every d_i . e_j an exact int8 dot product. The 28 digit products with i + j >= 6 are
// kept (the dropped ones weigh <= 2^-47 of the leading term); products of equal weight
// g = i + j share one int32 accumulator (|sum| <= 7 * 2^14 * K < 2^31 for K <= 16384), so a
// tile needs 7 accumulators of N columns in TMEM. Error: the fixed-point rounding of each
// operand (2^-54 of the row / column maximum) plus the truncation, i.e. the normwise error of
// an FP64 GEMM (measured against an exact long-double product: Frobenius-relative 1.1e-15
// against 6.6e-16 for FP64 BLAS on the C2 operand shapes, tests/test_gpu_oz.py), with no
// rounding at all along K.
//
// Shapes (the two the FP64 path has):
//   ax  : Y (M x NP) = A (M x K row-major) X, per-row scales of A (a_ef[M]); X as digit
//         planes of X^T (NP x K) with per-column scales (b_ef[NP]).
//   atx : Z = A^T W, A (K x M row-major) read in place; W as digit planes of W^T (NP x K).
//         Output Z^T (NP x M) or Z.
// Two forms of A's digits:
//   * stored (the optimistic pipeline's default, gemm_ozd_kernel): one pass over A per row
//     chunk (oz_scan_convert_kernel, or oz_scan + oz_convert_tiles for rows wider than 4608)
//     writes A's row-scaled digits pre-tiled for both shapes, and every pass bulk-copies them
//     (no FP64 tile, no conversion in the GEMM). The atx shape folds A's row scales into W
//     (W' = diag(2^(E_k - 53)) W, exact powers of two).
//   * in-kernel (gemm_oz_kernel: the robust rerun, or when the stored planes do not fit HBM):
//     converter warps form the digits of the TMA'd FP64 tile and write them straight into TMEM
//     for TS MMAs; per-column scales of A for the atx shape (oz_scan).
// The small operand's digits come from a prep kernel (launch_oz_digits_*).
//
// TMEM holds 7 x N int32 accumulator columns (plus, in-kernel, the A-digit buffers), so N <= 48
// per CTA: wider sketches run as column chunks of <= 48 whose CTAs share the A tile (stored:
// cluster multicast of the digit blocks; in-kernel: L2). MMAs: the 28 digit products issued as
// 9 wide MMAs (digit i of A against B's planes 6 - i .. 6 laid out back to back), one elected
// lane of a converged warp issuing. UMMA operands: K-major SWIZZLE_32B (rows of 32 int8 = one
// K = 32 MMA step, 8-row atoms of 256 B, 16-byte chunk c of row r stored at chunk
// c ^ ((r >> 2) & 1)); the stored atx blocks are MN-major SWIZZLE_128B.
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace rsvdb200 {
namespace oz {

constexpr int kDigits = 7;        // S
constexpr int kGroups = 7;        // g = i + j in [S - 1, 2S - 2]
constexpr int BM = 128;           // MMA M (rows of the tile)
constexpr int BK = 32;            // K per stage = one kind::i8 MMA
#ifndef OZ_FSTAGES
#define OZ_FSTAGES 4
#endif
#ifndef OZ_BSTAGES
#define OZ_BSTAGES 4
#endif
constexpr int kFStages = OZ_FSTAGES;  // FP64 A ring (TMA -> converters)
constexpr int kDStages = 3;       // A digits in TMEM (converters -> MMA): 7 N + 3 x 56 <= 512 columns
constexpr int kBStages = OZ_BSTAGES;  // B digit planes in shared memory (TMA -> MMA)
constexpr int kConvWarps = 8;     // warps 3..10: (row, k-half) per thread
constexpr int kThreads = 96 + 32 * kConvWarps;
constexpr int kMaxN = 48;         // columns per CTA: 7 accumulators of N + 3 x 56 digit columns
constexpr int kMaxChunks = 8;
constexpr uint32_t kAF64 = BM * BK * 8;       // 32 KB FP64 A tile
constexpr uint32_t kDigCols = BK / 4;         // TMEM columns of one A digit tile (4 int8 each)
constexpr uint32_t kBDigMax = kMaxN * BK;     // 1.5 KB per B digit plane (N <= 48)
constexpr uint32_t kBStage = kDigits * kBDigMax;  // 10752 B
constexpr uint32_t kRing = kFStages * kAF64 + kBStages * kBStage;  // 174080 B
constexpr uint64_t kDigitBias = 0x0080808080808080ull;  // sum_{i<7} 128 * 256^i

// SW32 K-major byte offset of (row r, 16-byte chunk c) in a digit tile
__device__ __forceinline__ uint32_t sw32(uint32_t r, uint32_t c) {
    return (r >> 3) * 256u + (r & 7u) * 32u + ((c ^ ((r >> 2) & 1u)) << 4);
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    // start, LBO 16 B (unused for a swizzled K-major operand of K = one swizzle row), SBO 256 B
    // (8-row atoms), version 1, layout SWIZZLE_32B (6)
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) |
           ((uint64_t)(256u >> 4) << 32) | (1ull << 46) | (6ull << 61);
}

// kind::i8 instruction descriptor: D s32, A s8, B s8, K-major both, M = 128, N
__device__ __forceinline__ uint32_t idesc(int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}

// A operand from TMEM (128 lanes = rows, 8 columns = 32 int8 of K), B from shared memory
__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id,
                                          uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}

// shared -> TMEM copy of a 128-row x 32-byte tile described by a matrix descriptor (the A
// operand of the following TS MMAs; executes in order with them)
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc_) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc_) : "memory");
}

__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c,
                                         uint32_t d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
                 "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

// 3-D TMA load broadcast to the same smem offset of every CTA in `mask` (complete_tx on the
// barrier at the same offset in each)
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* map, uint64_t* bar,
                                               int c0, int c1, int c2, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
        "h"(mask)
        : "memory");
}

// 1-D bulk copy global -> shared (bytes a multiple of 16), complete_tx on `bar`; the multicast
// form lands at the same offset of every CTA in `mask`
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_load_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(src)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"(mask)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d_mc_oz(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                  int c_inner, int c_outer, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c_inner), "r"(c_outer),
        "h"(mask)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_remote(uint32_t caddr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr)
                 : "memory");
}


__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = (int)r[i];
}

// The 7 digits of x at the fixed-point scale of biased exponent `ef_max` (the row / column
// maximum): X = round(x * 2^(53 - E)), |X| < 2^54; returns the bytes of (X + bias) ^ bias,
// i.e. byte i = d_i as int8 (balanced base-256 digits; byte 7 is 0). Zero / subnormal x -> 0.
__device__ __forceinline__ uint64_t digits_of(double x, int ef_max) {
    const uint64_t bits = (uint64_t)__double_as_longlong(x);
    const int ef = (int)((bits >> 52) & 0x7ff);
    const uint64_t m53 = (bits & 0x000FFFFFFFFFFFFFull) | 0x0010000000000000ull;
    const int d = min(max(ef_max - ef, 0), 63);  // ef <= ef_max
    uint64_t mag = m53 << 1;                     // X = m53 * 2^(1 - d), rounded to nearest
    if (d > 0) mag = (mag + (1ull << (d - 1))) >> d;
    if (ef == 0) mag = 0;
    const uint64_t X = (bits >> 63) ? (0ull - mag) : mag;
    return (X + kDigitBias) ^ kDigitBias;
}

// The fixed-point scale 2^(53 - E) of a row / column with maximum biased exponent ef_max, as
// two exactly representable factors (2^(1076 - ef_max) itself over- or underflows at the ends
// of the exponent range); 0 for an all-zero row.
__device__ __forceinline__ void fixed_scale(int ef_max, double& f1, double& f2) {
    const int e = 1076 - ef_max, e1 = e / 2, e2 = e - e1;
    f1 = ef_max == 0 ? 0.0 : __longlong_as_double((long long)(e1 + 1023) << 52);
    f2 = ef_max == 0 ? 0.0 : __longlong_as_double((long long)(e2 + 1023) << 52);
}

// digits_of with the scale applied on the FP64 pipe: (x f1) f2 is x 2^(53 - E) exactly, and
// the conversion rounds it to the nearest integer X (ties to even, where the integer path above
// rounds ties away from zero; the same X otherwise).
__device__ __forceinline__ uint64_t digits_scaled(double x, double f1, double f2) {
    const long long X = __double2ll_rn((x * f1) * f2);
    return (uint64_t)X + kDigitBias;  // the bias XOR is applied to the packed plane words
}

__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    while (!done) {
        __nanosleep(64);
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

// 4 consecutive k elements (digit words w[0..3]) -> 7 plane words (byte lane = k)
__device__ __forceinline__ void planes4(const uint64_t (&w)[4], uint32_t (&out)[kDigits]) {
    const uint32_t l0 = (uint32_t)w[0], l1 = (uint32_t)w[1], l2 = (uint32_t)w[2], l3 = (uint32_t)w[3];
    const uint32_t h0 = (uint32_t)(w[0] >> 32), h1 = (uint32_t)(w[1] >> 32),
                   h2 = (uint32_t)(w[2] >> 32), h3 = (uint32_t)(w[3] >> 32);
    uint32_t a = __byte_perm(l0, l1, 0x5140), b = __byte_perm(l2, l3, 0x5140);
    out[0] = __byte_perm(a, b, 0x5410);
    out[1] = __byte_perm(a, b, 0x7632);
    a = __byte_perm(l0, l1, 0x7362);
    b = __byte_perm(l2, l3, 0x7362);
    out[2] = __byte_perm(a, b, 0x5410);
    out[3] = __byte_perm(a, b, 0x7632);
    a = __byte_perm(h0, h1, 0x5140);
    b = __byte_perm(h2, h3, 0x5140);
    out[4] = __byte_perm(a, b, 0x5410);
    out[5] = __byte_perm(a, b, 0x7632);
    a = __byte_perm(h0, h1, 0x7362);
    b = __byte_perm(h2, h3, 0x7362);
    out[6] = __byte_perm(a, b, 0x5410);
}

struct BMaps {  // one B digit-plane map per column chunk (box rows = the chunk's N)
    CUtensorMap m[kMaxChunks];
};

// MN = false (ax): A tile = 128 rows x 32 k (two 16-wide SW128 boxes), converter thread = row.
// MN = true (atx): A tile = 32 k-rows x 128 columns (eight 16-wide boxes), thread = column.
// The FP64 A tiles come through a 4-stage TMA ring; the converters write A's digit tiles
// straight into TMEM (tcgen05.st, double-buffered after the accumulators), where the MMA reads
// them as its A operand, so shared memory carries only the FP64 tile and the B digit planes
// (4-stage TMA ring). Warps: 0 A producer, 1 TMEM owner + MMA issuer, 2 B producer,
// 3..10 converters / epilogue (thread = TMEM lane = tile row, and a k-half).
template <bool MN, bool OUT_T>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_oz_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ BMaps bmaps,
                   const int* __restrict__ a_ef, const int* __restrict__ b_ef, int M, int NP,
                   int nch, int nfirst, double* __restrict__ out, long ldo, long split_stride,
                   int k_tiles, int k_tiles_per_split, const int* __restrict__ abort_flag,
                   int diag, int mc) {
    if (abort_flag && *(const volatile int*)abort_flag) return;
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = align_smem_1024(smem_raw);
    char* ringA = smem;
    char* ringB = smem + kFStages * kAF64;
    uint64_t* full_a = reinterpret_cast<uint64_t*>(smem + kRing);
    uint64_t* empty_a = full_a + kFStages;
    uint64_t* full_b = empty_a + kFStages;
    uint64_t* empty_b = full_b + kBStages;
    uint64_t* conv = empty_b + kBStages;
    uint64_t* empty_d = conv + kDStages;
    uint64_t* accum = empty_d + kDStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncl = mc ? nch : 1;             // cluster size (multicast of the FP64 tile)
    const int ch = blockIdx.x % nch;          // column chunk
    const int tile = blockIdx.x / nch;
    const int m0 = tile * BM;
    const int c0 = ch * nfirst;
    const int N = min(nfirst, NP - c0);       // multiple of 16
    const uint32_t pb = (uint32_t)N * BK;     // bytes of one B digit plane
    const uint32_t dcol0 = (uint32_t)(kGroups * N);  // TMEM column of the A digit buffers
    const int kt0 = blockIdx.y * k_tiles_per_split;
    const int kt1 = min(k_tiles, kt0 + k_tiles_per_split);
    const int n_iter = max(0, kt1 - kt0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kFStages; ++s) {
            mbar_init(&full_a[s], 1);
            mbar_init(&empty_a[s], kConvWarps * ncl);  // every CTA's converters of the cluster
        }
        for (int s = 0; s < kBStages; ++s) {
            mbar_init(&full_b[s], 1);
            mbar_init(&empty_b[s], 1);
        }
        for (int s = 0; s < kDStages; ++s) {
            mbar_init(&conv[s], kConvWarps);
            mbar_init(&empty_d[s], 1);
        }
        mbar_init(accum, 1);
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    if (ncl > 1)
        cluster_sync_all();  // every CTA's barriers exist before a multicast targets them
    else
        __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint16_t cmask = (uint16_t)((1u << ncl) - 1u);
    const int crank = ncl > 1 ? ch : 0;

    if (warp == 0) {
        // ------------------------------------------------------------ A producer
        // the column-chunk CTAs of a tile form a cluster: rank ch loads the FP64 boxes
        // b = ch, ch + nch, ... and multicasts them, so the tile crosses L2 -> SM once; a stage
        // is refilled once the converters of every CTA hold it in registers
        if (lane == 0) {
            tma_prefetch_desc(&mapA);
            for (int it = 0; it < n_iter; ++it) {
                const int s = it % kFStages;
                if (it >= kFStages) mbar_wait_sleep(&empty_a[s], ((it / kFStages) - 1) & 1);
                char* st = ringA + s * kAF64;
                const int k = (kt0 + it) * BK;
                mbar_arrive_expect_tx(&full_a[s], kAF64);
                constexpr int nbox = MN ? BM / 16 : 2;
                constexpr uint32_t bbytes = kAF64 / nbox;
                for (int bx = crank; bx < nbox; bx += ncl) {
                    const int x = MN ? m0 + 16 * bx : k + 16 * bx, y = MN ? k : m0;
                    if (ncl > 1)
                        tma_load_2d_mc_oz(st + bx * bbytes, &mapA, &full_a[s], x, y, cmask);
                    else
                        tma_load_2d(st + bx * bbytes, &mapA, &full_a[s], x, y);
                }
            }
        }
    } else if (warp == 2) {
        // ---------------------------------------- B producer: digit planes back to back
        // (plane j at rows j N) so that MMA i reads planes 6 - i .. 6 as one operand
        if (lane == 0) {
            const CUtensorMap* mb = &bmaps.m[ch];
            tma_prefetch_desc(mb);
            for (int it = 0; it < n_iter; ++it) {
                const int s = it % kBStages;
                if (it >= kBStages) mbar_wait_sleep(&empty_b[s], ((it / kBStages) - 1) & 1);
                char* sb = ringB + s * kBStage;
                const int k = (kt0 + it) * BK;
                mbar_arrive_expect_tx(&full_b[s], kDigits * pb);
#pragma unroll
                for (int i = 0; i < kDigits; ++i)
                    tma_load_2d(sb + i * pb, mb, &full_b[s], k, i * NP + c0);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------- MMA issuer
        // digit i of A times planes j = 6 - i .. 6 of B in one operand: output block b (plane
        // 6 - i + b) is group g = i + j - 6 = b, TMEM columns [b N, (b + 1) N) for every i.
        // i = 6 covers all 7 groups and goes first (it initialises them in the first stage);
        // operands wider than 256 columns are issued in two MMAs. The 9 (or fewer) MMAs' B
        // descriptor offsets, instruction descriptors and TMEM addresses are set up once.
        // the whole warp runs the loop (warp-uniform control flow keeps the descriptors and
        // TMEM addresses in uniform registers); one elected lane issues
        // MMA list (compile-time shape): digit i, first plane offset (in planes), planes, TMEM
        // column offset (in units of N); i = 6 and 5 split in two (N <= 48 keeps every operand
        // <= 256 columns)
        constexpr int kNM = 9;
        constexpr int mi[kNM] = {6, 6, 5, 5, 4, 3, 2, 1, 0};
        constexpr int mp0[kNM] = {0, 4, 1, 4, 2, 3, 4, 5, 6};  // first plane j
        constexpr int mnp[kNM] = {4, 3, 3, 3, 5, 4, 3, 2, 1};  // planes
        constexpr int mdc[kNM] = {0, 4, 0, 3, 0, 0, 0, 0, 0};  // TMEM column block
        uint32_t idv[kNM];
#pragma unroll
        for (int j = 0; j < kNM; ++j) idv[j] = idesc(mnp[j] * N);
        const uint64_t bdesc0 = sdesc(smem_u32(ringB));
        for (int it = 0; it < n_iter; ++it) {
            const int sb = it % kBStages, sd = it % kDStages;
            const uint64_t bd = bdesc0 + ((uint64_t)(sb * kBStage) >> 4);
            const uint32_t ad = tmem + dcol0 + (uint32_t)sd * (kDigits * kDigCols);
            if (!(diag & 1)) mbar_wait(&full_b[sb], (it / kBStages) & 1);
            mbar_wait(&conv[sd], (it / kDStages) & 1);
            fence_after();
            if (elect_one()) {
#pragma unroll
                for (int j = 0; j < kNM; ++j)
                    mma_i8_ts(tmem + (uint32_t)(mdc[j] * N), ad + (uint32_t)mi[j] * kDigCols,
                              bd + (((uint64_t)mp0[j] * pb) >> 4), idv[j],
                              (it > 0 || j > 1) ? 1u : 0u);
                commit(&empty_b[sb]);
                commit(&empty_d[sd]);
            }
            __syncwarp();
        }
        if (n_iter > 0 && elect_one()) commit(accum);
        __syncwarp();
    } else {
        // ------------------------------------------- converters (warps 3..10)
        // thread -> tile row r (ax) / tile column r (atx) = its TMEM lane, and a k-half h
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int r = 32 * q + lane, h = (warp - 3) >> 2;
        const uint32_t tlane = tmem + ((uint32_t)(32 * q) << 16);
        const int grow = m0 + r;
        const int efm = grow < M ? a_ef[grow] : 0;
        double f1, f2;
        fixed_scale(efm, f1, f2);
        for (int it = 0; it < n_iter; ++it) {
            const int sa = it % kFStages, sd = it % kDStages;
            if (!(diag & 2)) mbar_wait(&full_a[sa], (it / kFStages) & 1);
            const char* st = ringA + sa * kAF64;
            double v[16];
            if constexpr (!MN) {
                const char* box = st + h * (kAF64 / 2);
#pragma unroll
                for (int e = 0; e < 16; e += 2) {
                    const double2 t = *reinterpret_cast<const double2*>(box + swz128(r, e));
                    v[e] = t.x;
                    v[e + 1] = t.y;
                }
            } else {
                const char* box = st + (r >> 4) * (kAF64 / 8);
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    v[e] = *reinterpret_cast<const double*>(box + swz128(h * 16 + e, r & 15));
            }
            if (ncl > 1) {
                // the FP64 tile is in registers: release it in every CTA of the cluster. A
                // release.cluster arrive costs a GPU-scope fence per warp and stage (measured:
                // membar stalls doubled the kernel); a relaxed arrive after the registers have
                // landed (the volatile moves wait on the shared-memory loads' scoreboard)
                // orders the reads before the producer's refill just the same
                uint64_t sink = 0;
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    asm volatile("xor.b64 %0, %0, %1;" : "+l"(sink) : "l"(__double_as_longlong(v[e])));
                asm volatile("" ::"l"(sink));
                __syncwarp();
                if (lane < ncl)
                    asm volatile(
                        "mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                            mapa_rank(smem_u32(&empty_a[sa]), (uint32_t)lane))
                        : "memory");
            } else {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_a[sa]);
            }
            uint32_t pw[kDigits][4];
            if (diag & 4) {
#pragma unroll
                for (int i = 0; i < kDigits; ++i)
#pragma unroll
                    for (int qd = 0; qd < 4; ++qd) pw[i][qd] = __double2loint(v[qd + i]);
            } else {
#pragma unroll
            for (int qd = 0; qd < 4; ++qd) {  // 4 consecutive k
                uint64_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) w[e] = digits_scaled(v[4 * qd + e], f1, f2);
                uint32_t pl[kDigits];
                planes4(w, pl);
#pragma unroll
                for (int i = 0; i < kDigits; ++i) pw[i][qd] = pl[i] ^ 0x80808080u;
            }
            }
            if (it >= kDStages) {
                mbar_wait(&empty_d[sd], ((it / kDStages) - 1) & 1);
                fence_after();
            }
            const uint32_t tb = tlane + dcol0 + (uint32_t)sd * (kDigits * kDigCols) + 4u * h;
#pragma unroll
            for (int i = 0; i < kDigits; ++i)
                tmem_st4(tb + (uint32_t)i * kDigCols, pw[i][0], pw[i][1], pw[i][2], pw[i][3]);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&conv[sd]);
        }

        // ------------------------------------------------------------ epilogue
        if (n_iter > 0) {
            mbar_wait(accum, 0);
            fence_after();
        }
        // the two warps of a lane quarter split the 16-column chunks
        double* ob = out + (size_t)blockIdx.y * split_stride;
        for (int cc = 16 * h; cc < N; cc += 32) {
            double y[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) y[i] = 0.0;
            if (n_iter > 0) {
                // t = sum_g G_g 256^g, most significant group first (Horner)
#pragma unroll
                for (int g = kGroups - 1; g >= 0; --g) {
                    int vv[16];
                    tmem_ld16(tlane + (uint32_t)(g * N + cc), vv);
#pragma unroll
                    for (int i = 0; i < 16; ++i) y[i] = fma(y[i], 256.0, (double)vv[i]);
                }
            }
            if (grow < M) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int c = c0 + cc + i;
                    // y_true = t * 2^(E_a + E_b - 58), E = ef - 1023
                    const double val = y[i] == 0.0 ? 0.0 : ldexp(y[i], efm + b_ef[c] - 2104);
                    if constexpr (OUT_T)
                        ob[(size_t)c * ldo + grow] = val;
                    else
                        ob[(size_t)grow * ldo + c] = val;
                }
            }
        }
    }
    fence_before();
    if (ncl > 1)
        cluster_sync_all();  // no multicast or remote arrive is still in flight into a peer
    else
        __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ------------------------------------------------------------------ digit preparation
// Biased exponent of the largest |x| of each row of a row-major (rows x cols) matrix, the
// largest over rows of each column, and the NaN/Inf flag, in one pass: CTA (cb, rb) covers
// columns [512 cb, 512 cb + 512) of rows [R rb, R rb + R); each warp owns 64 columns (one
// double2 per lane per row). Partial maxima go to row_part[cb][r] / col_part[rb][c] (the
// exponent field in place, bits 20-30 of the high word) and are reduced by oz_reduce_max.
constexpr int kScanRows = 512;

__global__ void __launch_bounds__(256) oz_scan_kernel(const double* __restrict__ A, long rows,
                                                      long cols, long lda, int* __restrict__ row_part,
                                                      int* __restrict__ col_part,
                                                      int* __restrict__ flag) {
    __shared__ int rmax[kScanRows];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long r0 = (long)blockIdx.y * kScanRows;
    const long c = (long)blockIdx.x * 512 + warp * 64 + 2 * lane;
    for (int i = threadIdx.x; i < kScanRows; i += 256) rmax[i] = 0;
    __syncthreads();
    uint32_t cm0 = 0, cm1 = 0;
    bool bad = false;
    const long r1 = min(rows, r0 + kScanRows);
    for (long r = r0; r < r1; ++r) {
        uint32_t h0 = 0, h1 = 0;
        const double* row = A + r * lda;
        if (c + 1 < cols) {
            const double2 v = *reinterpret_cast<const double2*>(row + c);
            h0 = (uint32_t)__double2hiint(v.x) & 0x7ff00000u;
            h1 = (uint32_t)__double2hiint(v.y) & 0x7ff00000u;
        } else if (c < cols) {
            h0 = (uint32_t)__double2hiint(row[c]) & 0x7ff00000u;
        }
        cm0 = max(cm0, h0);
        cm1 = max(cm1, h1);
        uint32_t rv = max(h0, h1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rv = max(rv, __shfl_xor_sync(0xffffffffu, rv, o));
        if (lane == 0) atomicMax(&rmax[r - r0], (int)rv);
    }
    bad = cm0 == 0x7ff00000u || cm1 == 0x7ff00000u;
    __syncthreads();
    for (long r = r0 + threadIdx.x; r < r1; r += 256) {
        row_part[(long)blockIdx.x * rows + r] = rmax[r - r0];
        bad |= rmax[r - r0] == 0x7ff00000;
    }
    if (c < cols) col_part[(long)blockIdx.y * cols + c] = (int)cm0;
    if (c + 1 < cols) col_part[(long)blockIdx.y * cols + c + 1] = (int)cm1;
    if (flag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
}

// out[e] = max_p part[p * count + e] >> 20 (the biased exponent); acc: max with out[e]
__global__ void oz_reduce_max_kernel(const int* __restrict__ part, int parts, long count,
                                     int* __restrict__ out, int acc) {
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < count;
         e += (long)gridDim.x * blockDim.x) {
        int m = 0;
        for (int p = 0; p < parts; ++p) m = max(m, part[(long)p * count + e]);
        out[e] = acc ? max(out[e], m >> 20) : m >> 20;
    }
}

// Digit planes dig[i][c][k] (i < 7, c < NP, k < ldb bytes) of the rows of Xt (NP x K, ldx;
// rows >= cols zero), each row at its own scale b_ef[c]. One CTA per row.
// Byte offset of digit plane i, row c, byte k of the small operand: the plain layout
// [i][c][k] (nfirst = 0: the in-kernel-digit GEMM's TMA boxes) or the stored-digit GEMM's
// tiled one (nfirst = its column-chunk width): per k-tile kt, per chunk, the 7 planes of the
// chunk's N rows x 32 B back to back in the SW32 K-major layout, so that one bulk copy moves a
// stage.
__device__ __forceinline__ long b_offset(int i, int c, long k, int NP, long ldb, int nfirst) {
    if (nfirst == 0) return ((long)i * NP + c) * ldb + k;
    const int ch = c / nfirst, cl = c - ch * nfirst, n = min(nfirst, NP - ch * nfirst);
    const long kt = k >> 5;
    return kt * kDigits * NP * BK + (long)kDigits * BK * ch * nfirst + (long)i * n * BK +
           sw32((uint32_t)cl, (uint32_t)((k >> 4) & 1)) + (k & 15);
}

__global__ void __launch_bounds__(256) oz_digits_rows_kernel(const double* __restrict__ Xt, long ldx,
                                                            int NP, int cols, long K,
                                                            uint8_t* __restrict__ dig, long ldb,
                                                            int* __restrict__ b_ef, int nfirst) {
    const int c = blockIdx.x;
    __shared__ int red[8];
    const double* row = Xt + (long)c * ldx;
    uint32_t m = 0;
    if (c < cols)
        for (long k = threadIdx.x; k < K; k += 256)
            m = max(m, (uint32_t)__double2hiint(row[k]) & 0x7ff00000u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = (int)m;
    __syncthreads();
    int ef = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) ef = max(ef, red[w]);
    ef >>= 20;
    if (threadIdx.x == 0) b_ef[c] = ef;
    for (long k4 = threadIdx.x * 4L; k4 < ldb; k4 += 1024) {
        uint64_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
            w[e] = (c < cols && k4 + e < K) ? digits_of(row[k4 + e], ef) : 0ull;
        uint32_t pl[kDigits];
        planes4(w, pl);
#pragma unroll
        for (int i = 0; i < kDigits; ++i)
            *reinterpret_cast<uint32_t*>(dig + b_offset(i, c, k4, NP, ldb, nfirst)) = pl[i];
    }
}

// Column maxima of W (K x NP row-major, columns >= cols zero) into colmax[NP] (hi-word
// exponent fields, atomicMax; colmax zeroed by the caller).
// row scale of W' = diag(2^(row_ef[k] - 1076)) W (stored-digit atx passes), 1 without row_ef
__device__ __forceinline__ double row_scale(const int* row_ef, long k) {
    if (!row_ef) return 1.0;
    const int e = row_ef[k] - 1076 + 1023;  // biased exponent of 2^(E_k - 53)
    return e >= 1 ? __longlong_as_double((long long)e << 52) : 0.0;
}

__global__ void __launch_bounds__(256) oz_colmax_kernel(const double* __restrict__ W, long ldw, int NP,
                                                       int cols, long K, int* __restrict__ colmax,
                                                       const int* __restrict__ row_ef) {
    // thread -> one column of a group of 256 / NP consecutive rows per step (coalesced rows),
    // running max in a register, one shared atomic per thread at the end
    __shared__ int sm[288];
    for (int i = threadIdx.x; i < NP; i += 256) sm[i] = 0;
    __syncthreads();
    const int rpb = max(1, 256 / NP);  // rows per step
    const int c = threadIdx.x % NP, rl = threadIdx.x / NP;
    uint32_t m = 0;
    if (rl < rpb && c < cols)
        for (long k = (long)blockIdx.x * rpb + rl; k < K; k += (long)gridDim.x * rpb)
            m = max(m, (uint32_t)__double2hiint(W[k * ldw + c] * row_scale(row_ef, k)) & 0x7ff00000u);
    if (m) atomicMax(&sm[c], (int)m);
    __syncthreads();
    for (int i = threadIdx.x; i < NP; i += 256)
        if (sm[i]) atomicMax(&colmax[i], sm[i]);
}

// Digit planes dig[i][c][k] of the columns of W (K x NP, ldw) at the scales colmax[c] >> 20
// (written to b_ef): 64-row slabs of W transposed through shared memory.
__global__ void __launch_bounds__(256) oz_digits_cols_kernel(const double* __restrict__ W, long ldw,
                                                            int NP, int cols, long K,
                                                            uint8_t* __restrict__ dig, long ldb,
                                                            const int* __restrict__ colmax,
                                                            int* __restrict__ b_ef,
                                                            const int* __restrict__ row_ef,
                                                            int nfirst) {
    // one k-tile (32 rows of W) per CTA; the slab is column-major (33-double stride) so that
    // every thread's 4 consecutive k of one column are contiguous, and the row scales of W' are
    // read once per row (the digits keep the integer path's rounding: ties away from zero)
    extern __shared__ double slab[];  // NP x 33
    __shared__ double rs[32];
    constexpr int ld = 33;
    const long k0 = (long)blockIdx.x * 32;
    if (threadIdx.x < 32) {
        const long k = k0 + threadIdx.x;
        rs[threadIdx.x] = k < K ? row_scale(row_ef, k) : 0.0;
    }
    if (blockIdx.x == 0)
        for (int c = threadIdx.x; c < NP; c += 256) b_ef[c] = colmax[c] >> 20;
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * NP; e += 256) {
        const int kk = e / NP, c = e - kk * NP;
        const long k = k0 + kk;
        slab[c * ld + kk] = (k < K && c < cols) ? W[k * ldw + c] * rs[kk] : 0.0;
    }
    __syncthreads();
    // thread -> (column c, 4 consecutive k): 8 k-quads per column; a warp writes 4 columns'
    // 32-byte rows of each plane
    for (int e = threadIdx.x; e < NP * 8; e += 256) {
        const int c = e >> 3, kq = (e & 7) * 4;
        if (k0 + kq >= ldb) continue;
        const int ef = colmax[c] >> 20;
        uint64_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = digits_of(slab[c * ld + kq + j], ef);
        uint32_t pl[kDigits];
        planes4(w, pl);
#pragma unroll
        for (int i = 0; i < kDigits; ++i)
            *reinterpret_cast<uint32_t*>(dig + b_offset(i, c, k0 + kq, NP, ldb, nfirst)) = pl[i];
    }
}


// Streaming form of the same conversion, with the row exponents given (oz_scan): one CTA per
// 128-row x 128-column block of A (256 threads; thread -> 16-column chunk t & 7 of row
// 32 it + t / 8, it = 0..3), so that every warp store lands on contiguous bytes of both tiled
// layouts (4 rows x 128 B of a SW32 ax tile, 4 rows x 128 B of an atx block) instead of 32
// scattered 16-byte pieces (a row-per-CTA conversion measured 3.2 TB/s of combined traffic). Rows
// >= `rows` and columns >= `cols` are zero digits; row block rb = blockIdx.y + r0 / 128.
// dig_ax may be null (only the atx blocks: the pipeline's stored-digit atx passes).
__global__ void __launch_bounds__(256) oz_convert_tiles_kernel(
    const double* __restrict__ A, long r0, long rows, long cols, long lda,
    uint8_t* __restrict__ dig_ax, uint8_t* __restrict__ dig_atx, const int* __restrict__ row_ef) {
    const int t = threadIdx.x, chunk = t & 7, rq = t >> 3;
    const long KT = (cols + 31) / 32, JB = (cols + 127) / 128;
    const long jb = blockIdx.x, rb = (r0 >> 7) + blockIdx.y;
    const long c0 = jb * 128 + chunk * 16;
    const long kt = c0 >> 5;
    const uint32_t half = (uint32_t)(chunk & 1);
#pragma unroll 1
    for (int it = 0; it < 4; ++it) {
        const uint32_t rl = (uint32_t)(it * 32 + rq);
        const long r = rb * 128 + rl;
        double v[16];
        if (r < rows && c0 + 16 <= cols) {
            const double* row = A + r * lda + c0;
#pragma unroll
            for (int e = 0; e < 16; e += 2) {
                const double2 x = __ldcs(reinterpret_cast<const double2*>(row + e));
                v[e] = x.x;
                v[e + 1] = x.y;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e)
                v[e] = (r < rows && c0 + e < cols) ? A[r * lda + c0 + e] : 0.0;
        }
        double f1, f2;
        fixed_scale(r < rows ? row_ef[r] : 0, f1, f2);
        uint32_t pw[kDigits][4];
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
            uint64_t wd[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) wd[e] = digits_scaled(v[4 * qd + e], f1, f2);
            uint32_t pl[kDigits];
            planes4(wd, pl);
#pragma unroll
            for (int i = 0; i < kDigits; ++i) pw[i][qd] = pl[i] ^ 0x80808080u;
        }
        const uint32_t kl = rl & 31;
        uint8_t* ax = dig_ax + ((rb * KT + kt) * kDigits) * 4096 + sw32(rl, half);
        uint8_t* at = dig_atx + ((((r >> 5) * JB) + jb) * kDigits) * 4096 + kl * 128 +
                      (((uint32_t)chunk ^ (kl & 7)) << 4);
#pragma unroll
        for (int i = 0; i < kDigits; ++i) {
            const uint4 q = make_uint4(pw[i][0], pw[i][1], pw[i][2], pw[i][3]);
            if (dig_ax && kt < KT) __stcs(reinterpret_cast<uint4*>(ax + i * 4096), q);
            __stcs(reinterpret_cast<uint4*>(at + i * 4096), q);
        }
    }
}

// Row exponents, NaN/Inf check and the stored digits (atx blocks, optionally ax tiles) in one
// pass over A (the optimistic
// pipeline's stored-digit atx passes need no column maxima): persistent CTAs (3 per SM) take
// 4-row groups; pass 1 (two warps per row) reduces each row's maximum exponent, pass 2
// re-reads the group — 128 KB per CTA, 57 MB in flight, so from L2 — and writes every warp's
// 4 rows x 128 columns as 512 contiguous bytes of each plane of an atx block. Rows [r0, r1)
// (r0 % 128 == 0; the last group of the matrix also zero-fills the pad rows up to 128).
// Measured at C2: 2.62 ms, DRAM read 6.83 GB of 6.64 (8-row groups at 2 CTAs / SM: 2.93 ms,
// 7.45 GB; the separate scan + tile conversion: 1.09 + 1.94 ms).
#ifndef OZ_SC_ROWS
#define OZ_SC_ROWS 4
#endif
constexpr int kScRows = OZ_SC_ROWS;            // rows per group: 8 (2 CTAs / SM) or 4 (3 / SM)
#ifndef OZ_SC_CTAS
#define OZ_SC_CTAS (kScRows == 8 ? 2 : 3)
#endif
constexpr int kScCtas = OZ_SC_CTAS;  // resident CTAs per SM (the L2 working set)
__global__ void __launch_bounds__(256, kScCtas) oz_scan_convert_kernel(
    const double* __restrict__ A, long r0, long r1, long rows, long cols, long lda,
    uint8_t* __restrict__ dig_ax, uint8_t* __restrict__ dig_atx, int* __restrict__ row_ef,
    int* __restrict__ flag) {
    __shared__ int ef_sh[kScRows];
    __shared__ uint32_t mx_sh[8];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    constexpr int kWpr = 8 / kScRows;  // warps per row in pass 1
    const long JB = (cols + 127) / 128, KT = (cols + 31) / 32;
    bool bad = false;
    for (long g0 = r0 + (long)blockIdx.x * kScRows; g0 < r1; g0 += (long)gridDim.x * kScRows) {
        {  // pass 1: warps w, w + kScRows, ... -> row g0 + w % kScRows, interleaved columns
            const int rw = w % kScRows, part = w / kScRows;
            const long r = g0 + rw;
            uint32_t m = 0;
            if (r < rows) {
                const double* row = A + r * lda;
                long c = 2L * lane + 64L * part;
#pragma unroll 4
                for (; c + 1 < cols; c += 64 * kWpr) {
                    const double2 x = *reinterpret_cast<const double2*>(row + c);
                    m = max(m, max((uint32_t)__double2hiint(x.x) & 0x7ff00000u,
                                   (uint32_t)__double2hiint(x.y) & 0x7ff00000u));
                }
                if (c < cols) m = max(m, (uint32_t)__double2hiint(row[c]) & 0x7ff00000u);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) mx_sh[w] = m;
        }
        __syncthreads();
        if (t < kScRows) {
            uint32_t m = 0;
            for (int pw = 0; pw < kWpr; ++pw) m = max(m, mx_sh[t + pw * kScRows]);
            const int ef = (int)(m >> 20);
            const long r = g0 + t;
            bad |= ef == 0x7ff;
            ef_sh[t] = r < rows ? ef : 0;
            if (r < rows) row_ef[r] = ef;
        }
        __syncthreads();
        // pass 2: warp w -> 4 rows of the group (lane / 8) and 128-column blocks
        constexpr int kQuads = kScRows / 4, kJStep = 8 / kQuads;
        const int chunk = lane & 7, rq = 4 * (w % kQuads) + (lane >> 3);
        const long r = g0 + rq;
        double f1, f2;
        fixed_scale(ef_sh[rq], f1, f2);
        const uint32_t kl = (uint32_t)(r & 31);
        for (long jb = w / kQuads; jb < JB; jb += kJStep) {
            const long c0 = jb * 128 + chunk * 16;
            double v[16];
            if (r < rows && c0 + 16 <= cols) {
                const double* row = A + r * lda + c0;
#pragma unroll
                for (int e = 0; e < 16; e += 2) {
                    const double2 x = __ldcs(reinterpret_cast<const double2*>(row + e));
                    v[e] = x.x;
                    v[e + 1] = x.y;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    v[e] = (r < rows && c0 + e < cols) ? A[r * lda + c0 + e] : 0.0;
            }
            uint32_t pw[kDigits][4];
#pragma unroll
            for (int qd = 0; qd < 4; ++qd) {
                uint64_t wd[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) wd[e] = digits_scaled(v[4 * qd + e], f1, f2);
                uint32_t pl[kDigits];
                planes4(wd, pl);
#pragma unroll
                for (int i = 0; i < kDigits; ++i) pw[i][qd] = pl[i] ^ 0x80808080u;
            }
            uint8_t* at = dig_atx + ((((r >> 5) * JB) + jb) * kDigits) * 4096 + kl * 128 +
                          (((uint32_t)chunk ^ (kl & 7)) << 4);
#pragma unroll
            for (int i = 0; i < kDigits; ++i)
                __stcs(reinterpret_cast<uint4*>(at + i * 4096),
                       make_uint4(pw[i][0], pw[i][1], pw[i][2], pw[i][3]));
            const long kt = c0 >> 5;
            if (dig_ax && kt < KT) {  // the ax tile (4 rows x 32 B of each plane per k-tile)
                uint8_t* ax = dig_ax + (((r >> 7) * KT + kt) * kDigits) * 4096 +
                              sw32((uint32_t)(r & 127), (uint32_t)(chunk & 1));
#pragma unroll
                for (int i = 0; i < kDigits; ++i)
                    __stcs(reinterpret_cast<uint4*>(ax + i * 4096),
                           make_uint4(pw[i][0], pw[i][1], pw[i][2], pw[i][3]));
            }
        }
        __syncthreads();  // ef_sh is rewritten by the next group
    }
    if (flag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
}

// ------------------------------------------------------------ GEMM from stored digits
// Both pass shapes from A's row-scaled digit planes (oz_scan_convert / oz_convert_tiles) and the
// small operand's
// digit planes:
//   MN = false (ax):  Y (M x NP) = A X. A operand = 128 rows x 32 k of each plane (K-major,
//                     SW32 TMA boxes); out = T 2^(a_ef[row] + b_ef[c] - 2104).
//   MN = true  (atx): Z = A^T W'. A operand = A^T: 128 columns x 32 rows of each plane, read
//                     in place as an MN-major operand (SW128 TMA boxes of 32 rows x 128 B);
//                     W' = diag(2^(E_row - 53)) W carries A's row scales (exact powers of two),
//                     so out = T 2^(b_ef[c] - 1028).
// Pure TMA + tcgen05 pipeline: warp 0 TMA producer (7 A tiles + 7 B planes per stage), warp 1
// TMEM owner + MMA issuer (whole warp, elected lane), warps 2-5 epilogue.
constexpr int kDsStages = 5;
constexpr int kDsThreads = 192;
constexpr uint32_t kDsADig = BM * BK;                       // 4 KB per A digit tile
constexpr uint32_t kDsBPlane = 64 * BK;                     // N <= 64
constexpr uint32_t kDsStage = kDigits * kDsADig + kDigits * kDsBPlane;  // 43008 B

__device__ __forceinline__ uint64_t sdesc_mn128(uint32_t saddr) {
    // MN-major SWIZZLE_128B: 128 B of M per row (one atom wide), 8-row (K) atoms 1024 B apart
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) |
           ((uint64_t)(1024u >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

template <bool MN, bool OUT_T>
__global__ void __launch_bounds__(kDsThreads, 1)
    gemm_ozd_kernel(const uint8_t* __restrict__ adig, long a_inner, const uint8_t* __restrict__ bdig,
                    const int* __restrict__ a_ef, const int* __restrict__ b_ef, int M, int NP,
                    int nch, int nfirst, double* __restrict__ out, long ldo,
                    long split_stride, int k_tiles, int k_tiles_per_split,
                    const int* __restrict__ abort_flag) {
    if (abort_flag && *(const volatile int*)abort_flag) return;
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = align_smem_1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kDsStages * kDsStage);
    uint64_t* empty = full + kDsStages;
    uint64_t* accum = empty + kDsStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // the nch column-chunk CTAs of an M tile form a cluster (rank = chunk): each loads
    // planes i = rank, rank + nch, ... of A's digits and multicasts them to all, so A's digits
    // cross L2 -> SM once per tile; a stage is refilled once every CTA's MMAs are done with it
    const int ch = blockIdx.x % nch;
    const int tile = blockIdx.x / nch;
    const int m0 = tile * BM;
    const int c0 = ch * nfirst;
    const int N = min(nfirst, NP - c0);
    const uint32_t pb = (uint32_t)N * BK;
    const int kt0 = blockIdx.y * k_tiles_per_split;
    const int kt1 = min(k_tiles, kt0 + k_tiles_per_split);
    const int n_iter = max(0, kt1 - kt0);
    const uint16_t cmask = (uint16_t)((1u << nch) - 1u);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kDsStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nch);
        }
        mbar_init(accum, 1);
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    if (nch > 1)
        cluster_sync_all();  // every CTA's barriers exist before a multicast targets them
    else
        __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // A: the (M tile, k-tile) block of 7 pre-swizzled 4 KB digit tiles, contiguous
            // (ax: block tile * a_inner + kt; atx: block kt * a_inner + tile); rank ch copies
            // its 1 / nch of it and multicasts. B: the chunk's 7 planes of the k-tile, contiguous.
            constexpr uint32_t kABlock = kDigits * kDsADig;
            const uint32_t part = ((kABlock / nch) + 15) & ~15u;  // 16-byte multiples
            // A's blocks come from HBM: prefetch them into L2 kPf stages ahead of the copies
            constexpr int kPf = 8;
            auto ablk = [&](long kt) {
                return adig + (MN ? kt * a_inner + tile : (long)tile * a_inner + kt) * kABlock;
            };
            const uint32_t off = (uint32_t)ch * part;
            const uint32_t len = ch == nch - 1 ? kABlock - off : part;
            for (int it = 0; it < min(kPf, n_iter); ++it) bulk_prefetch_l2(ablk(kt0 + it) + off, len);
            for (int it = 0; it < n_iter; ++it) {
                const int s = it % kDsStages;
                if (it >= kDsStages) mbar_wait(&empty[s], ((it / kDsStages) - 1) & 1);
                char* st = smem + s * kDsStage;
                const long kt = kt0 + it;
                if (it + kPf < n_iter) bulk_prefetch_l2(ablk(kt + kPf) + off, len);
                mbar_arrive_expect_tx(&full[s], kABlock + kDigits * pb);
                const uint8_t* src = ablk(kt);
                if (nch > 1)
                    bulk_load_mc(st + off, src + off, len, &full[s], cmask);
                else
                    bulk_load(st, src, kABlock, &full[s]);
                bulk_load(st + kABlock, bdig + kt * kDigits * NP * BK + (long)kDigits * BK * c0,
                          kDigits * pb, &full[s]);
            }
        }
    } else if (warp == 1) {
        constexpr int kNM = 9;
        constexpr int mi[kNM] = {6, 6, 5, 5, 4, 3, 2, 1, 0};
        constexpr int mp0[kNM] = {0, 4, 1, 4, 2, 3, 4, 5, 6};
        constexpr int mnp[kNM] = {4, 3, 3, 3, 5, 4, 3, 2, 1};
        constexpr int mdc[kNM] = {0, 4, 0, 3, 0, 0, 0, 0, 0};
        uint32_t idv[kNM];
#pragma unroll
        for (int j = 0; j < kNM; ++j) idv[j] = idesc(mnp[j] * N) | (MN ? (1u << 15) : 0u);
        const uint32_t sm0 = smem_u32(smem);
        for (int it = 0; it < n_iter; ++it) {
            const int s = it % kDsStages;
            const uint32_t st = sm0 + s * kDsStage;
            const uint64_t bd = sdesc(st + kDigits * kDsADig);
            mbar_wait(&full[s], (it / kDsStages) & 1);
            fence_after();
            if (elect_one()) {
#ifndef OZD_AX_CP
                if constexpr (!MN) {
                    // K-major A digits straight from shared memory (SW32): 1.81 ms per C2 pass,
                    // against 2.26 ms copying the 7 tiles into TMEM first (tcgen05.cp bound)
#pragma unroll
                    for (int j = 0; j < kNM; ++j)
                        mma_i8(tmem + (uint32_t)(mdc[j] * N), sdesc(st + (uint32_t)mi[j] * kDsADig),
                               bd + (((uint64_t)mp0[j] * pb) >> 4), idv[j],
                               (it > 0 || j > 1) ? 1u : 0u);
                } else
#endif
                if constexpr (!MN) {
                    // (OZD_AX_CP) K-major A digits: copy the 7 tiles into a TMEM buffer (3 after
                    // the accumulators, in-order with the MMAs) and run the MMAs with A from TMEM
                    const uint32_t tb = tmem + (uint32_t)(kGroups * N) + (uint32_t)(it % 3) * 56u;
#pragma unroll
                    for (int i = 0; i < kDigits; ++i)
                        tmem_cp_128x256b(tb + 8u * i, sdesc(st + (uint32_t)i * kDsADig));
#pragma unroll
                    for (int j = 0; j < kNM; ++j)
                        mma_i8_ts(tmem + (uint32_t)(mdc[j] * N), tb + 8u * mi[j],
                                  bd + (((uint64_t)mp0[j] * pb) >> 4), idv[j],
                                  (it > 0 || j > 1) ? 1u : 0u);
                } else {
#pragma unroll
                    for (int j = 0; j < kNM; ++j) {
                        const uint32_t a = st + (uint32_t)mi[j] * kDsADig;
                        mma_i8(tmem + (uint32_t)(mdc[j] * N), sdesc_mn128(a),
                               bd + (((uint64_t)mp0[j] * pb) >> 4), idv[j],
                               (it > 0 || j > 1) ? 1u : 0u);
                    }
                }
                if (nch > 1)
                    commit_mc(&empty[s], cmask);
                else
                    commit(&empty[s]);
            }
            __syncwarp();
        }
        if (n_iter > 0 && elect_one()) commit(accum);
        __syncwarp();
    } else {
        // ------------------------------------------------------------ epilogue (warps 2-5)
        const int q = warp & 3;
        const int grow = m0 + 32 * q + lane;
        const int efa = MN ? 1076 : (grow < M ? a_ef[grow] : 0);
        if (n_iter > 0) {
            mbar_wait_sleep(accum, 0);
            fence_after();
        }
        const uint32_t tlane = tmem + ((uint32_t)(32 * q) << 16);
        double* ob = out + (size_t)blockIdx.y * split_stride;
        for (int cc = 0; cc < N; cc += 16) {
            double y[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) y[i] = 0.0;
            if (n_iter > 0) {
#pragma unroll
                for (int g = kGroups - 1; g >= 0; --g) {
                    int vv[16];
                    tmem_ld16(tlane + (uint32_t)(g * N + cc), vv);
#pragma unroll
                    for (int i = 0; i < 16; ++i) y[i] = fma(y[i], 256.0, (double)vv[i]);
                }
            }
            if (grow < M) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int c = c0 + cc + i;
                    const double val = y[i] == 0.0 ? 0.0 : ldexp(y[i], efa + b_ef[c] - 2104);
                    if constexpr (OUT_T)
                        ob[(size_t)c * ldo + grow] = val;
                    else
                        ob[(size_t)grow * ldo + c] = val;
                }
            }
        }
    }
    fence_before();
    if (nch > 1)
        cluster_sync_all();  // no multicast commit or TMA is still in flight into a peer
    else
        __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// INT8 tensor-core issue-rate probe: every CTA issues back-to-back M = 128, N = 256, K = 32
// kind::i8 MMAs from zeroed shared memory (one commit per 8), the roofline denominator of the
// emulated FP64 passes (MEASURED_PEAKS.json has no INT8 entry).
__global__ void __launch_bounds__(128, 1) imma_peak_kernel(int iters, int* sink) {
    extern __shared__ __align__(1024) char smem_raw[];
    char* sm = align_smem_1024(smem_raw);
    __shared__ uint64_t bar[4];
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < 12 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        fence_barrier_init();
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tslot)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x < 32) {
        const uint64_t a = sdesc(smem_u32(sm)), b = sdesc(smem_u32(sm + 4096));
        const uint32_t id = idesc(256);
        // commits waited two rounds later, so the tensor pipe never drains
        for (int it = 0; it < iters; ++it) {
            if (elect_one()) {
#pragma unroll
                for (int j = 0; j < 8; ++j) mma_i8(tmem, a, b, id, 1u);
                commit(&bar[it & 3]);
            }
            __syncwarp();
            if (it >= 2) mbar_wait(&bar[(it - 2) & 3], ((it - 2) >> 2) & 1);
        }
        for (int it = iters - 2; it < iters; ++it) mbar_wait(&bar[it & 3], (it >> 2) & 1);
    }
    fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
    }
    if (threadIdx.x == 0 && iters < 0) *sink = 1;
}

}  // namespace oz

cudaError_t measure_imma_peak(cudaStream_t st, double* tops) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, smem = 16 * 1024;
    cudaError_t e = cudaFuncSetAttribute(oz::imma_peak_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    oz::imma_peak_kernel<<<148, 128, smem, st>>>(iters, nullptr);  // warm-up (clocks up)
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0, st);
        oz::imma_peak_kernel<<<148, 128, smem, st>>>(iters, nullptr);
        cudaEventRecord(e1, st);
        e = cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *tops = 2.0 * 128 * 256 * 32 * 8.0 * iters * 148 / (best * 1e-3) / 1e12;
    return e;
}

// ======================================================================== host side
namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn oz_encode() {
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

int oz_map(CUtensorMap* map, CUtensorMapDataType dt, int esize, const void* base, long rows,
           long cols, long ld_elems, int box_cols, int box_rows, CUtensorMapSwizzle swz) {
    auto encode = oz_encode();
    if (!encode) return -1;
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld_elems * esize) & 15)) return -2;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld_elems * esize)};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -3;
}

unsigned oz_grid(long work, long per = 256) {
    long b = (work + per - 1) / per;
    if (b > 148L * 16) b = 148L * 16;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

// Column chunks: NP <= 64 one chunk, else chunks of round_up(NP / nch, 16) (the last smaller).
void oz_chunks(int NP, int* nch, int* nfirst) {
    const int n = (NP + oz::kMaxN - 1) / oz::kMaxN;
    const int f = ((NP + n - 1) / n + 15) & ~15;
    *nch = (NP + f - 1) / f;
    *nfirst = f;
}

long oz_ldb(long K) { return (K + 31) & ~31L; }
size_t oz_digits_bytes(int NP, long K) { return (size_t)oz::kDigits * NP * oz_ldb(K); }

cudaError_t launch_gemm_oz(const GemmOz& p, cudaStream_t st) {
    if (p.NP < 16 || p.NP > 256 || (p.NP % 16) != 0) return cudaErrorInvalidValue;
    int nch, nfirst;
    oz_chunks(p.NP, &nch, &nfirst);
    if (nch > oz::kMaxChunks) return cudaErrorInvalidValue;
    CUtensorMap mA;
    if (!p.mn) {
        if (oz_map(&mA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, p.A, p.M, p.K, p.lda, 16, oz::BM,
                   CU_TENSOR_MAP_SWIZZLE_128B))
            return cudaErrorInvalidValue;
    } else {
        if (oz_map(&mA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, p.A, p.K, p.M, p.lda, 16, oz::BK,
                   CU_TENSOR_MAP_SWIZZLE_128B))
            return cudaErrorInvalidValue;
    }
    oz::BMaps bm;
    for (int c = 0; c < nch; ++c) {
        const int n = std::min(nfirst, p.NP - c * nfirst);
        if (oz_map(&bm.m[c], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, p.bdig, (long)oz::kDigits * p.NP,
                   p.ldb, p.ldb, oz::BK, n, CU_TENSOR_MAP_SWIZZLE_32B))
            return cudaErrorInvalidValue;
    }
    for (int c = nch; c < oz::kMaxChunks; ++c) bm.m[c] = bm.m[0];
    const int k_tiles = (int)((p.K + oz::BK - 1) / oz::BK);
    int splits = p.splits < 1 ? 1 : p.splits;
    int per = (k_tiles + splits - 1) / splits;
    if (per > kOzMaxKTiles) return cudaErrorInvalidValue;  // int32 accumulator headroom
    const size_t smem = oz::kRing + 24 * 8 + 16 + 1024;
    // RSVD_B200_OZ_DIAG (profiling only; results are wrong): 1 = MMA skips the B-ready wait,
    // 2 = converters skip the A-ready wait, 4 = converters skip the digit arithmetic
    static const int diag = getenv("RSVD_B200_OZ_DIAG") ? atoi(getenv("RSVD_B200_OZ_DIAG")) : 0;
    // RSVD_B200_OZ_MC=1: the column-chunk CTAs of a tile share the FP64 tile by cluster
    // multicast (measured 2x slower than independent loads served by L2: 5.1 vs 2.6 ms at C2)
    static const int mc = getenv("RSVD_B200_OZ_MC") ? atoi(getenv("RSVD_B200_OZ_MC")) : 0;
    const unsigned gx = (unsigned)(((p.M + oz::BM - 1) / oz::BM) * nch);
    dim3 grid(gx, (unsigned)splits);
#define OZ_LAUNCH(MN, OT)                                                                        \
    do {                                                                                         \
        auto kern = oz::gemm_oz_kernel<MN, OT>;                                                  \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             (int)smem);                                         \
        if (e != cudaSuccess) return e;                                                          \
        cudaLaunchConfig_t cfg = {};                                                             \
        cfg.gridDim = grid;                                                                      \
        cfg.blockDim = dim3(oz::kThreads);                                                       \
        cfg.dynamicSmemBytes = smem;                                                             \
        cfg.stream = st;                                                                         \
        cudaLaunchAttribute attr[1];                                                             \
        attr[0].id = cudaLaunchAttributeClusterDimension;                                        \
        attr[0].val.clusterDim.x = mc ? (unsigned)nch : 1u;                                      \
        attr[0].val.clusterDim.y = 1;                                                            \
        attr[0].val.clusterDim.z = 1;                                                            \
        cfg.attrs = attr;                                                                        \
        cfg.numAttrs = 1;                                                                        \
        e = cudaLaunchKernelEx(&cfg, kern, mA, bm, p.a_ef, p.b_ef, (int)p.M, p.NP, nch, nfirst,  \
                               p.out, p.ldo, p.split_stride, k_tiles, per, p.abort, diag, mc);   \
        if (e != cudaSuccess) return e;                                                          \
    } while (0)
    if (!p.mn) {
        if (p.out_t) return cudaErrorInvalidValue;
        OZ_LAUNCH(false, false);
    } else if (p.out_t) {
        OZ_LAUNCH(true, true);
    } else {
        OZ_LAUNCH(true, false);
    }
#undef OZ_LAUNCH
    return cudaGetLastError();
}

// planes x rows x cols bytes (row stride ld, plane stride plane_bytes)
int oz_map3(CUtensorMap* map, const void* base, long planes, long plane_bytes, long rows,
            long cols, long ld, int box_cols, int box_rows, CUtensorMapSwizzle swz) {
    auto encode = oz_encode();
    if (!encode) return -1;
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld & 15) || (plane_bytes & 15)) return -2;
    cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)ld, (cuuint64_t)plane_bytes};
    cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -3;
}

cudaError_t launch_gemm_ozd(const GemmOzd& p, cudaStream_t st) {
    if (p.NP < 16 || p.NP > 256 || (p.NP % 16) != 0) return cudaErrorInvalidValue;
    int nch, nfirst;
    oz_chunks(p.NP, &nch, &nfirst);
    if (nch > oz::kMaxChunks) return cudaErrorInvalidValue;
    const int k_tiles = (int)((p.K + oz::BK - 1) / oz::BK);
    const int splits = p.splits < 1 ? 1 : p.splits;
    const int per = (k_tiles + splits - 1) / splits;
    if (per > kOzMaxKTiles) return cudaErrorInvalidValue;
    const size_t smem = oz::kDsStages * oz::kDsStage + 16 * 8 + 16 + 1024;
    const unsigned gx = (unsigned)(((p.M + oz::BM - 1) / oz::BM) * nch);
    dim3 grid(gx, (unsigned)splits);
#define OZD_LAUNCH(MN, OT)                                                                       \
    do {                                                                                         \
        auto kern = oz::gemm_ozd_kernel<MN, OT>;                                                 \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             (int)smem);                                         \
        if (e != cudaSuccess) return e;                                                          \
        cudaLaunchConfig_t cfg = {};                                                             \
        cfg.gridDim = grid;                                                                      \
        cfg.blockDim = dim3(oz::kDsThreads);                                                     \
        cfg.dynamicSmemBytes = smem;                                                             \
        cfg.stream = st;                                                                         \
        cudaLaunchAttribute attr[1];                                                             \
        attr[0].id = cudaLaunchAttributeClusterDimension;                                        \
        attr[0].val.clusterDim.x = (unsigned)nch;                                                \
        attr[0].val.clusterDim.y = 1;                                                            \
        attr[0].val.clusterDim.z = 1;                                                            \
        cfg.attrs = attr;                                                                        \
        cfg.numAttrs = 1;                                                                        \
        e = cudaLaunchKernelEx(&cfg, kern, p.adig, p.a_inner, p.bdig, p.a_ef, p.b_ef, (int)p.M,  \
                               p.NP, nch, nfirst, p.out, p.ldo, p.split_stride, k_tiles, per,    \
                               p.abort);                                                         \
        if (e != cudaSuccess) return e;                                                          \
    } while (0)
    if (!p.mn) {
        if (p.out_t) return cudaErrorInvalidValue;
        OZD_LAUNCH(false, false);
    } else if (p.out_t) {
        OZD_LAUNCH(true, true);
    } else {
        OZD_LAUNCH(true, false);
    }
#undef OZD_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_oz_scan(const double* A, long rows, long cols, long lda, int* row_ef,
                           int* col_ef, int* part, int* flag, cudaStream_t st, bool col_acc) {
    if ((reinterpret_cast<uintptr_t>(A) & 15) || (lda & 1)) return cudaErrorInvalidValue;
    const long cb = (cols + 511) / 512, rb = (rows + oz::kScanRows - 1) / oz::kScanRows;
    int* row_part = part;
    int* col_part = part + cb * rows;
    oz::oz_scan_kernel<<<dim3((unsigned)cb, (unsigned)rb), 256, 0, st>>>(A, rows, cols, lda,
                                                                         row_part, col_part, flag);
    oz::oz_reduce_max_kernel<<<oz_grid(rows), 256, 0, st>>>(row_part, (int)cb, rows, row_ef, 0);
    oz::oz_reduce_max_kernel<<<oz_grid(cols), 256, 0, st>>>(col_part, (int)rb, cols, col_ef,
                                                            col_acc ? 1 : 0);
    return cudaGetLastError();
}

size_t oz_scan_part_ints(long rows, long cols) {
    const long cb = (cols + 511) / 512, rb = (rows + oz::kScanRows - 1) / oz::kScanRows;
    return (size_t)(cb * rows + rb * cols);
}

size_t oz_ax_bytes(long rows, long cols) {
    return (size_t)((rows + 127) / 128) * ((cols + 31) / 32) * oz::kDigits * oz::kDsADig;
}

size_t oz_atx_bytes(long rows, long cols) {  // rows padded to whole 128-row blocks (convert)
    return (size_t)((rows + 127) / 128 * 4) * ((cols + 127) / 128) * oz::kDigits * oz::kDsADig;
}

size_t oz_tiled_bytes(long rows, long cols) {
    const size_t blk = (size_t)oz::kDigits * oz::kDsADig;
    const size_t ax = (size_t)((rows + 127) / 128) * ((cols + 31) / 32) * blk;
    const size_t at = (size_t)((rows + 31) / 32) * ((cols + 127) / 128) * blk;
    return std::max(ax, at);
}


cudaError_t launch_oz_convert_tiles(const double* A, long r0, long r1, long rows, long cols,
                                    long lda, uint8_t* dig_ax, uint8_t* dig_atx,
                                    const int* row_ef, cudaStream_t st) {
    if ((reinterpret_cast<uintptr_t>(A) & 15) || (lda & 1) || (r0 & 127)) return cudaErrorInvalidValue;
    if (r1 >= rows) r1 = (rows + 127) / 128 * 128;  // the last chunk also zeroes the pad rows
    else if (r1 & 127) return cudaErrorInvalidValue;
    if (r1 <= r0) return cudaSuccess;
    const dim3 grid((unsigned)((cols + 127) / 128), (unsigned)((r1 - r0) / 128));
    oz::oz_convert_tiles_kernel<<<grid, 256, 0, st>>>(A, r0, rows, cols, lda, dig_ax, dig_atx,
                                                      row_ef);
    return cudaGetLastError();
}

cudaError_t launch_oz_scan_convert(const double* A, long r0, long r1, long rows, long cols,
                                   long lda, uint8_t* dig_ax, uint8_t* dig_atx, int* row_ef,
                                   int* flag, cudaStream_t st) {
    if ((reinterpret_cast<uintptr_t>(A) & 15) || (lda & 1) || (r0 & 127)) return cudaErrorInvalidValue;
    if (r1 >= rows) r1 = (rows + 127) / 128 * 128;  // the last chunk also zeroes the pad rows
    else if (r1 & 127) return cudaErrorInvalidValue;
    if (r1 <= r0) return cudaSuccess;
    const long groups = (r1 - r0) / oz::kScRows;
    const unsigned grid = (unsigned)std::min<long>(groups, (long)oz::kScCtas * 148);
    oz::oz_scan_convert_kernel<<<grid, 256, 0, st>>>(A, r0, r1, rows, cols, lda, dig_ax,
                                                     dig_atx, row_ef, flag);
    return cudaGetLastError();
}

cudaError_t launch_oz_digits_rows(const double* Xt, long ldx, int NP, int cols, long K,
                                  uint8_t* dig, int* b_ef, cudaStream_t st, int nfirst) {
    oz::oz_digits_rows_kernel<<<NP, 256, 0, st>>>(Xt, ldx, NP, cols, K, dig, oz_ldb(K), b_ef,
                                                  nfirst);
    return cudaGetLastError();
}

cudaError_t launch_oz_digits_cols(const double* W, long ldw, int NP, int cols, long K,
                                  uint8_t* dig, int* b_ef, int* colmax, cudaStream_t st,
                                  const int* row_ef, int nfirst) {
    cudaError_t e = cudaMemsetAsync(colmax, 0, NP * sizeof(int), st);
    if (e != cudaSuccess) return e;
    oz::oz_colmax_kernel<<<(unsigned)std::min<long>(148L * 8, (K + 3) / 4), 256, 0, st>>>(
        W, ldw, NP, cols, K, colmax, row_ef);
    const size_t smem = (size_t)NP * 33 * sizeof(double);
    e = cudaFuncSetAttribute(oz::oz_digits_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return e;
    const long ldb = oz_ldb(K);
    oz::oz_digits_cols_kernel<<<(unsigned)((ldb + 31) / 32), 256, smem, st>>>(
        W, ldw, NP, cols, K, dig, ldb, colmax, b_ef, row_ef, nfirst);
    return cudaGetLastError();
}

}  // namespace rsvdb200
