// FP32-input GEMMs of the rSVD on the 5th-generation tensor cores (tcgen05, sm_100a):
// 3xTF32 split products accumulated in TMEM, operands staged by TMA.
//
// The FP32 path (BASELINE config C4: A stored in FP32) runs every product with an
// m-dimension on tcgen05.mma.kind::tf32. The tensor core reads an FP32 operand as TF32
// (the low 13 mantissa bits are ignored), so x = hi + lo with hi = x itself and
// lo = x - trunc_tf32(x) (exact in FP32); the product is accumulated as
// a_hi b_hi + a_hi b_lo + a_lo b_hi (a_lo b_lo is below FP32 rounding). Per product the
// error is ~3 * 2^-20 relative; the tensor core's FP32 accumulation adds ~1e-5 of
// sum |a||b| on long positive sums (tests/test_gpu_tf32.py) — FP32-class accuracy at a third
// of the TF32 tensor rate.
//
// Two operand shapes, the same two the FP64 path has (gemm_f64.cu):
//   ax  (K-major A and B): D[M x NP] = A (M x K row-major) * B, B given as Bt (NP x K
//       row-major). Y = A*Omega, Y = A*Z, Q = Y*R^-1, U = Q*U_B.
//   atx (MN-major A and B): D[M x NP] = A^T W, A (K x M row-major) read in place,
//       W (K x NP row-major). (A^T Q)^T, Q^T A, the tall Gram Y^T Y. Split-K over K.
// The B operand's lo part comes precomputed from global memory (Blo, same layout: the
// FP32 epilogue below writes it next to every tall FP32 output, cvt_f64_f32 for the
// small operands); only A's lo part is formed in shared memory.
//
// CTA = 6 warps: warp 0 issues TMA, warp 1 owns the TMEM allocation and issues the MMAs
// (M = 128, N = NP in chunks of at most 256), warps 2-5 split A (and scan it for NaN/Inf when
// asked), then drain the accumulator (tcgen05.ld 32x32b) in the epilogue. Four pipeline
// stages of K = 16. Default (TS): the converter warps write A and A_lo into a TMEM buffer per
// stage and all three products read A from TMEM, so shared memory carries only the TMA writes
// and the B reads (profiles/r2_ncu_tf32_ts.md). The shared-memory form (RSVD_B200_TF32_SS)
// writes A_lo next to A in the stage and runs a b, a b_lo as soon as TMA lands and a_lo b
// once the converters signal. mbarriers: full (TMA tx), conv (4 converter warps), empty
// (tcgen05.commit), accum.
//
// UMMA shared-memory descriptors (version 1):
//   K-major : SWIZZLE_64B (layout 4): rows of 64 B (16 fp32 along K), 8-row atoms of
//             512 B (SBO = 512, LBO unused); the two 8-wide K steps start 0 / 32 B in.
//   MN-major: 32-bit MN-major operands only exist as SWIZZLE_128B_BASE32B (layout 1, TMA
//             CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): rows of 128 B (32 fp32 along M/N)
//             indexed by K, 4-row atoms (SBO = 512), 32-wide M/N chunks one TMA box apart
//             (LBO = 2048); the two K steps start 0 / 1024 B in.
#include "common.cuh"
#include "kernels.h"

namespace rsvdb200 {
namespace tf32 {

constexpr int BM = 128;
constexpr int BK = 16;
constexpr int kStages = 4;
constexpr int kStagesTs = 4;  // TS (a fifth stage fits without the A_lo region: measured equal)
constexpr int kThreads = 192;
constexpr uint32_t kABytes = BM * BK * 4;  // 8 KB per A tile (raw or lo)
constexpr uint32_t kBoxMN = 32 * BK * 4;   // 2 KB: one MN-major box (32 M/N x 16 K)

__device__ __forceinline__ float lo_part(float x) {
    return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                          uint64_t layout) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (layout << 61);
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, M = 128, N, operand majors.
__device__ __forceinline__ uint32_t idesc(int N, bool mn) {
    const uint32_t maj = mn ? 1u : 0u;
    return (1u << 4) | (2u << 7) | (2u << 10) | (maj << 15) | (maj << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}

// A operand from TMEM (128 lanes x 8 tf32 columns at a_tmem)
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id,
                                       uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
        "r"(v[15])
        : "memory");
}

__device__ __forceinline__ bool elect_one_tf32() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// the commit's arrive lands on the barrier at the same offset in every CTA of `mask`
__device__ __forceinline__ void commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// TMA load broadcast into the same smem offset of every CTA in `mask` (complete_tx on the
// barrier at the same offset in each)
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar,
                                               int c_inner, int c_outer, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c_inner), "r"(c_outer),
        "h"(mask)
        : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}

__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
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
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Bytes of one B tile (raw or lo): K-major NP rows of 64 B; MN-major ceil(NP/32) boxes.
__host__ __device__ __forceinline__ uint32_t b_bytes(int NP, bool mn) {
    return mn ? (uint32_t)((NP + 31) / 32) * kBoxMN : (uint32_t)NP * (BK * 4);
}
__host__ __device__ __forceinline__ uint32_t stage_bytes(int NP, bool mn, bool ts = false) {
    return (ts ? 1 : 2) * kABytes + 2 * b_bytes(NP, mn);
}
// TS: TMEM columns of the accumulator (32-aligned) and of the per-stage A hi / lo buffers
__host__ __device__ __forceinline__ uint32_t ts_abase(int NP) { return (uint32_t)((NP + 31) & ~31); }
constexpr uint32_t kTsCols = 2 * BK;  // hi (16 columns) + lo (16 columns) per stage

// Drain the 128 x NP FP32 accumulator (warps 2-5: each its TMEM lane quarter) and store it
// (FP32 + lo parts, FP64, or transposed), slab blockIdx.y of a split-K launch.
// c_off > 0 (upper-triangle Gram): the accumulator holds output columns c_off.. at TMEM
// column 0; columns below c_off are written as zeros.
template <bool OUT64, bool OUT_T>
__device__ __forceinline__ void epilogue(uint32_t tmem, int warp, int lane, int m0, int M, int NP,
                                         bool have, void* __restrict__ out,
                                         float* __restrict__ out_lo, long ldo, long split_stride,
                                         int c_off) {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = m0 + 32 * q + lane;
    const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16);
    char* ob = reinterpret_cast<char*>(out) + (size_t)blockIdx.y * split_stride * (OUT64 ? 8 : 4);
    for (int c0 = 0; c0 < NP; c0 += 16) {
        float v[16];
        if (have && c0 >= c_off) {
            tmem_ld16(trow + (c0 - c_off), v);
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        if (row < M) {
            if constexpr (OUT_T) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const size_t o = (size_t)(c0 + i) * ldo + row;
                    if constexpr (OUT64)
                        reinterpret_cast<double*>(ob)[o] = (double)v[i];
                    else
                        reinterpret_cast<float*>(ob)[o] = v[i];
                }
            } else if constexpr (OUT64) {
                double2* d = reinterpret_cast<double2*>(reinterpret_cast<double*>(ob) +
                                                        (size_t)row * ldo + c0);
#pragma unroll
                for (int i = 0; i < 8; ++i) d[i] = make_double2(v[2 * i], v[2 * i + 1]);
            } else {
                float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(ob) +
                                                      (size_t)row * ldo + c0);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    d[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                if (out_lo) {  // lo parts for the next product that reads this as B
                    float4* dl = reinterpret_cast<float4*>(out_lo + (size_t)row * ldo + c0);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        dl[i] = make_float4(lo_part(v[4 * i]), lo_part(v[4 * i + 1]),
                                            lo_part(v[4 * i + 2]), lo_part(v[4 * i + 3]));
                }
            }
        }
    }
}

// PAIR: the CTA is one of a 2-CTA cluster (adjacent M tiles, same K range) that shares the
// B operand: each CTA loads half of B and B_lo and multicasts it into both, so B's L2
// traffic (re-read by every M tile) halves. A stage may then only be refilled once both
// CTAs' MMAs are done with it: every MMA commit arrives on the empty barrier of both.
// TS: the A operand goes to TMEM instead of shared memory. The converter warps (thread = tile
// row = TMEM lane) read the stage's A tile, write it (the hi part: the tensor core ignores the
// low mantissa bits) and its lo part into a 32-column TMEM buffer per stage with tcgen05.st,
// and all three products read A from there: shared memory then carries only the TMA writes
// and the MMAs' B reads (per 16-wide K stage at NP = 272: ~101 KB instead of ~157 KB: the
// A tile, read by 3 products x 2 N chunks, and the A_lo writes leave the shared-memory pipe,
// which bounds the SS form). The MN-major A tile is one unswizzled 128 x 16 box (conflict-free
// row reads); the MMA warp runs the loop converged and one elected lane issues.
template <bool MN, bool OUT64, bool OUT_T, bool PAIR, bool TS>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tf32_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB,
                     const __grid_constant__ CUtensorMap mapBlo, void* __restrict__ out,
                     float* __restrict__ out_lo, long ldo, long split_stride, int M, int NP,
                     int k_tiles, int k_tiles_per_split, int* __restrict__ flag, int upper,
                     const int* __restrict__ abort_flag) {
    // an aborted optimistic pipeline skips its remaining passes (both CTAs of a pair read
    // the same flag, set before this launch in stream order, so they return together)
    if (abort_flag && *(const volatile int*)abort_flag) return;
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = align_smem_1024(smem_raw);
    constexpr int NS = TS ? kStagesTs : kStages;
    const uint32_t bB = b_bytes(NP, MN);
    const uint32_t kStage = (TS ? 1 : 2) * kABytes + 2 * bB;
    constexpr uint32_t kAOff = TS ? kABytes : 2 * kABytes;  // B raw offset in a stage
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * kStage);
    uint64_t* conv = full + NS;
    uint64_t* empty = conv + NS;
    uint64_t* accum = empty + NS;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BM;
    const int kt0 = blockIdx.y * k_tiles_per_split;
    const int kt1 = min(k_tiles, kt0 + k_tiles_per_split);
    const int n_iter = max(0, kt1 - kt0);
    const uint32_t tneed = TS ? ts_abase(NP) + NS * kTsCols : (uint32_t)NP;
    const uint32_t tmem_cols =
        tneed <= 32 ? 32 : tneed <= 64 ? 64 : tneed <= 128 ? 128 : tneed <= 256 ? 256 : 512;
    // upper (a symmetric Gram, MN shape): rows m0.. only need columns m0.. (multiple of 128)
    const int c_off = (MN && upper) ? min(m0, (NP - 16) & ~31) : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], 4);
            mbar_init(&empty[s], PAIR ? 2 : 1);
        }
        mbar_init(accum, 1);
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    if constexpr (PAIR)
        cluster_sync();  // the peer's multicasts may target our barriers from here on
    else
        __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t crank = PAIR ? cluster_rank() : 0;

    // stage layout: A raw | A lo | B raw | B lo
    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&mapA);
            tma_prefetch_desc(&mapB);
            tma_prefetch_desc(&mapBlo);
            for (int it = 0; it < n_iter; ++it) {
                const int s = it % NS;
                if (it >= NS) mbar_wait(&empty[s], ((it / NS) - 1) & 1);
                char* st = smem + s * kStage;
                char* sb = st + kAOff;
                const int k = (kt0 + it) * BK;
                mbar_arrive_expect_tx(&full[s], kABytes + 2 * bB);
                if constexpr (!MN) {
                    tma_load_2d(st, &mapA, &full[s], k, m0);
                    if constexpr (PAIR) {  // rows [crank NP/2, (crank + 1) NP/2) of B, to both
                        const int rows = NP / 2, r0 = (int)crank * rows;
                        tma_load_2d_mc(sb + r0 * (BK * 4), &mapB, &full[s], k, r0, 3);
                        tma_load_2d_mc(sb + bB + r0 * (BK * 4), &mapBlo, &full[s], k, r0, 3);
                    } else {
                        const int parts = NP > 256 ? 2 : 1;
                        const int rows = NP / parts;
                        for (int p = 0; p < parts; ++p) {
                            tma_load_2d(sb + p * rows * (BK * 4), &mapB, &full[s], k, p * rows);
                            tma_load_2d(sb + bB + p * rows * (BK * 4), &mapBlo, &full[s], k,
                                        p * rows);
                        }
                    }
                } else {
                    const int nb = (NP + 31) / 32;
                    if constexpr (TS) {
                        tma_load_2d(st, &mapA, &full[s], m0, k);  // one 128 x 16 box
                    } else {
#pragma unroll
                        for (int i = 0; i < BM / 32; ++i)
                            tma_load_2d(st + i * kBoxMN, &mapA, &full[s], m0 + 32 * i, k);
                    }
                    if constexpr (PAIR) {  // every other 32-wide box of B, to both
                        for (int j = (int)crank; j < nb; j += 2) {
                            tma_load_2d_mc(sb + j * kBoxMN, &mapB, &full[s], 32 * j, k, 3);
                            tma_load_2d_mc(sb + bB + j * kBoxMN, &mapBlo, &full[s], 32 * j, k, 3);
                        }
                    } else {
                        for (int j = 0; j < nb; ++j) {
                            tma_load_2d(sb + j * kBoxMN, &mapB, &full[s], 32 * j, k);
                            tma_load_2d(sb + bB + j * kBoxMN, &mapBlo, &full[s], 32 * j, k);
                        }
                    }
                }
            }
        }
    } else if (warp == 1 && TS) {
        // ------------------------------------------------------- MMA issuer (TS)
        const uint32_t lbo = MN ? kBoxMN : 16u, sbo = 512u;
        const uint64_t lay = MN ? 1u : 4u;
        const int ne = NP - c_off;
        const int n1 = ne > 256 ? ((ne / 2 + 31) & ~31) : ne, n2 = ne - n1;
        const uint32_t id1 = idesc(n1, MN) & ~(1u << 15), id2 = n2 > 0 ? idesc(n2, MN) & ~(1u << 15) : 0u;
        const uint32_t co = (uint32_t)n1 * (MN ? kBoxMN / 32u : BK * 4u);
        const uint32_t bo = (uint32_t)(c_off / 32) * kBoxMN;
        const uint32_t abuf = tmem + ts_abase(NP);
        for (int it = 0; it < n_iter; ++it) {
            const int s = it % NS;
            const uint32_t b_raw = smem_u32(smem + s * kStage) + kAOff + bo, b_lo = b_raw + bB;
            const uint32_t a_hi = abuf + (uint32_t)s * kTsCols, a_lo = a_hi + BK;
            mbar_wait(&full[s], (it / NS) & 1);
            mbar_wait(&conv[s], (it / NS) & 1);
            fence_after();
            if (elect_one_tf32()) {
#pragma unroll
                for (int pr = 0; pr < 3; ++pr) {  // a_hi b_hi, a_hi b_lo, a_lo b_hi
                    const uint32_t a = pr == 2 ? a_lo : a_hi, b = pr == 1 ? b_lo : b_raw;
#pragma unroll
                    for (int ks = 0; ks < BK / 8; ++ks) {
                        const uint32_t ko = MN ? ks * 1024u : ks * 32u;
                        const uint32_t acc = (it > 0 || pr > 0 || ks > 0) ? 1u : 0u;
                        mma_ts(tmem, a + 8u * ks, sdesc(b + ko, lbo, sbo, lay), id1, acc);
                        if (n2 > 0)
                            mma_ts(tmem + (uint32_t)n1, a + 8u * ks,
                                   sdesc(b + co + ko, lbo, sbo, lay), id2, acc);
                    }
                }
                if constexpr (PAIR)
                    commit_mc(&empty[s], 3);
                else
                    commit(&empty[s]);
            }
            __syncwarp();
        }
        if (n_iter > 0 && elect_one_tf32()) commit(accum);
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------------------- MMA issuer
        if (lane == 0) {
            const uint32_t lbo = MN ? kBoxMN : 16u, sbo = 512u;
            const uint64_t lay = MN ? 1u : 4u;
            // N > 256 is two MMAs of balanced width (272 = 160 + 112): a narrow second chunk
            // (256 + 16) costs nearly as much as a wide one (measured: NP 272 took 1.45x NP 256)
            const int ne = NP - c_off;  // columns this CTA computes (c_off: 32-column boxes)
            const int n1 = ne > 256 ? ((ne / 2 + 31) & ~31) : ne, n2 = ne - n1;
            const uint32_t id1 = idesc(n1, MN), id2 = n2 > 0 ? idesc(n2, MN) : 0u;
            const uint32_t co = (uint32_t)n1 * (MN ? kBoxMN / 32u : BK * 4u);  // B offset of chunk 2
            const uint32_t bo = (uint32_t)(c_off / 32) * kBoxMN;  // B offset of column c_off
            auto issue = [&](uint32_t a, uint32_t b, uint32_t acc0) {
#pragma unroll
                for (int ks = 0; ks < BK / 8; ++ks) {
                    const uint32_t ko = MN ? ks * 1024u : ks * 32u;
                    const uint64_t ad = sdesc(a + ko, lbo, sbo, lay);
                    const uint32_t acc = (ks == 0) ? acc0 : 1u;
                    mma(tmem, ad, sdesc(b + ko, lbo, sbo, lay), id1, acc);
                    if (n2 > 0)
                        mma(tmem + (uint32_t)n1, ad, sdesc(b + co + ko, lbo, sbo, lay), id2, acc);
                }
            };
            for (int it = 0; it < n_iter; ++it) {
                const int s = it % NS;
                const uint32_t st = smem_u32(smem + s * kStage);
                const uint32_t a_raw = st, a_lo = st + kABytes;
                const uint32_t b_raw = st + 2 * kABytes + bo, b_lo = b_raw + bB;
                mbar_wait(&full[s], (it / NS) & 1);
                fence_after();
                issue(a_raw, b_raw, it > 0 ? 1u : 0u);  // a_hi b_hi
                issue(a_raw, b_lo, 1u);                 // a_hi b_lo
                mbar_wait(&conv[s], (it / NS) & 1);
                fence_after();
                issue(a_lo, b_raw, 1u);                 // a_lo b_hi
                if constexpr (PAIR)
                    commit_mc(&empty[s], 3);
                else
                    commit(&empty[s]);
            }
            if (n_iter > 0) commit(accum);
        }
    } else if (TS) {
        // ------------------------- A hi / lo into TMEM (warps 2-5: thread = row = lane)
        const int q = warp & 3;
        const int r = 32 * q + lane;
        const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16) + ts_abase(NP);
        bool bad = false;
        for (int it = 0; it < n_iter; ++it) {
            const int s = it % NS;
            mbar_wait(&full[s], (it / NS) & 1);
            const char* st = smem + s * kStage;
            uint32_t hi[16], lo[16];
            if constexpr (!MN) {  // K-major, SWIZZLE_64B: 16-byte chunk c of row r at c ^ (r/2 % 4)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float4 v = *reinterpret_cast<const float4*>(
                        st + r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
                    hi[4 * c] = __float_as_uint(v.x);
                    hi[4 * c + 1] = __float_as_uint(v.y);
                    hi[4 * c + 2] = __float_as_uint(v.z);
                    hi[4 * c + 3] = __float_as_uint(v.w);
                }
            } else {  // MN-major, unswizzled 128 (M) x 16 (K): row k of 512 bytes
#pragma unroll
                for (int kk = 0; kk < 16; ++kk)
                    hi[kk] = *reinterpret_cast<const uint32_t*>(st + kk * 512 + r * 4);
            }
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
                if (flag) bad |= (hi[kk] & 0x7f800000u) == 0x7f800000u;
                lo[kk] = __float_as_uint(lo_part(__uint_as_float(hi[kk])));
            }
            tmem_st16(tl + (uint32_t)s * kTsCols, hi);
            tmem_st16(tl + (uint32_t)s * kTsCols + BK, lo);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&conv[s]);
        }
        if (flag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
        if (n_iter > 0) {
            mbar_wait(accum, 0);
            fence_after();
        }
        epilogue<OUT64, OUT_T>(tmem, warp, lane, m0, M, NP, n_iter > 0, out, out_lo, ldo,
                               split_stride, c_off);
    } else {
        // ------------------------------------------------- A lo split (warps 2-5)
        const int ct = threadIdx.x - 64;
        bool bad = false;
        for (int it = 0; it < n_iter; ++it) {
            const int s = it % NS;
            mbar_wait(&full[s], (it / NS) & 1);
            char* st = smem + s * kStage;
            const float4* ar = reinterpret_cast<const float4*>(st);
            float4* al = reinterpret_cast<float4*>(st + kABytes);
#pragma unroll
            for (int i = ct; i < (int)(kABytes / 16); i += 128) {
                const float4 v = ar[i];
                if (flag) {
                    const uint32_t e = 0x7f800000u;
                    bad |= ((__float_as_uint(v.x) & e) == e) | ((__float_as_uint(v.y) & e) == e) |
                           ((__float_as_uint(v.z) & e) == e) | ((__float_as_uint(v.w) & e) == e);
                }
                al[i] = make_float4(lo_part(v.x), lo_part(v.y), lo_part(v.z), lo_part(v.w));
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&conv[s]);
        }
        if (flag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);

        // ------------------------------------------------------------ epilogue
        if (n_iter > 0) {
            mbar_wait(accum, 0);
            fence_after();
        }
        epilogue<OUT64, OUT_T>(tmem, warp, lane, m0, M, NP, n_iter > 0, out, out_lo, ldo,
                               split_stride, c_off);
    }
    fence_before();
    // PAIR: the peer's last commits arrive on our empty barriers; they precede its accum
    // commit, which its epilogue waited for before this barrier
    if constexpr (PAIR)
        cluster_sync();
    else
        __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(tmem_cols));
    }
}

}  // namespace tf32


// ----------------------------------------------------------------------------------------
// 2-SM variant of the K-major (ax) shape: a CTA pair runs tcgen05.mma.cta_group::2 with
// M = 256 (each CTA's 128 rows of A in its own shared memory, its own 128 x NP accumulator in
// its own TMEM) and each CTA holds only its half of every N chunk of B and B_lo. The tensor
// cores of the pair share the B halves, so per CTA a stage is 8 KB A + 8 KB A_lo + NP x 64 B of
// B/B_lo halves (33 KB at NP = 272, against 50 KB single-CTA): the kernel is bound by shared-
// memory traffic (TMA writes + UMMA operand reads), which drops by a third, and six stages fit.
//   full[s]  (leader)  B halves of both CTAs landed (each CTA's TMA signals the leader's barrier)
//   afull[s] (each)    this CTA's A tile landed (for its converter warps)
//   conv[s]  (leader)  A_lo of both CTAs written (8 converter-warp arrivals, 4 remote)
//   empty[s] (each)    the leader's MMAs of stage s are done (commit multicast to both)
//   accum    (each)    the last MMA is done (commit multicast)
namespace tf32 {

constexpr int kStages2 = 6;

__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr)
                 : "memory");
}

// TMA load into this CTA's smem, completion signalled on an mbarrier that may live in the
// peer CTA of the pair (cluster address)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar,
                                                 int c_inner, int c_outer) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c_inner), "r"(c_outer)
        : "memory");
}

__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void commit2_mc(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

// M = 256 kind::tf32 descriptor (K-major operands)
__device__ __forceinline__ uint32_t idesc2(int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

__host__ __device__ __forceinline__ uint32_t stage_bytes2(int NP) {
    return 2 * kABytes + 2 * (uint32_t)(NP / 2) * (BK * 4);
}

template <bool OUT64, bool OUT_T>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tf32_2sm_kernel(const __grid_constant__ CUtensorMap mapA,
                         const __grid_constant__ CUtensorMap mapB1,
                         const __grid_constant__ CUtensorMap mapBlo1,
                         const __grid_constant__ CUtensorMap mapB2,
                         const __grid_constant__ CUtensorMap mapBlo2, void* __restrict__ out,
                         float* __restrict__ out_lo, long ldo, long split_stride, int M, int NP,
                         int k_tiles, int k_tiles_per_split, int* __restrict__ flag) {
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = align_smem_1024(smem_raw);
    const int n1 = NP > 256 ? 256 : NP, n2 = NP - n1;  // N chunks; each CTA holds half of each
    const uint32_t h1 = (uint32_t)(n1 / 2) * (BK * 4), h2 = (uint32_t)(n2 / 2) * (BK * 4);
    const uint32_t bH = h1 + h2;  // this CTA's B (or B_lo) half
    const uint32_t kStage = 2 * kABytes + 2 * bH;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages2 * kStage);
    uint64_t* afull = full + kStages2;
    uint64_t* conv = afull + kStages2;
    uint64_t* empty = conv + kStages2;
    uint64_t* accum = empty + kStages2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = cluster_rank();
    const bool leader = crank == 0;
    const int m0 = blockIdx.x * BM;
    const int kt0 = blockIdx.y * k_tiles_per_split;
    const int kt1 = min(k_tiles, kt0 + k_tiles_per_split);
    const int n_iter = max(0, kt1 - kt0);
    const uint32_t tmem_cols = NP <= 32 ? 32 : NP <= 64 ? 64 : NP <= 128 ? 128 : NP <= 256 ? 256 : 512;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages2; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&afull[s], 1);
            mbar_init(&conv[s], 8);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accum, 1);
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
    fence_after();
    const uint32_t tmem = *tmem_slot;

    // stage layout: A raw | A lo | B half (chunk-1 half, chunk-2 half) | B_lo half
    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&mapA);
            tma_prefetch_desc(&mapB1);
            tma_prefetch_desc(&mapBlo1);
            if (n2 > 0) {
                tma_prefetch_desc(&mapB2);
                tma_prefetch_desc(&mapBlo2);
            }
            for (int it = 0; it < n_iter; ++it) {
                const int s = it % kStages2;
                if (it >= kStages2) mbar_wait(&empty[s], ((it / kStages2) - 1) & 1);
                char* st = smem + s * kStage;
                char* sb = st + 2 * kABytes;
                const int k = (kt0 + it) * BK;
                const uint32_t fb = mapa_u32(smem_u32(&full[s]), 0);  // the leader's full[s]
                if (leader) mbar_arrive_expect_tx(&full[s], 4 * bH);  // both CTAs' B + B_lo halves
                mbar_arrive_expect_tx(&afull[s], kABytes);
                tma_load_2d(st, &mapA, &afull[s], k, m0);
                tma_load_2d_pair(sb, &mapB1, fb, k, (int)crank * (n1 / 2));
                tma_load_2d_pair(sb + bH, &mapBlo1, fb, k, (int)crank * (n1 / 2));
                if (n2 > 0) {
                    tma_load_2d_pair(sb + h1, &mapB2, fb, k, n1 + (int)crank * (n2 / 2));
                    tma_load_2d_pair(sb + bH + h1, &mapBlo2, fb, k, n1 + (int)crank * (n2 / 2));
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------- MMA issuer (leader CTA only)
        if (leader && lane == 0) {
            const uint32_t lbo = 16u, sbo = 512u;
            const uint64_t lay = 4u;
            const uint32_t id1 = idesc2(n1), id2 = n2 > 0 ? idesc2(n2) : 0u;
            auto issue = [&](uint32_t a, uint32_t b, uint32_t acc0) {
#pragma unroll
                for (int ks = 0; ks < BK / 8; ++ks) {
                    const uint32_t ko = ks * 32u;
                    const uint64_t ad = sdesc(a + ko, lbo, sbo, lay);
                    const uint32_t acc = (ks == 0) ? acc0 : 1u;
                    mma2(tmem, ad, sdesc(b + ko, lbo, sbo, lay), id1, acc);
                    if (n2 > 0) mma2(tmem + 256, ad, sdesc(b + h1 + ko, lbo, sbo, lay), id2, acc);
                }
            };
            for (int it = 0; it < n_iter; ++it) {
                const int s = it % kStages2;
                const uint32_t st = smem_u32(smem + s * kStage);
                const uint32_t a_raw = st, a_lo = st + kABytes;
                const uint32_t b_raw = st + 2 * kABytes, b_lo = b_raw + bH;
                mbar_wait(&full[s], (it / kStages2) & 1);
                mbar_wait(&conv[s], (it / kStages2) & 1);  // also: both A tiles landed
                fence_after();
                issue(a_raw, b_raw, it > 0 ? 1u : 0u);  // a_hi b_hi
                issue(a_raw, b_lo, 1u);                 // a_hi b_lo
                issue(a_lo, b_raw, 1u);                 // a_lo b_hi
                commit2_mc(&empty[s]);
            }
            if (n_iter > 0) commit2_mc(accum);
        }
    } else {
        // ------------------------------------------------- A lo split (warps 2-5)
        const int ct = threadIdx.x - 64;
        bool bad = false;
        for (int it = 0; it < n_iter; ++it) {
            const int s = it % kStages2;
            mbar_wait(&afull[s], (it / kStages2) & 1);
            char* st = smem + s * kStage;
            const float4* ar = reinterpret_cast<const float4*>(st);
            float4* al = reinterpret_cast<float4*>(st + kABytes);
#pragma unroll
            for (int i = ct; i < (int)(kABytes / 16); i += 128) {
                const float4 v = ar[i];
                if (flag) {
                    const uint32_t e = 0x7f800000u;
                    bad |= ((__float_as_uint(v.x) & e) == e) | ((__float_as_uint(v.y) & e) == e) |
                           ((__float_as_uint(v.z) & e) == e) | ((__float_as_uint(v.w) & e) == e);
                }
                al[i] = make_float4(lo_part(v.x), lo_part(v.y), lo_part(v.z), lo_part(v.w));
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_u32(smem_u32(&conv[s]), 0));
        }
        if (flag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);

        // ------------------------------------------------------------ epilogue
        if (n_iter > 0) {
            mbar_wait(accum, 0);
            fence_after();
        }
        epilogue<OUT64, OUT_T>(tmem, warp, lane, m0, M, NP, n_iter > 0, out, out_lo, ldo,
                               split_stride, 0);
    }
    fence_before();
    cluster_sync();  // no multicast commit or remote arrive is still in flight into the peer
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(tmem_cols));
    }
}

}  // namespace tf32

// ================================================================ host side
namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
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

// Row-major FP32 (rows x cols, ld elements), box {box_cols, box_rows}.
int map_f32(CUtensorMap* map, const float* base, long rows, long cols, long ld, int box_cols,
            int box_rows, CUtensorMapSwizzle swz) {
    auto encode = encode_fn();
    if (!encode) return -1;
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * 4) & 15)) return -2;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -3;
}

template <bool MN, bool OUT64, bool OUT_T, bool PAIR, bool TS>
cudaError_t launch_t(const GemmTf32& p, const CUtensorMap& mA, const CUtensorMap& mB,
                     const CUtensorMap& mBlo, cudaStream_t st) {
    const int ns = TS ? tf32::kStagesTs : tf32::kStages;
    const size_t smem = ns * tf32::stage_bytes(p.NP, MN, TS) + (3 * ns + 1) * 8 + 16 + 1024;
    auto kern = tf32::gemm_tf32_kernel<MN, OUT64, OUT_T, PAIR, TS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int k_tiles = (int)((p.K + tf32::BK - 1) / tf32::BK);
    int splits = p.splits < 1 ? 1 : p.splits;
    int per = (k_tiles + splits - 1) / splits;
    if (p.k_per_split > 0) {  // an explicit split length (a row range of a larger split-K)
        per = p.k_per_split;
        splits = (k_tiles + per - 1) / per;
    }
    unsigned gx = (unsigned)((p.M + tf32::BM - 1) / tf32::BM);
    if (PAIR) gx = (gx + 1) & ~1u;  // the odd tile's partner only reads zeros past M
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gx, (unsigned)splits);
    cfg.blockDim = dim3(tf32::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PAIR ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, mA, mB, mBlo, p.out, static_cast<float*>(p.out_lo), p.ldo,
                           p.split_stride, (int)p.M, p.NP, k_tiles, per, p.flag, (int)p.upper,
                           p.abort);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <bool OUT64, bool OUT_T>
cudaError_t launch_2sm(const GemmTf32& p, const CUtensorMap& mA, const CUtensorMap* mB,
                       cudaStream_t st) {
    const size_t smem = tf32::kStages2 * tf32::stage_bytes2(p.NP) + (5 * tf32::kStages2 + 1) * 8 +
                        16 + 1024;
    auto kern = tf32::gemm_tf32_2sm_kernel<OUT64, OUT_T>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int k_tiles = (int)((p.K + tf32::BK - 1) / tf32::BK);
    const int splits = p.splits < 1 ? 1 : p.splits;
    const int per = (k_tiles + splits - 1) / splits;
    unsigned gx = (unsigned)((p.M + tf32::BM - 1) / tf32::BM);
    gx = (gx + 1) & ~1u;  // the odd tile's partner only reads zeros past M
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gx, (unsigned)splits);
    cfg.blockDim = dim3(tf32::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, mA, mB[0], mB[1], mB[2], mB[3], p.out,
                           static_cast<float*>(p.out_lo), p.ldo, p.split_stride, (int)p.M, p.NP,
                           k_tiles, per, p.flag);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// 2-CTA clusters sharing B: only for more than one M tile, and for an odd count only when
// the idle pad tile it needs is a small fraction (with few M tiles, e.g. the s x s Gram's 3,
// it would cost a whole extra wave of the split-K grid)
bool use_pair(const GemmTf32& p) {
    static const bool pair = !getenv("RSVD_B200_TF32_NO_PAIR");
    const long tiles = (p.M + tf32::BM - 1) / tf32::BM;
    return pair && tiles > 1 && (tiles % 2 == 0 || tiles >= 16);
}

// A operand in TMEM (TS) unless RSVD_B200_TF32_SS is set (the shared-memory form, kept for A/B)
bool use_ts() {
    static const bool ss = getenv("RSVD_B200_TF32_SS") != nullptr;
    return !ss;
}

template <bool MN, bool OUT64, bool OUT_T>
cudaError_t launch_p(const GemmTf32& p, const CUtensorMap& mA, const CUtensorMap& mB,
                     const CUtensorMap& mBlo, cudaStream_t st) {
    if (use_ts()) {
        if (use_pair(p)) return launch_t<MN, OUT64, OUT_T, true, true>(p, mA, mB, mBlo, st);
        return launch_t<MN, OUT64, OUT_T, false, true>(p, mA, mB, mBlo, st);
    }
    if (use_pair(p)) return launch_t<MN, OUT64, OUT_T, true, false>(p, mA, mB, mBlo, st);
    return launch_t<MN, OUT64, OUT_T, false, false>(p, mA, mB, mBlo, st);
}

}  // namespace

cudaError_t launch_gemm_tf32(const GemmTf32& p, cudaStream_t st) {
    if (p.NP < 16 || p.NP > 288 || (p.NP % 16) != 0 || !p.Blo) return cudaErrorInvalidValue;
    if (p.out_lo && (p.out64 || p.out_t || p.splits > 1)) return cudaErrorInvalidValue;
    CUtensorMap mA, mB, mBlo;
    // cta_group::2 variant: correct but measured slower (2.45 ms flat in NP at C4 size against
    // 1.7-2.5 ms for the 1-SM kernel), so opt-in only (RSVD_B200_TF32_2SM=1)
    static const bool two_sm = getenv("RSVD_B200_TF32_2SM") != nullptr;
    if (!p.mn && two_sm && p.M > tf32::BM) {
        // cta_group::2: A boxes of 128 rows; B / B_lo as the two CTAs' halves of each N chunk
        const int n1 = p.NP > 256 ? 256 : p.NP, n2 = p.NP - n1;
        const auto sw = CU_TENSOR_MAP_SWIZZLE_64B;
        CUtensorMap mb[4];
        if (map_f32(&mA, p.A, p.M, p.K, p.lda, tf32::BK, tf32::BM, sw) ||
            map_f32(&mb[0], p.B, p.NP, p.K, p.ldb, tf32::BK, n1 / 2, sw) ||
            map_f32(&mb[1], p.Blo, p.NP, p.K, p.ldb, tf32::BK, n1 / 2, sw))
            return cudaErrorInvalidValue;
        if (n2 > 0) {
            if (map_f32(&mb[2], p.B, p.NP, p.K, p.ldb, tf32::BK, n2 / 2, sw) ||
                map_f32(&mb[3], p.Blo, p.NP, p.K, p.ldb, tf32::BK, n2 / 2, sw))
                return cudaErrorInvalidValue;
        } else {
            mb[2] = mb[0];
            mb[3] = mb[1];
        }
        if (p.out64) return p.out_t ? launch_2sm<true, true>(p, mA, mb, st)
                                    : launch_2sm<true, false>(p, mA, mb, st);
        return p.out_t ? launch_2sm<false, true>(p, mA, mb, st)
                       : launch_2sm<false, false>(p, mA, mb, st);
    }
    if (!p.mn) {  // A: M x K (lda), Bt: NP x K (ldb); 64-byte rows of K
        // one box per B half: the paired kernel loads NP / 2 rows per CTA, the single one
        // NP (<= 256) or two halves
        const int brows = (p.NP > 256 || use_pair(p))
                              ? p.NP / 2
                              : p.NP;
        const auto sw = CU_TENSOR_MAP_SWIZZLE_64B;
        if (map_f32(&mA, p.A, p.M, p.K, p.lda, tf32::BK, tf32::BM, sw) ||
            map_f32(&mB, p.B, p.NP, p.K, p.ldb, tf32::BK, brows, sw) ||
            map_f32(&mBlo, p.Blo, p.NP, p.K, p.ldb, tf32::BK, brows, sw))
            return cudaErrorInvalidValue;
    } else {  // A: K x M (lda), W: K x NP (ldb); 128-byte rows of M / N
        const auto sw = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
        const bool ts = use_ts();  // TS: A is read by the converters only, one plain box
        if (map_f32(&mA, p.A, p.K, p.M, p.lda, ts ? tf32::BM : 32, tf32::BK,
                    ts ? CU_TENSOR_MAP_SWIZZLE_NONE : sw) ||
            map_f32(&mB, p.B, p.K, p.NP, p.ldb, 32, tf32::BK, sw) ||
            map_f32(&mBlo, p.Blo, p.K, p.NP, p.ldb, 32, tf32::BK, sw))
            return cudaErrorInvalidValue;
    }
    if (!p.mn) {
        if (p.out64) return p.out_t ? launch_p<false, true, true>(p, mA, mB, mBlo, st)
                                    : launch_p<false, true, false>(p, mA, mB, mBlo, st);
        return p.out_t ? launch_p<false, false, true>(p, mA, mB, mBlo, st)
                       : launch_p<false, false, false>(p, mA, mB, mBlo, st);
    }
    if (p.out64) return p.out_t ? launch_p<true, true, true>(p, mA, mB, mBlo, st)
                                : launch_p<true, true, false>(p, mA, mB, mBlo, st);
    return p.out_t ? launch_p<true, false, true>(p, mA, mB, mBlo, st)
                   : launch_p<true, false, false>(p, mA, mB, mBlo, st);
}

// ------------------------------------------------------------ conversions
// out = (float)in (0 outside rows_valid x cols_valid); lo (optional) = out - trunc_tf32(out).
__global__ void cvt_f64_f32_kernel(const double* __restrict__ in, long ldi, long rows, long cols,
                                   long rows_valid, long cols_valid, float* __restrict__ out,
                                   float* __restrict__ lo, long ldo) {
    const long total = rows * cols;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const long r = e / cols, c = e % cols;
        const float x = (r < rows_valid && c < cols_valid) ? (float)in[r * ldi + c] : 0.f;
        out[r * ldo + c] = x;
        if (lo) lo[r * ldo + c] = tf32::lo_part(x);
    }
}

__global__ void cvt_f32_f64_kernel(const float* __restrict__ in, long ldi, long rows, long cols,
                                   double* __restrict__ out, long ldo) {
    const long total = rows * cols;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const long r = e / cols, c = e % cols;
        out[r * ldo + c] = (double)in[r * ldi + c];
    }
}

__global__ void split_lo_kernel(const float* __restrict__ in, long rows, long cols, long ld,
                                float* __restrict__ lo) {
    const long total = rows * cols;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const long r = e / cols, c = e % cols;
        lo[r * ld + c] = tf32::lo_part(in[r * ld + c]);
    }
}

__global__ void transpose_f32_kernel(const float* __restrict__ in, long rows, long cols, long ldi,
                                     float* __restrict__ out, long ldo) {
    __shared__ float tile[32][33];
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

cudaError_t launch_transpose_f32(const float* in, long rows, long cols, long ldi, float* out,
                                 long ldo, cudaStream_t st) {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    transpose_f32_kernel<<<grid, dim3(32, 8), 0, st>>>(in, rows, cols, ldi, out, ldo);
    return cudaGetLastError();
}

static unsigned cvt_grid(long work) {
    long b = (work + 255) / 256;
    if (b > 148L * 32) b = 148L * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

cudaError_t launch_cvt_f64_f32(const double* in, long ldi, long rows, long cols, long rows_valid,
                               long cols_valid, float* out, long ldo, cudaStream_t st, float* lo) {
    cvt_f64_f32_kernel<<<cvt_grid(rows * cols), 256, 0, st>>>(in, ldi, rows, cols, rows_valid,
                                                              cols_valid, out, lo, ldo);
    return cudaGetLastError();
}

cudaError_t launch_cvt_f32_f64(const float* in, long ldi, long rows, long cols, double* out,
                               long ldo, cudaStream_t st) {
    cvt_f32_f64_kernel<<<cvt_grid(rows * cols), 256, 0, st>>>(in, ldi, rows, cols, out, ldo);
    return cudaGetLastError();
}

cudaError_t launch_split_lo(const float* in, long rows, long cols, long ld, float* lo,
                            cudaStream_t st) {
    split_lo_kernel<<<cvt_grid(rows * cols), 256, 0, st>>>(in, rows, cols, ld, lo);
    return cudaGetLastError();
}

}  // namespace rsvdb200
