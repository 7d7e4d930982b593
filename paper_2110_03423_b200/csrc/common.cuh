// Shared device helpers for the B200 (sm_100a) rSVD kernels: mbarrier / TMA PTX
// wrappers, the FP64 tensor-core MMA (DMMA) wrapper and the 128-byte swizzle
// address map that the TMA boxes are laid out in.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rsvdb200 {

constexpr int kWarp = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

// --------------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// 2-D tiled bulk tensor load global -> shared, completion signalled on `bar`
// (complete_tx::bytes). Coordinates are element indices {inner, outer}.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c_inner, int c_outer) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c_inner), "r"(c_outer)
        : "memory");
}

// 3-D tiled bulk tensor load (coordinates {c0 inner, c1, c2}); out-of-range elements of any
// dimension are zero-filled.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// ---------------------------------------------------------- FP64 tensor core
// mma.sync m16n8k16 f64 (lowered to 8x DMMA.8x8x4 on sm_100a). Fragment maps
// (g = lane>>2, t = lane&3; CuTe SM90_16x8x16_F64F64F64F64_TN traits):
//   a[v]: row g + 8*(v&1),  k-slot t + 4*(v>>1)
//   b[v]: col g,            k-slot t + 4*v
//   c[v]: row g + 8*(v>>1), col 2t + (v&1)
__device__ __forceinline__ void dmma_16x8x16(double (&c)[4], const double (&a)[8],
                                             const double (&b)[4]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
          "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// The dynamic shared-memory window rounded up to 1024 bytes (128B-swizzle atoms) by pointer
// arithmetic on the __shared__ array itself: a round trip through uintptr_t would make every
// derived access a generic LD.E/ST.E with 64-bit addresses instead of LDS/STS.
__device__ __forceinline__ char* align_smem_1024(char* smem_raw) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
    return smem_raw + ((1024u - (a & 1023u)) & 1023u);
}

// Byte offset of element (row, col) inside a TMA box written with
// CU_TENSOR_MAP_SWIZZLE_128B whose rows are exactly 128 bytes (16 doubles).
// The box base must be 1024-byte aligned.
__device__ __forceinline__ uint32_t swz128(uint32_t row, uint32_t col) {
    return row * 128u + ((((col >> 1) ^ (row & 7u)) & 7u) << 4) + ((col & 1u) << 3);
}

__device__ __forceinline__ double lds_f64(const char* smem_base, uint32_t byte_off) {
    return *reinterpret_cast<const double*>(smem_base + byte_off);
}

// shared::cta address -> the same offset in cluster CTA `rank` (shared::cluster address)
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace rsvdb200
