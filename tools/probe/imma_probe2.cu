// tcgen05 kind::i8 issue/throughput probe, one template instance per pattern (so that the
// issue loop's code is exactly the pattern's): 148 CTAs, warp 0 runs the loop, an elected
// lane issues; one commit every `every` rounds, waited `lag` commits later.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46) | (6ull << 61);
}
__device__ __forceinline__ uint32_t idesc(int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t par) {
    uint32_t done;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(su32(bar)), "r"(par) : "memory");
    } while (!done);
}
__device__ __forceinline__ bool elect() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
    return pred;
}

template <int P>
__global__ void probe(int N, int iters, int every, long long* out) {
    extern __shared__ __align__(1024) char sm[];
    __shared__ uint64_t bars[8];
    __shared__ uint32_t tslot;
    char* base = (char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (threadIdx.x < 32) {
        const uint32_t A = su32(base), B = su32(base + 32 * 1024);
        const uint32_t pb = N * 32;
        const uint64_t bd = sdesc(B);
        constexpr int mi[9] = {6, 6, 5, 5, 4, 3, 2, 1, 0};
        constexpr int mp0[9] = {0, 4, 1, 4, 2, 3, 4, 5, 6};
        constexpr int mnp[9] = {4, 3, 3, 3, 5, 4, 3, 2, 1};
        constexpr int mdc[9] = {0, 4, 0, 3, 0, 0, 0, 0, 0};
        uint32_t idv[9];
        for (int j = 0; j < 9; ++j) idv[j] = idesc(mnp[j] * N);
        const uint32_t idn = idesc(N), id3 = idesc(3 * N), id256 = idesc(256);
        int nc = 0;
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t ad = tmem + 400 + (it & 1) * 56;
            if (elect()) {
                if constexpr (P == 0) {  // the Ozaki pattern, 9 MMAs
#pragma unroll
                    for (int j = 0; j < 9; ++j)
                        mma_ts(tmem + mdc[j] * N, ad + mi[j] * 8, bd + ((mp0[j] * pb) >> 4), idv[j], 1);
                } else if constexpr (P == 1) {  // 28 single-plane products
#pragma unroll
                    for (int i = 0; i < 7; ++i)
#pragma unroll
                        for (int j = 6 - i; j < 7; ++j)
                            mma_ts(tmem + (i + j - 6) * N, ad + i * 8, bd + ((j * pb) >> 4), idn, 1);
                } else if constexpr (P == 2) {  // 9 uniform 3-plane MMAs
#pragma unroll
                    for (int j = 0; j < 9; ++j)
                        mma_ts(tmem + (j % 3) * N, ad + (j % 7) * 8, bd, id3, 1);
                } else if constexpr (P == 5) {  // the Ozaki pattern, A from smem (SW32)
#pragma unroll
                    for (int j = 0; j < 9; ++j)
                        mma_ss(tmem + mdc[j] * N, sdesc(A + (it & 1) * 28672 / 2 + mi[j] * 4096), bd + ((mp0[j] * pb) >> 4), idv[j], 1);
                } else if constexpr (P == 3) {  // 8 x N=256 SS (peak reference)
#pragma unroll
                    for (int j = 0; j < 8; ++j) mma_ss(tmem, sdesc(A), bd, id256, 1);
                } else if constexpr (P == 4) {  // 8 x N=256 TS
#pragma unroll
                    for (int j = 0; j < 8; ++j) mma_ts(tmem, ad, bd, id256, 1);
                }
                if ((it + 1) % every == 0) commit(&bars[nc % 4]);
            }
            __syncwarp();
            if ((it + 1) % every == 0) {
                if (nc >= 2) wait(&bars[(nc - 2) % 4], ((nc - 2) / 4) & 1);
                ++nc;
            }
        }
        for (int c = nc - 2 > 0 ? nc - 2 : 0; c < nc; ++c) wait(&bars[c % 4], (c / 4) & 1);
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

template <int P>
void run(const char* name, int N, int every, double ops_per_round, long long* d) {
    cudaFuncSetAttribute(probe<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 4096;
    probe<P><<<148, 128, 100 * 1024>>>(N, iters, every, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0; for (int i = 0; i < 148; ++i) cyc += h[i]; cyc /= 148;
    printf("%-50s every %2d: %8.1f cycles/round  %6.0f ops/clk/SM (%.0f%% of 16384)\n", name, every, cyc / iters,
           ops_per_round * iters / cyc, 100.0 * ops_per_round * iters / cyc / 16384);
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    for (int every : {1}) {
        run<5>("oz pattern (9 SS MMAs, N=48)", 48, every, 2.0 * 128 * 28 * 48 * 32, d);
        run<5>("oz pattern (9 SS MMAs, N=32)", 32, every, 2.0 * 128 * 28 * 32 * 32, d);
        run<0>("oz pattern (9 TS MMAs, N=48)", 48, every, 2.0 * 128 * 28 * 48 * 32, d);
        run<0>("oz pattern (9 TS MMAs, N=32)", 32, every, 2.0 * 128 * 28 * 32 * 32, d);
        run<1>("28 single-plane TS MMAs N=48", 48, every, 2.0 * 128 * 28 * 48 * 32, d);
        run<2>("9 uniform TS MMAs N=144", 48, every, 2.0 * 128 * 27 * 48 * 32, d);
        run<3>("8 x N=256 SS", 48, every, 2.0 * 128 * 256 * 32 * 8, d);
        run<4>("8 x N=256 TS", 48, every, 2.0 * 128 * 256 * 32 * 8, d);
    }
    return 0;
}
