// Microbenchmark of tcgen05 kind::i8 MMA throughput for the Ozaki kernel's shapes
// (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 imma_probe.cu -o imma_probe).
// One CTA per SM issues `iters` rounds of an MMA pattern from one thread, committing each
// round to an mbarrier and waiting for it `lag` rounds later; prints cycles per round and
// achieved int8 ops/cycle/SM. Operands are zeros (the rate does not depend on values).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t sbo, uint64_t lay) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (lay << 61);
}
__device__ __forceinline__ uint32_t idesc(int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
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

// mode 0: the Ozaki pattern, A in smem (SW32); 1: same, A in TMEM; 2: one N=256 MMA per
// round (x nrep); 3: pattern with N = 32 chunks; swz: B/A layout 6 = SW32, 2 = SW128 (K offset)
__global__ void probe(int mode, int N, int iters, int lag, long long* out, int nrep) {
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
    if (mode >= 10 && threadIdx.x < 32) {
        // whole warp runs the loop (uniform control flow); one elected lane issues
        const uint32_t A = su32(base), B = su32(base + 32 * 1024);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            uint32_t pred;
            asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
            if (pred) {
                for (int r = 0; r < nrep; ++r) {
                    if (mode == 10)
                        mma_ss(tmem, sdesc(A, 256, 6), sdesc(B, 256, 6), idesc(N), 1);
                    else if (mode == 11)
                        mma_ts(tmem, tmem + 400 + 8 * (r & 3), sdesc(B, 256, 6), idesc(N), 1);
                    else if (mode == 12)  // 28 products of N each into 7 group accumulators
                        mma_ts(tmem + (r % 7) * N, tmem + 400 + 8 * (r % 7), sdesc(B + (r % 7) * N * 32, 256, 6), idesc(N), 1);
                    else if (mode == 13)  // alternating N: N, 2N, 3N
                        mma_ts(tmem, tmem + 400 + 8 * (r % 7), sdesc(B, 256, 6), idesc(N * (1 + r % 3)), 1);
                    else if (mode == 14)  // fixed 3N, accumulator offsets vary
                        mma_ts(tmem + (r % 3) * N, tmem + 400 + 8 * (r % 7), sdesc(B, 256, 6), idesc(3 * N), 1);
                }
                commit(&bars[it % 4]);
            }
            __syncwarp();
            if (it >= lag) wait(&bars[(it - lag) % 4], ((it - lag) / 4) & 1);
        }
        for (int it = iters - lag > 0 ? iters - lag : 0; it < iters; ++it) wait(&bars[it % 4], (it / 4) & 1);
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    } else if (mode < 10 && threadIdx.x == 0) {
        const uint32_t A = su32(base), B = su32(base + 32 * 1024);
        const uint32_t pb = N * 32;
        const int mi[9] = {6, 6, 5, 5, 4, 3, 2, 1, 0};
        const int mp0[9] = {0, 4, 1, 4, 2, 3, 4, 5, 6};
        const int mnp[9] = {4, 3, 3, 3, 5, 4, 3, 2, 1};
        const int mdc[9] = {0, 4, 0, 3, 0, 0, 0, 0, 0};
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (mode <= 1 || mode == 3) {
                for (int r = 0; r < nrep; ++r)
                for (int j = 0; j < 9; ++j) {
                    const uint64_t b = sdesc(B + mp0[j] * pb, 256, 6);
                    if (mode == 1)
                        mma_ts(tmem + mdc[j] * N, tmem + 400 + mi[j] * 8, b, idesc(mnp[j] * N), 1);
                    else
                        mma_ss(tmem + mdc[j] * N, sdesc(A + mi[j] * 4096, 256, 6), b, idesc(mnp[j] * N), 1);
                }
            } else if (mode == 2) {
                for (int r = 0; r < nrep; ++r)
                    mma_ss(tmem, sdesc(A, 256, 6), sdesc(B, 256, 6), idesc(N), 1);
            } else if (mode == 4) {  // SW128 K-major, K step r % 4 = 32 B into the 128 B row
                for (int r = 0; r < nrep; ++r)
                    mma_ss(tmem, sdesc(A + 32 * (r & 3), 1024, 2), sdesc(B + 32 * (r & 3), 1024, 2), idesc(N), 1);
            } else if (mode == 5) {  // TS, B SW128
                for (int r = 0; r < nrep; ++r)
                    mma_ts(tmem, tmem + 400 + 8 * (r & 3), sdesc(B + 32 * (r & 3), 1024, 2), idesc(N), 1);
            } else if (mode == 6) {  // SW64 (64 B rows, 2 K steps), SBO 512
                for (int r = 0; r < nrep; ++r)
                    mma_ss(tmem, sdesc(A + 32 * (r & 1), 512, 4), sdesc(B + 32 * (r & 1), 512, 4), idesc(N), 1);
            } else if (mode == 7) {  // SW32 but 8 MMAs into 8 different accumulators
                for (int r = 0; r < nrep; ++r)
                    mma_ss(tmem + (r & 7) * N, sdesc(A, 256, 6), sdesc(B, 256, 6), idesc(N), 1);
            }
            commit(&bars[it % 4]);
            if (it >= lag) wait(&bars[(it - lag) % 4], ((it - lag) / 4) & 1);
        }
        for (int it = iters - lag > 0 ? iters - lag : 0; it < iters; ++it) wait(&bars[it % 4], (it / 4) & 1);
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    struct Cfg { int mode, N, lag, nrep; const char* name; } cfgs[] = {
        {0, 48, 1, 1, "oz pattern SS SW32 N48, wait each round"},
        {0, 48, 3, 1, "oz pattern SS SW32 N48, lag 3"},
        {1, 48, 3, 1, "oz pattern TS (A tmem) N48, lag 3"},
        {1, 32, 3, 1, "oz pattern TS N32, lag 3"},
        {0, 48, 3, 4, "oz pattern SS N48 x4 per round, lag 3"},
        {2, 256, 3, 8, "single N=256 SS x8, lag 3"},
        {2, 128, 3, 8, "single N=128 SS x8, lag 3"},
        {2, 48, 3, 8, "single N=48 SS x8, lag 3"},
        {2, 16, 3, 8, "single N=16 SS x8, lag 3"},
        {4, 256, 3, 8, "SW128 N=256 SS x8 (K steps)"},
        {4, 128, 3, 8, "SW128 N=128 SS x8 (K steps)"},
        {4, 48, 3, 8, "SW128 N=48 SS x8 (K steps)"},
        {5, 128, 3, 8, "SW128 N=128 TS x8 (K steps)"},
        {5, 48, 3, 8, "SW128 N=48 TS x8 (K steps)"},
        {6, 128, 3, 8, "SW64 N=128 SS x8 (K steps)"},
        {6, 48, 3, 8, "SW64 N=48 SS x8 (K steps)"},
        {7, 48, 3, 8, "SW32 N=48 SS x8, 8 accumulators"},
        {2, 128, 3, 32, "single N=128 SS x32, lag 3"},
        {10, 128, 3, 8, "elect: N=128 SS x8"},
        {10, 128, 3, 32, "elect: N=128 SS x32"},
        {10, 48, 3, 8, "elect: N=48 SS x8"},
        {10, 48, 3, 32, "elect: N=48 SS x32"},
        {10, 256, 3, 8, "elect: N=256 SS x8"},
        {11, 48, 3, 8, "elect: N=48 TS x8"},
        {11, 48, 3, 32, "elect: N=48 TS x32"},
        {12, 48, 3, 28, "elect: 28 separate N=48 TS (7 accumulators)"},
        {12, 48, 3, 56, "elect: 56 separate N=48 TS"},
        {13, 48, 3, 9, "elect: 9 TS alternating N 48/96/144"},
        {13, 48, 3, 36, "elect: 36 TS alternating N 48/96/144"},
        {14, 48, 3, 9, "elect: 9 TS N=144 offsets vary"},
        {14, 48, 3, 36, "elect: 36 TS N=144 offsets vary"},
    };
    for (auto& c : cfgs) {
        const int iters = 2000;
        probe<<<148, 128, 100 * 1024>>>(c.mode, c.N, iters, c.lag, d, c.nrep);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", c.name, cudaGetErrorString(e)); return 1; }
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double cyc = 0; for (int i = 0; i < 148; ++i) cyc += h[i]; cyc /= 148;
        double nsum = c.mode == 13 ? c.N * 2.0 : c.mode == 14 ? c.N * 3.0 : c.N;
        double ops_round = c.mode >= 2 && c.mode != 3 ? 2.0 * 128 * nsum * 32 * c.nrep : 2.0 * 128 * 28 * c.N * 32 * c.nrep;
        printf("%-45s %8.1f cycles/round  %7.0f int8 ops/cycle/SM (peak 16384)\n", c.name, cyc / iters, ops_round * iters / cyc);
    }
    return 0;
}
