// Dependent-chain latencies of the instructions on the small-side critical paths (probe only).
#include <cstdio>
__device__ __forceinline__ double rcp_nr(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}
__global__ void k(double* out, long long* cyc, double x0) {
    __shared__ double sm[64];
    const int lane = threadIdx.x;
    sm[lane] = 1.0 + lane * 1e-3; sm[lane + 32] = 0.5;
    __syncwarp();
    double x = x0 + lane * 1e-9;
    const int N = 256;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = fma(x, 0.999, 1e-3);
    t1 = clock64(); if (lane == 0) cyc[0] = (t1 - t0) / N;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = x * 1.0000001;
    t1 = clock64(); if (lane == 0) cyc[1] = (t1 - t0) / N;
    // 64-bit shfl chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
    t1 = clock64(); if (lane == 0) cyc[2] = (t1 - t0) / N;
    // rcp_nr chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = rcp_nr(x);
    t1 = clock64(); if (lane == 0) cyc[3] = (t1 - t0) / N;
    // IEEE division chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = 1.0 / x;
    t1 = clock64(); if (lane == 0) cyc[4] = (t1 - t0) / N;
    // sqrt chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = sqrt(x + 1.0);
    t1 = clock64(); if (lane == 0) cyc[5] = (t1 - t0) / N;
    // rsqrt chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = rsqrt(x + 1.0);
    t1 = clock64(); if (lane == 0) cyc[9] = (t1 - t0) / N;
    // MUFU.RSQ64H seed chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) asm("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(x));
    t1 = clock64(); if (lane == 0) cyc[10] = (t1 - t0) / N;
    // LDS dependent (pointer chasing through value)
    int idx = lane;
    t0 = clock64();
    for (int i = 0; i < N; ++i) idx = (int)sm[idx & 31] & 31;
    t1 = clock64(); if (lane == 0) cyc[6] = (t1 - t0) / N;
    // 32-bit shfl chain
    int v = lane;
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
    t1 = clock64(); if (lane == 0) cyc[7] = (t1 - t0) / N;
    // __syncthreads (1 warp)
    t0 = clock64();
    for (int i = 0; i < N; ++i) __syncthreads();
    t1 = clock64(); if (lane == 0) cyc[8] = (t1 - t0) / N;
    out[lane] = x + idx + v;
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 256); cudaMalloc(&c, 128);
    k<<<1, 32>>>(o, c, 1.5);
    k<<<1, 32>>>(o, c, 1.5);
    long long h[16];
    cudaMemcpy(h, c, 88, cudaMemcpyDeviceToHost);
    const char* n[] = {"DFMA", "DMUL", "SHFL.64", "rcp_nr", "div", "sqrt", "LDS", "SHFL.32", "bar(1w)", "rsqrt", "rsq.approx"};
    for (int i = 0; i < 11; ++i) printf("%-8s %lld cycles\n", n[i], h[i]);
}
