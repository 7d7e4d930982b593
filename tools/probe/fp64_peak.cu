// Microbenchmark: FP64 throughput on B200 — DFMA (SIMT) vs DMMA (mma.sync f64 shapes).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

template <int SHAPE>
__global__ void dmma_loop(double* out, int iters) {
  double acc[4][4];
  for (int t = 0; t < 4; ++t) for (int r = 0; r < 4; ++r) acc[t][r] = 0;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = (threadIdx.x + i) * 1e-3;
  for (int i = 0; i < 4; ++i) b[i] = (threadIdx.x - i) * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if constexpr (SHAPE == 0) {  // m8n8k4: A 1 reg, B 1 reg, C 2 regs (only use acc[t][0..1])
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[t][0]), "+d"(acc[t][1]) : "d"(a[t]), "d"(b[t]));
      } else if constexpr (SHAPE == 1) {  // m16n8k4: A 2, B 1, C 4
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3]) : "d"(a[t]), "d"(a[t+1]), "d"(b[t]));
      } else if constexpr (SHAPE == 2) {  // m16n8k8: A 4, B 2, C 4
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[t&1]), "d"(b[2+(t&1)]));
      } else {  // m16n8k16: A 8, B 4, C 4
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) for (int r = 0; r < 4; ++r) s += acc[t][r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}

int main() {
  double* out; cudaMalloc(&out, 148 * 16 * 1024 * sizeof(double));
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  for (int blocks_per_sm : {1, 2, 4}) {
    int grid = 148 * blocks_per_sm, threads = 256, iters = 4096;
    float ms = time_it([&] { dfma_loop<<<grid, threads>>>(out, iters); });
    double flops = 2.0 * 64 * iters * (double)grid * threads;
    printf("DFMA grid=%d: %.3f ms  %.2f TFLOP/s\n", grid, ms, flops / ms / 1e9);
  }
  const int kShape[4][3] = {{8, 8, 4}, {16, 8, 4}, {16, 8, 8}, {16, 8, 16}};
  for (int shape = 0; shape < 4; ++shape)
    for (int blocks_per_sm : {1, 2, 4}) {
      int grid = 148 * blocks_per_sm, threads = 256, iters = 2048;
      float ms = time_it([&] {
        if (shape == 0) dmma_loop<0><<<grid, threads>>>(out, iters);
        if (shape == 1) dmma_loop<1><<<grid, threads>>>(out, iters);
        if (shape == 2) dmma_loop<2><<<grid, threads>>>(out, iters);
        if (shape == 3) dmma_loop<3><<<grid, threads>>>(out, iters);
      });
      double per = 2.0 * kShape[shape][0] * kShape[shape][1] * kShape[shape][2];
      double flops = per * 4 * iters * (double)grid * (threads / 32);
      printf("DMMA m%dn%dk%d grid=%d: %.3f ms  %.2f TFLOP/s (%s)\n", kShape[shape][0], kShape[shape][1], kShape[shape][2],
             grid, ms, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
