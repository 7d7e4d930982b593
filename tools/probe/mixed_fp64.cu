// Microbenchmark: do DMMA (FP64 tensor) and DFMA (FP64 SIMT) share one pipe on B200?
// Warps [0, split) run m16n8k16 DMMA chains, warps [split, 8) run DFMA chains, in the same
// CTA; if the two pipes were independent, the combined FLOP/s would exceed either alone.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
      "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// iters_mma DMMA rounds (4 chains) for DMMA warps, iters_fma rounds (64 DFMA) for DFMA warps;
// mode 2 = every warp interleaves both.
__global__ void mixed(double* out, int split, int iters_mma, int iters_fma, int mode) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  const bool do_mma = mode == 2 || warp < split;
  const bool do_fma = mode == 2 || warp >= split;
  double acc[4][4];
  for (int t = 0; t < 4; ++t) for (int r = 0; r < 4; ++r) acc[t][r] = 0;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = (threadIdx.x + i) * 1e-3;
  for (int i = 0; i < 4; ++i) b[i] = (threadIdx.x - i) * 1e-3;
  double f0 = threadIdx.x * 1e-3, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3, f4 = f0 + 4, f5 = f0 + 5,
         f6 = f0 + 6, f7 = f0 + 7;
  const double fb = 0.999999, fc = 1e-7;
  const int n = mode == 2 ? iters_mma : (do_mma ? iters_mma : iters_fma);
  for (int i = 0; i < n; ++i) {
    if (do_mma) {
#pragma unroll
      for (int t = 0; t < 4; ++t) dmma(acc[t], a, b);
    }
    if (do_fma) {
      const int reps = mode == 2 ? 1 : 8;
      for (int j = 0; j < reps; ++j) {
        f0 = fma(f0, fb, fc); f1 = fma(f1, fb, fc); f2 = fma(f2, fb, fc); f3 = fma(f3, fb, fc);
        f4 = fma(f4, fb, fc); f5 = fma(f5, fb, fc); f6 = fma(f6, fb, fc); f7 = fma(f7, fb, fc);
      }
    }
  }
  for (int t = 0; t < 4; ++t) for (int r = 0; r < 4; ++r) s += acc[t][r];
  s += f0 + f1 + f2 + f3 + f4 + f5 + f6 + f7;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 4 * 256 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 148 * 2, threads = 256;
  auto run = [&](int split, int im, int ifm, int mode, const char* name) {
    mixed<<<grid, threads>>>(out, split, im, ifm, mode);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    mixed<<<grid, threads>>>(out, split, im, ifm, mode);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const int wm = mode == 2 ? 8 : split, wf = mode == 2 ? 8 : 8 - split;
    const int ifm_eff = mode == 2 ? im : ifm;
    const int fma_per_iter = mode == 2 ? 8 : 64;
    double fl_m = 2.0 * 16 * 8 * 16 * 4 * (double)im * wm * grid;
    double fl_f = 2.0 * fma_per_iter * 32 * (double)ifm_eff * wf * grid;
    printf("%-28s %.3f ms  DMMA %.2f + DFMA %.2f = %.2f TFLOP/s (%s)\n", name, ms,
           fl_m / ms / 1e9, fl_f / ms / 1e9, (fl_m + fl_f) / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(8, 2048, 0, 0, "DMMA only (8 warps)");
  run(0, 0, 4096, 0, "DFMA only (8 warps)");
  run(4, 2048, 4096, 0, "4 DMMA + 4 DFMA warps");
  run(4, 2048, 2048, 0, "4 DMMA + 4 DFMA (half fma)");
  run(6, 2048, 1024, 0, "6 DMMA + 2 DFMA warps");
  run(0, 2048, 0, 2, "interleaved 4 DMMA : 8 DFMA");
  return 0;
}
