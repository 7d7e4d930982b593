// Gaussian sketch generator: the reference's counter-based SplitMix64 stream and
// Box-Muller transform (rng.cpp:9-51), evaluated in parallel and written straight
// into the transposed operand layout the ax GEMM consumes (Omega^T, NP x n).
//
// Stream facts restated from the reference:
//   word(c)  = mix64(seed + c * 0x9E3779B97F4A7C15), counters start at 1 (rng.cpp:24-27)
//   uniform  = ((word >> 11) + 1) * 2^-53 in (0, 1]                   (rng.cpp:29-32)
//   normals come in pairs: pair p uses counters 2p+1 (u1) and 2p+2 (u2);
//   normal 2p = r*cos(2*pi*u2), normal 2p+1 = r*sin(2*pi*u2), r = sqrt(-2 log u1)
//   (the sine half is cached for the next draw, rng.cpp:34-46)
//   Omega(r, c) = normal #(r*s + c) of a fresh sampler (rng.cpp:48-53, rsvd.cpp:128).
// Words and uniforms are exact integer / power-of-two arithmetic; sqrt and the three
// products are single IEEE roundings on both sides; log and sincos are glibc 2.39's FMA
// builds restated instruction for instruction (glibc_libm.cuh), the functions the
// reference's compiled rng.cpp calls on this image. So Omega is the reference's Omega bit
// for bit (tests/test_gpu_parity.py compares with array_equal; the C2 Omega hashes to the
// SURVEY.md Appendix A prefix 4df3a9577d3f11db).
#include "common.cuh"
#include "glibc_libm.cuh"
#include "kernels.h"

namespace rsvdb200 {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

__device__ __forceinline__ uint64_t word_at(uint64_t seed, uint64_t counter) {
    return mix64(seed + counter * 0x9E3779B97F4A7C15ULL);
}

__device__ __forceinline__ double uniform_from_word(uint64_t w) {
    return static_cast<double>((w >> 11) + 1) * 0x1.0p-53;
}

// Both normals of the pair whose words sit at counters base + 1 (radius) and base + 2
// (angle); a fresh sampler's pair p has base 2p.
__device__ __forceinline__ void box_muller_at(uint64_t seed, uint64_t base, double& n0,
                                              double& n1) {
    const double u1 = uniform_from_word(word_at(seed, base + 1));
    const double u2 = uniform_from_word(word_at(seed, base + 2));
    const double radius = __dsqrt_rn(__dmul_rn(-2.0, glibc239::log(u1)));
    const double angle = __dmul_rn(2.0 * 3.14159265358979323846, u2);
    double s, c;
    glibc239::sincos(angle, &s, &c);
    n0 = __dmul_rn(radius, c);
    n1 = __dmul_rn(radius, s);
}

// Output element i (0 <= i < total) is the i-th normal a GaussianSampler in state `pos`
// would return (rng.cpp:34-46): its cached sine half first when pos.has_cached (passed in
// bit for bit), then pairs j = 0, 1, ... built from the words at counters
// pos.counter + 2j + 1 (radius) and pos.counter + 2j + 2 (angle), cosine half first.
template <class Store>
__device__ __forceinline__ void stream_normals(uint64_t seed, StreamPos pos, long total,
                                               Store store) {
    if (total <= 0) return;
    const long off = pos.has_cached ? 1 : 0;
    if (off && blockIdx.x == 0 && threadIdx.x == 0) store(0, pos.cached);
    const long rest = total - off, pairs = (rest + 1) / 2;
    for (long j = blockIdx.x * (long)blockDim.x + threadIdx.x; j < pairs;
         j += (long)gridDim.x * blockDim.x) {
        double v0, v1;
        box_muller_at(seed, pos.counter + 2 * (uint64_t)j, v0, v1);
        store(off + 2 * j, v0);
        if (2 * j + 1 < rest) store(off + 2 * j + 1, v1);
    }
}

__global__ void omega_t_kernel(uint64_t seed, StreamPos pos, long n, int s, int NP,
                               double* __restrict__ out, long ld) {
    const long total = n * (long)s;
    stream_normals(seed, pos, total,
                   [&](long i, double v) { out[(i % s) * ld + i / s] = v; });
    // zero the padding rows s..NP-1 of Omega^T
    const long pad = (long)(NP - s) * n;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < pad;
         e += (long)gridDim.x * blockDim.x)
        out[(s + e / n) * ld + e % n] = 0.0;
}

__global__ void gaussian_rowmajor_kernel(uint64_t seed, StreamPos pos, long total,
                                         double* __restrict__ out) {
    stream_normals(seed, pos, total, [&](long i, double v) { out[i] = v; });
}

__global__ void words_kernel(uint64_t seed, uint64_t first, long count, uint64_t* out) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count;
         i += (long)gridDim.x * blockDim.x)
        out[i] = word_at(seed, first + (uint64_t)i);
}

__global__ void uniforms_kernel(uint64_t seed, uint64_t first, long count, double* out) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count;
         i += (long)gridDim.x * blockDim.x)
        out[i] = uniform_from_word(word_at(seed, first + (uint64_t)i));
}

static unsigned grid_for(long work, int threads) {
    long b = (work + threads - 1) / threads;
    if (b > 148L * 16) b = 148L * 16;
    return (unsigned)(b < 1 ? 1 : b);
}

cudaError_t launch_omega(uint64_t seed, long n, int s, int NP, double* omega_t, long ld,
                         cudaStream_t st, StreamPos pos) {
    const long work = (n * (long)s + 2) / 2;
    omega_t_kernel<<<grid_for(work, 256), 256, 0, st>>>(seed, pos, n, s, NP, omega_t, ld);
    return cudaGetLastError();
}

cudaError_t launch_gaussian_rowmajor(uint64_t seed, long rows, long cols, double* out,
                                     cudaStream_t st, StreamPos pos) {
    const long total = rows * cols;
    gaussian_rowmajor_kernel<<<grid_for((total + 2) / 2, 256), 256, 0, st>>>(seed, pos, total,
                                                                             out);
    return cudaGetLastError();
}

cudaError_t launch_splitmix_words(uint64_t seed, uint64_t first_counter, long count,
                                  uint64_t* out, cudaStream_t st) {
    words_kernel<<<grid_for(count, 256), 256, 0, st>>>(seed, first_counter, count, out);
    return cudaGetLastError();
}

cudaError_t launch_uniforms(uint64_t seed, uint64_t first_counter, long count, double* out,
                            cudaStream_t st) {
    uniforms_kernel<<<grid_for(count, 256), 256, 0, st>>>(seed, first_counter, count, out);
    return cudaGetLastError();
}

}  // namespace rsvdb200
