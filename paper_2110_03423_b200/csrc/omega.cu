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
// Words and uniforms are exact integer / power-of-two arithmetic and match the
// reference bit for bit; sqrt and the two products are single IEEE roundings on
// both sides. log, sin and cos are evaluated here in double-double arithmetic
// (~104 bits) and rounded once, i.e. correctly rounded; the reference calls glibc,
// whose results are within ~0.52 ulp, so the two agree except where glibc itself
// misrounds (~0.2% of Omega entries, by 1 ulp; the reference's own Omega already
// differs between glibc's FMA and non-FMA code paths). Bit-exact Omega parity is
// available through validation mode (rsvd_b200_set_omega).
#include "common.cuh"
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

// ------------------------------------------------ double-double arithmetic
struct dd {
    double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}
__device__ __forceinline__ dd fast_two_sum(double a, double b) {  // |a| >= |b|
    const double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
    const double p = __dmul_rn(a, b);
    return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    const dd t = two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = fast_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return fast_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo = __fma_rn(a.hi, b.lo, __fma_rn(a.lo, b.hi, p.lo));
    return fast_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
    dd p = two_prod(a.hi, b);
    p.lo = __fma_rn(a.lo, b, p.lo);
    return fast_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_div(dd a, dd b) {
    const double q1 = __ddiv_rn(a.hi, b.hi);
    dd r = dd_sub(a, dd_mul_d(b, q1));
    const double q2 = __ddiv_rn(r.hi, b.hi);
    r = dd_sub(r, dd_mul_d(b, q2));
    const double q3 = __ddiv_rn(r.hi, b.hi);
    return dd_add(fast_two_sum(q1, q2), dd{q3, 0.0});
}

// 1/(2j+1), j = 0..24, as double-doubles (hi + lo, exact rational rounding; generated)
__constant__ double kInvOdd[25][2] = {
    {0x1.0000000000000p+0, 0x0.0p+0},
    {0x1.5555555555555p-2, 0x1.5555555555555p-56},
    {0x1.999999999999ap-3, -0x1.999999999999ap-57},
    {0x1.2492492492492p-3, 0x1.2492492492492p-57},
    {0x1.c71c71c71c71cp-4, 0x1.c71c71c71c71cp-58},
    {0x1.745d1745d1746p-4, -0x1.745d1745d1746p-59},
    {0x1.3b13b13b13b14p-4, -0x1.3b13b13b13b14p-58},
    {0x1.1111111111111p-4, 0x1.1111111111111p-60},
    {0x1.e1e1e1e1e1e1ep-5, 0x1.e1e1e1e1e1e1ep-61},
    {0x1.af286bca1af28p-5, 0x1.af286bca1af28p-59},
    {0x1.8618618618618p-5, 0x1.8618618618618p-59},
    {0x1.642c8590b2164p-5, 0x1.642c8590b2164p-60},
    {0x1.47ae147ae147bp-5, -0x1.eb851eb851eb8p-61},
    {0x1.2f684bda12f68p-5, 0x1.2f684bda12f68p-59},
    {0x1.1a7b9611a7b96p-5, 0x1.1a7b9611a7b96p-61},
    {0x1.0842108421084p-5, 0x1.0842108421084p-60},
    {0x1.f07c1f07c1f08p-6, -0x1.f07c1f07c1f08p-61},
    {0x1.d41d41d41d41dp-6, 0x1.0750750750750p-60},
    {0x1.bacf914c1bad0p-6, -0x1.bacf914c1bad0p-60},
    {0x1.a41a41a41a41ap-6, 0x1.0690690690690p-60},
    {0x1.8f9c18f9c18fap-6, -0x1.f3831f3831f38p-61},
    {0x1.7d05f417d05f4p-6, 0x1.7d05f417d05f4p-62},
    {0x1.6c16c16c16c17p-6, -0x1.f49f49f49f49fp-61},
    {0x1.5c9882b931057p-6, 0x1.310572620ae4cp-61},
    {0x1.4e5e0a72f0539p-6, 0x1.e0a72f0539783p-60},
};
// 1/n!, n = 0..31, as double-doubles
__constant__ double kInvFact[32][2] = {
    {0x1.0000000000000p+0, 0x0.0p+0},
    {0x1.0000000000000p+0, 0x0.0p+0},
    {0x1.0000000000000p-1, 0x0.0p+0},
    {0x1.5555555555555p-3, 0x1.5555555555555p-57},
    {0x1.5555555555555p-5, 0x1.5555555555555p-59},
    {0x1.1111111111111p-7, 0x1.1111111111111p-63},
    {0x1.6c16c16c16c17p-10, -0x1.f49f49f49f49fp-65},
    {0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-73},
    {0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76},
    {0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73},
    {0x1.27e4fb7789f5cp-22, 0x1.cbbc05b4fa99ap-76},
    {0x1.ae64567f544e4p-26, -0x1.c062e06d1f209p-80},
    {0x1.1eed8eff8d898p-29, -0x1.2aec959e14c06p-83},
    {0x1.6124613a86d09p-33, 0x1.f28e0cc748ebep-87},
    {0x1.93974a8c07c9dp-37, 0x1.05d6f8a2efd1fp-92},
    {0x1.ae7f3e733b81fp-41, 0x1.1d8656b0ee8cbp-97},
    {0x1.ae7f3e733b81fp-45, 0x1.1d8656b0ee8cbp-101},
    {0x1.952c77030ad4ap-49, 0x1.ac981465ddc6cp-103},
    {0x1.6827863b97d97p-53, 0x1.eec01221a8b0bp-107},
    {0x1.2f49b46814157p-57, 0x1.2650f61dbdcb4p-112},
    {0x1.e542ba4020225p-62, 0x1.ea72b4afe3c2fp-120},
    {0x1.71b8ef6dcf572p-66, -0x1.d043ae40c4647p-120},
    {0x1.0ce396db7f853p-70, -0x1.aebcdbd20331cp-124},
    {0x1.761b41316381ap-75, -0x1.3423c7d91404fp-130},
    {0x1.f2cf01972f578p-80, -0x1.9ada5fcc1ab14p-135},
    {0x1.3f3ccdd165fa9p-84, -0x1.58ddadf344487p-139},
    {0x1.88e85fc6a4e5ap-89, -0x1.71c37ebd16540p-143},
    {0x1.d1ab1c2dccea3p-94, 0x1.054d0c78aea14p-149},
    {0x1.0a18a2635085dp-98, 0x1.b9e2e28e1aa54p-153},
    {0x1.259f98b4358adp-103, 0x1.eaf8c39dd9bc5p-157},
    {0x1.3932c5047d60ep-108, 0x1.832b7b530a627p-162},
    {0x1.434d2e783f5bcp-113, 0x1.0b87b91be9affp-167},
};

__device__ __forceinline__ dd kdd(const double (&t)[2]) { return dd{t[0], t[1]}; }

// Correctly rounded (to ~2^-104 before the final rounding) natural log of u in (0, 1]:
// u = 2^e m, m in [sqrt(2)/2, sqrt(2)); log m = 2 atanh(f), f = (m - 1)/(m + 1).
__device__ double log_cr(double u) {
    if (u == 1.0) return 0.0;
    int e;
    double m = frexp(u, &e);  // m in [0.5, 1)
    if (m < 0.70710678118654752440) {
        m *= 2.0;
        e -= 1;
    }
    const dd num = {__dsub_rn(m, 1.0), 0.0};  // exact (Sterbenz)
    const dd den = two_sum(m, 1.0);
    const dd f = dd_div(num, den);
    const dd f2 = dd_mul(f, f);
    // atanh(f)/f = sum_j f^(2j) / (2j + 1), |f| <= 0.1716: 24 terms reach 2^-120
    dd acc = kdd(kInvOdd[24]);
    for (int j = 23; j >= 0; --j) acc = dd_add(dd_mul(acc, f2), kdd(kInvOdd[j]));
    dd lm = dd_mul(dd_mul_d(f, 2.0), acc);
    const dd ln2 = {0.69314718055994528623, 2.3190468138462996e-17};
    return dd_add(dd_mul_d(ln2, (double)e), lm).hi;
}

// Correctly rounded sin and cos of x in [0, 2*pi]: reduce by pi/2 with a
// triple-double pi/2, then Taylor series in double-double.
__device__ void sincos_cr(double x, double* sn, double* cs) {
    const double p1 = 1.5707963267948966192, p2 = 6.123233995736766036e-17,
                 p3 = -1.4973849048591698e-33;
    const double kq = rint(x * 0.63661977236758134308);
    dd r = dd_sub(dd{x, 0.0}, two_prod(kq, p1));
    r = dd_sub(r, two_prod(kq, p2));
    r = dd_sub(r, dd{kq * p3, 0.0});
    const dd r2 = dd_mul(r, r);
    // sin r = r * sum (-1)^j r^(2j) / (2j+1)!,  cos r = sum (-1)^j r^(2j) / (2j)!, j <= 15
    dd s = kdd(kInvFact[31]), c = kdd(kInvFact[30]);
    for (int j = 14; j >= 0; --j) {
        s = dd_add(dd_neg(dd_mul(s, r2)), kdd(kInvFact[2 * j + 1]));
        c = dd_add(dd_neg(dd_mul(c, r2)), kdd(kInvFact[2 * j]));
    }
    s = dd_mul(s, r);
    const int q = ((int)kq) & 3;
    double sv = s.hi, cv = c.hi;
    switch (q) {
        case 0: *sn = sv; *cs = cv; break;
        case 1: *sn = cv; *cs = -sv; break;
        case 2: *sn = -sv; *cs = -cv; break;
        default: *sn = -cv; *cs = sv; break;
    }
}

// Both normals of the pair whose words sit at counters base + 1 (radius) and base + 2
// (angle); a fresh sampler's pair p has base 2p.
__device__ __forceinline__ void box_muller_at(uint64_t seed, uint64_t base, double& n0,
                                              double& n1) {
    const double u1 = uniform_from_word(word_at(seed, base + 1));
    const double u2 = uniform_from_word(word_at(seed, base + 2));
    const double radius = __dsqrt_rn(__dmul_rn(-2.0, log_cr(u1)));
    const double angle = __dmul_rn(2.0 * 3.14159265358979323846, u2);
    double s, c;
    sincos_cr(angle, &s, &c);
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
