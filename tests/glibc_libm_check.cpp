// Host check of csrc/glibc_libm.cuh (the restated glibc 2.39 __log_fma / __sincos_fma)
// against this host's libm, bit for bit. Built and run by tests/test_glibc_libm.py.
//   glibc_libm_check <n> <seed>
// draws n uniforms exactly as the reference sampler does (rng.cpp:22-32) and checks
// log(u) and sincos(2 pi u); then n arbitrary doubles spread over the domain of each
// branch ([2^-53, 4] for log; (-2 pi, 2 pi) and the branch boundaries for sincos).
// Prints "mismatches <log> <sin> <cos> of <count>" and exits non-zero on any mismatch.
#define _GNU_SOURCE 1
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_2110_03423_b200/csrc/glibc_libm.cuh"

extern "C" void sincos(double, double*, double*);
extern "C" double log(double);

static uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

// through pointers so the compiler cannot fold or substitute builtins
static double (*volatile libm_log)(double) = &log;
static void (*volatile libm_sincos)(double, double*, double*) = &sincos;

static long bad_log = 0, bad_sin = 0, bad_cos = 0, count = 0;

static bool same(double a, double b) { return memcmp(&a, &b, 8) == 0; }

static void check_log(double u) {
    const double want = libm_log(u), got = glibc239::log(u);
    if (!same(want, got) && bad_log++ < 5)
        printf("log(%a): libm %a restated %a\n", u, want, got);
}

static void check_sincos(double x) {
    double ws, wc, gs, gc;
    libm_sincos(x, &ws, &wc);
    glibc239::sincos(x, &gs, &gc);
    if (!same(ws, gs) && bad_sin++ < 5) printf("sin(%a): libm %a restated %a\n", x, ws, gs);
    if (!same(wc, gc) && bad_cos++ < 5) printf("cos(%a): libm %a restated %a\n", x, wc, gc);
    ++count;
}

int main(int argc, char** argv) {
    const long n = argc > 1 ? atol(argv[1]) : 1000000;
    const uint64_t seed = argc > 2 ? strtoull(argv[2], nullptr, 0) : 42;
    // the sampler's own inputs
    for (long c = 1; c <= n; ++c) {
        const uint64_t w = mix64(seed + (uint64_t)c * 0x9E3779B97F4A7C15ULL);
        const double u = (double)((w >> 11) + 1) * 0x1.0p-53;
        check_log(u);
        check_sincos(2.0 * M_PI * u);
    }
    // arbitrary doubles over every branch of the domain
    uint64_t st = seed ^ 0x5DEECE66DULL;
    for (long i = 0; i < n; ++i) {
        st = mix64(st + 0x9E3779B97F4A7C15ULL);
        const double f = (double)(st >> 11) * 0x1.0p-53;  // [0, 1)
        const int e = (int)(st & 63);
        check_log(std::ldexp(0.5 + f, -(e % 54)));          // [2^-54, 1)
        check_log(0.9375 + f * 0.13);                        // the |x - 1| < 1/16 branch
        check_log(1.0 + 3.0 * f);
        const double x = (2.0 * f - 1.0) * 6.283185307179586;
        check_sincos(x);
        check_sincos(std::ldexp(x, -(e % 30)));              // small angles, Taylor branch
        // the branch boundaries 2^-27, 0.855469, 2.426265 and pi/2 multiples
        const double edges[] = {0x1p-27, 0.85546875, 2.426265, 1.5707963267948966,
                                3.141592653589793, 4.71238898038469, 6.283185307179586};
        const double ed = edges[st % 7] * (1.0 + (f - 0.5) * 1e-6);
        check_sincos(ed);
        check_sincos(-ed);
    }
    printf("mismatches %ld %ld %ld of %ld\n", bad_log, bad_sin, bad_cos, count);
    return (bad_log || bad_sin || bad_cos) ? 1 : 0;
}
