// TEST INFRASTRUCTURE ONLY — extern "C" shim over the UNMODIFIED reference library.
//
// oracle/Makefile compiles this file together with the reference sources
// (/root/reference/proj/src/{matrix,parallel,gemm,qr,svd,rng,rsvd}.cpp, read in
// place, never copied) into oracle/_ref/libranddsvd_ref.so. It exists so that
// tests/ can pin the C restatement (oracle/rsvd_oracle.c) and the golden
// fixtures to the reference's own outputs, and so that bench.py's
// `--impl reference` / cpu_baseline legs can time the reference CPU path
// itself. Signatures mirror oracle/rsvd_oracle.h with a `ref_` prefix.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include <sstream>

#include "randsvd/bench.hpp"
#include "randsvd/errors.hpp"
#include "randsvd/gemm.hpp"
#include "randsvd/matrix.hpp"
#include "randsvd/parallel.hpp"
#include "randsvd/qr.hpp"
#include "randsvd/rng.hpp"
#include "randsvd/rsvd.hpp"
#include "randsvd/svd.hpp"
#include "randsvd/synth.hpp"

using namespace randsvd;

namespace {

thread_local std::string g_err;

DenseMatrix from(const double* p, std::size_t r, std::size_t c) {
    return DenseMatrix(r, c, std::vector<double>(p, p + r * c));
}

void to(const DenseMatrix& m, double* out) {
    if (out) std::memcpy(out, m.data().data(), m.size() * sizeof(double));
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ArgumentError& e) {
        g_err = e.what();
        return 1;
    } catch (const DimensionError& e) {
        g_err = e.what();
        return 2;
    } catch (const ConvergenceError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_max_threads(unsigned n) { set_max_threads(n); }

void ref_splitmix_words(std::uint64_t seed, std::size_t count, std::uint64_t* out) {
    GaussianSampler s(seed);
    for (std::size_t i = 0; i < count; ++i) out[i] = s.next_u64();
}

void ref_uniforms(std::uint64_t seed, std::size_t count, double* out) {
    GaussianSampler s(seed);
    for (std::size_t i = 0; i < count; ++i) out[i] = s.uniform01();
}

void ref_gaussian_matrix(std::uint64_t seed, std::size_t rows, std::size_t cols, double* out) {
    GaussianSampler s(seed);
    to(gaussian_matrix(s, rows, cols), out);
}

// `count` normals of a sampler that first returned `skip_words` raw words (next_u64) and
// then `skip_normals` normals: the continuation cases of sketch / gaussian_matrix
void ref_sampler_normals(std::uint64_t seed, std::size_t skip_words, std::size_t skip_normals,
                         std::size_t count, double* out) {
    GaussianSampler s(seed);
    for (std::size_t i = 0; i < skip_words; ++i) s.next_u64();
    for (std::size_t i = 0; i < skip_normals; ++i) s.normal();
    for (std::size_t i = 0; i < count; ++i) out[i] = s.normal();
}

// synth::synth_matrix (synth.cpp:58-71); kind 0 fast, 1 sharp(beta), 2 slow
int ref_synth_matrix(std::size_t rows, std::size_t cols, int kind, double beta,
                     std::uint64_t seed, double* out) {
    return guarded([&] {
        const synth::SpectrumKind k = kind == 0   ? synth::SpectrumKind::fast()
                                      : kind == 1 ? synth::SpectrumKind::sharp(beta)
                                                  : synth::SpectrumKind::slow();
        to(synth::synth_matrix({rows, cols, k, seed}), out);
    });
}

// bench::run_grid of a named preset (bench.cpp:112-172, 239-260) with `reps` repetitions,
// written by bench::write_csv into buf (NUL-terminated); returns the CSV length, or -1
// (error text in ref_last_error) / -2 (buffer too small).
long ref_run_grid_csv(const char* preset, std::size_t reps, char* buf, std::size_t cap) {
    std::string csv;
    const int rc = guarded([&] {
        bench::GridConfig g = bench::preset(preset);
        g.repetitions = reps;
        std::ostringstream os;
        bench::write_csv(bench::run_grid(g).rows, os);
        csv = os.str();
    });
    if (rc != 0) return -1;
    if (csv.size() + 1 > cap) return -2;
    std::memcpy(buf, csv.c_str(), csv.size() + 1);
    return (long)csv.size();
}

double ref_pairwise_dot(const double* x, const double* y, std::size_t n) {
    return pairwise_dot(std::span<const double>(x, n), std::span<const double>(y, n));
}

int ref_gemm(double alpha, const double* a, std::size_t ar, std::size_t ac, int ta,
             const double* b, std::size_t br, std::size_t bc, int tb, double beta,
             const double* c, double* out) {
    return guarded([&] {
        const std::size_t m = ta ? ac : ar, n = tb ? br : bc;
        const DenseMatrix cm = beta != 0.0 ? from(c, m, n) : DenseMatrix(1, 1);
        to(gemm(alpha, from(a, ar, ac), ta != 0, from(b, br, bc), tb != 0, beta, cm), out);
    });
}

int ref_householder_qr(const double* a, std::size_t m, std::size_t n, double* q, double* r) {
    return guarded([&] {
        const QrFactors f = householder_qr(from(a, m, n));
        to(f.q, q);
        to(f.r, r);
    });
}

int ref_dense_svd(const double* a, std::size_t m, std::size_t n, double* u, double* sigma,
                  double* v) {
    return guarded([&] {
        const SvdFactors f = dense_svd(from(a, m, n));
        to(f.u, u);
        std::memcpy(sigma, f.sigma.data(), f.sigma.size() * sizeof(double));
        to(f.v, v);
    });
}

int ref_extend_orthonormal(const double* u, std::size_t m, std::size_t r0, std::size_t target,
                           double* out) {
    return guarded([&] { to(extend_orthonormal(from(u, m, r0), target), out); });
}

std::size_t ref_sketch_width(std::size_t k, std::size_t oversample, double epsilon,
                             int epsilon_mode, std::size_t m, std::size_t n) {
    RsvdConfig cfg;
    cfg.k = k;
    cfg.oversample = oversample;
    cfg.epsilon = epsilon;
    cfg.epsilon_mode = epsilon_mode != 0;
    return cfg.sketch_width(m, n);
}

int ref_sketch(const double* a, std::size_t m, std::size_t n, std::size_t s, std::uint64_t seed,
               double* y0) {
    return guarded([&] {
        GaussianSampler sampler(seed);
        to(sketch(from(a, m, n), s, sampler), y0);
    });
}

int ref_power_iterate(const double* a, std::size_t m, std::size_t n, const double* y0,
                      std::size_t s, std::size_t q, double* w) {
    return guarded([&] { to(power_iterate(from(a, m, n), from(y0, m, s), q), w); });
}

int ref_range_basis(const double* y, std::size_t m, std::size_t s, double* q,
                    std::size_t* cols_out) {
    return guarded([&] {
        const DenseMatrix out = range_basis(from(y, m, s));
        to(out, q);
        *cols_out = out.cols();
    });
}

int ref_project_and_solve(const double* a, std::size_t m, std::size_t n, const double* qb,
                          std::size_t sq, std::size_t k, double* u, double* sigma, double* v,
                          std::size_t* sketch_width) {
    return guarded([&] {
        const RsvdResult r = project_and_solve(from(a, m, n), from(qb, m, sq), k);
        to(r.factors.u, u);
        std::memcpy(sigma, r.factors.sigma.data(), r.factors.sigma.size() * sizeof(double));
        to(r.factors.v, v);
        *sketch_width = r.sketch_width;
    });
}

// Full pipeline. The input is borrowed through a DenseMatrix copy made OUTSIDE
// any timing the caller does around ref_randomized_ksvd_prepared below.
int ref_randomized_ksvd(const double* a, std::size_t m, std::size_t n, std::size_t k,
                        std::size_t oversample, std::size_t power_q, std::uint64_t seed,
                        double epsilon, int epsilon_mode, int values_only, double* u,
                        double* sigma, double* v, std::size_t* sketch_width) {
    return guarded([&] {
        RsvdConfig cfg;
        cfg.k = k;
        cfg.oversample = oversample;
        cfg.power_q = power_q;
        cfg.seed = seed;
        cfg.epsilon = epsilon;
        cfg.epsilon_mode = epsilon_mode != 0;
        const DenseMatrix am = from(a, m, n);
        if (values_only) {
            const std::vector<double> s = singular_values_only(am, cfg);
            std::memcpy(sigma, s.data(), s.size() * sizeof(double));
            if (sketch_width) *sketch_width = 0;
            return;
        }
        const RsvdResult r = randomized_ksvd(am, cfg);
        to(r.factors.u, u);
        std::memcpy(sigma, r.factors.sigma.data(), r.factors.sigma.size() * sizeof(double));
        to(r.factors.v, v);
        if (sketch_width) *sketch_width = r.sketch_width;
    });
}

// Timing helpers for the CPU baseline: hold a DenseMatrix built once so the
// timed call is exactly randsvd::randomized_ksvd(a, cfg), as cli.cpp:256-266 times it.
void* ref_matrix_new(const double* a, std::size_t m, std::size_t n) {
    return new DenseMatrix(from(a, m, n));
}
void ref_matrix_free(void* h) { delete static_cast<DenseMatrix*>(h); }

int ref_randomized_ksvd_prepared(const void* h, std::size_t k, std::size_t oversample,
                                 std::size_t power_q, std::uint64_t seed, double* sigma_out) {
    return guarded([&] {
        RsvdConfig cfg;
        cfg.k = k;
        cfg.oversample = oversample;
        cfg.power_q = power_q;
        cfg.seed = seed;
        const RsvdResult r = randomized_ksvd(*static_cast<const DenseMatrix*>(h), cfg);
        if (sigma_out)
            std::memcpy(sigma_out, r.factors.sigma.data(), r.factors.sigma.size() * sizeof(double));
    });
}

double ref_residual_fro(const double* a, std::size_t m, std::size_t n, const double* u,
                        const double* sigma, const double* v, std::size_t k) {
    RsvdResult r{SvdFactors{from(u, m, k), std::vector<double>(sigma, sigma + k), from(v, n, k)},
                 k};
    return r.residual_fro(from(a, m, n));
}

}  // extern "C"
