// C++ drop-in for the reference API (include/randsvd/*.hpp) over the C-ABI.
//
// A user of the reference's `randsvd::randomized_ksvd(const DenseMatrix&,
// const RsvdConfig&)` (rsvd.hpp:58) relinks against librsvd_b200.so and keeps
// the same calls, value types, layout and exception types. Each host thread
// lazily owns one rsvd_b200_handle on its selected device.
#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <memory>
#include <string>

#include "../../include/randsvd/pca.hpp"
#include "../../include/randsvd/qr.hpp"
#include "../../include/randsvd/rsvd.hpp"
#include "../../include/rsvd_b200.h"

namespace randsvd {

namespace {

std::string shape_str(std::size_t r, std::size_t c) {
    return std::to_string(r) + "x" + std::to_string(c);
}

[[noreturn]] void rethrow(rsvd_b200_status st) {
    const std::string msg = rsvd_b200_last_error();
    switch (st) {
        case RSVD_B200_ARGUMENT_ERROR: throw ArgumentError(msg);
        case RSVD_B200_DIMENSION_ERROR: throw DimensionError(msg);
        case RSVD_B200_CONVERGENCE_ERROR:
            // svd.cpp:148 reports 0 iterations for a failed basis completion, svd.cpp:202
            // the sweep count, which is kSvdMaxSweeps when the Jacobi loop runs out
            throw ConvergenceError(msg, msg.find("orthonormal basis") != std::string::npos
                                            ? 0
                                            : kSvdMaxSweeps);
        default: throw DeviceError(msg);
    }
}

void check(rsvd_b200_status st) {
    if (st != RSVD_B200_OK) rethrow(st);
}

struct HandleDeleter {
    void operator()(rsvd_b200_handle* h) const { rsvd_b200_destroy(h); }
};

int default_device() {
    const char* env = std::getenv("RSVD_B200_DEVICE");
    return env ? std::atoi(env) : 0;
}

thread_local int t_device = -1;
thread_local std::unique_ptr<rsvd_b200_handle, HandleDeleter> t_handle;

rsvd_b200_handle* handle() {
    if (t_device < 0) t_device = default_device();
    if (!t_handle) {
        rsvd_b200_handle* h = nullptr;
        check(rsvd_b200_create(t_device, &h));
        t_handle.reset(h);
    }
    return t_handle.get();
}

rsvd_b200_config to_c(const RsvdConfig& cfg) {
    rsvd_b200_config c;
    c.k = cfg.k;
    c.oversample = cfg.oversample;
    c.power_q = cfg.power_q;
    c.seed = cfg.seed;
    c.epsilon = cfg.epsilon;
    c.epsilon_mode = cfg.epsilon_mode ? 1 : 0;
    return c;
}

}  // namespace

// ------------------------------------------------------------------ DenseMatrix
DenseMatrix::DenseMatrix(std::size_t rows, std::size_t cols)
    : r_(rows), c_(cols), v_(rows * cols, 0.0) {
    if (rows == 0 || cols == 0)
        throw DimensionError("DenseMatrix requires rows >= 1 and cols >= 1, got " +
                             shape_str(rows, cols));
}

DenseMatrix::DenseMatrix(std::size_t rows, std::size_t cols, std::vector<double> data)
    : r_(rows), c_(cols), v_(std::move(data)) {
    if (rows == 0 || cols == 0)
        throw DimensionError("DenseMatrix requires rows >= 1 and cols >= 1, got " +
                             shape_str(rows, cols));
    if (v_.size() != rows * cols)
        throw DimensionError("DenseMatrix " + shape_str(rows, cols) + " needs " +
                             std::to_string(rows * cols) + " values, got " +
                             std::to_string(v_.size()));
}

DenseMatrix DenseMatrix::identity(std::size_t n) {
    DenseMatrix m(n, n);
    for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
}

DenseMatrix DenseMatrix::transposed() const {
    DenseMatrix t(c_, r_);
    for (std::size_t i = 0; i < r_; ++i)
        for (std::size_t j = 0; j < c_; ++j) t(j, i) = (*this)(i, j);
    return t;
}

DenseMatrix DenseMatrix::left_cols(std::size_t count) const {
    if (count == 0 || count > c_)
        throw DimensionError("left_cols(" + std::to_string(count) + ") on a " +
                             shape_str(r_, c_) + " matrix");
    DenseMatrix out(r_, count);
    for (std::size_t i = 0; i < r_; ++i)
        for (std::size_t j = 0; j < count; ++j) out(i, j) = (*this)(i, j);
    return out;
}

bool DenseMatrix::all_finite() const noexcept {
    for (double x : v_)
        if (!std::isfinite(x)) return false;
    return true;
}

namespace {

constexpr std::size_t kPairwiseBase = 64;  // matrix.cpp's cascade base case

double cascade_sum(const double* x, std::size_t n) {
    if (n <= kPairwiseBase) {
        double acc = 0.0;
        for (std::size_t i = 0; i < n; ++i) acc += x[i];
        return acc;
    }
    const std::size_t h = n / 2;
    return cascade_sum(x, h) + cascade_sum(x + h, n - h);
}

double cascade_dot(const double* x, const double* y, std::size_t n) {
    if (n <= kPairwiseBase) {
        double acc = 0.0;
        for (std::size_t i = 0; i < n; ++i) acc += x[i] * y[i];
        return acc;
    }
    const std::size_t h = n / 2;
    return cascade_dot(x, y, h) + cascade_dot(x + h, y + h, n - h);
}

}  // namespace

double pairwise_sum(std::span<const double> x) { return cascade_sum(x.data(), x.size()); }

double pairwise_dot(std::span<const double> x, std::span<const double> y) {
    if (x.size() != y.size())
        throw DimensionError("dot of length " + std::to_string(x.size()) + " against length " +
                             std::to_string(y.size()));
    return cascade_dot(x.data(), y.data(), x.size());
}

double frobenius_norm(const DenseMatrix& a) {
    return std::sqrt(cascade_dot(a.data().data(), a.data().data(), a.size()));
}

double max_abs(const DenseMatrix& a) {
    double best = 0.0;
    for (double x : a.data()) best = std::max(best, std::abs(x));
    return best;
}

double max_abs_diff(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols())
        throw DimensionError("max_abs_diff between " + shape_str(a.rows(), a.cols()) + " and " +
                             shape_str(b.rows(), b.cols()));
    double best = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i)
        best = std::max(best, std::abs(a.data()[i] - b.data()[i]));
    return best;
}

// ------------------------------------------------------------------ GaussianSampler
// The scalar draws restate rng.cpp:22-46 on the host (same libm calls as the reference).
namespace {
constexpr std::uint64_t kGoldenGamma = 0x9E3779B97F4A7C15ULL;

std::uint64_t mix64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
}  // namespace

std::uint64_t GaussianSampler::next_u64() { return mix64(seed_ + (++counter_) * kGoldenGamma); }

double GaussianSampler::uniform01() {
    return static_cast<double>((next_u64() >> 11) + 1) * 0x1.0p-53;
}

double GaussianSampler::normal() {
    if (has_cached_) {
        has_cached_ = false;
        return cached_;
    }
    const double u1 = uniform01();
    const double u2 = uniform01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double t = 2.0 * M_PI * u2;
    cached_ = r * std::sin(t);
    has_cached_ = true;
    return r * std::cos(t);
}

namespace detail {
// Device draws continue the sampler's state and advance it as `count` normal() calls would.
struct SamplerAccess {
    static void draw(GaussianSampler& g, std::size_t count,
                     const std::function<void(std::uint64_t, int, double)>& device) {
        device(g.counter_, g.has_cached_ ? 1 : 0, g.cached_);
        std::size_t rest = count;
        if (g.has_cached_ && rest > 0) {
            g.has_cached_ = false;
            --rest;
        }
        const std::uint64_t base = g.counter_;
        g.counter_ += 2 * ((rest + 1) / 2);
        if (rest % 2 == 1) {  // the last pair's sine half stays cached in the sampler
            double two[2];
            check(rsvd_b200_gaussian_stream(handle(), g.seed_, base + rest - 1, 0, 0.0, 1, 2,
                                            two));
            g.cached_ = two[1];
            g.has_cached_ = true;
        }
    }
};
}  // namespace detail

// ------------------------------------------------------------------ thread budget
namespace {
std::atomic<unsigned> g_threads{1};
}

void set_max_threads(unsigned n) { g_threads.store(n == 0 ? 1 : n); }

unsigned max_threads() { return g_threads.load(); }

void parallel_for(std::size_t count, const std::function<void(std::size_t, std::size_t)>& body) {
    const std::size_t workers = std::min<std::size_t>(g_threads.load(), count);
    if (workers <= 1) {
        body(0, count);
        return;
    }
    const std::size_t chunk = (count + workers - 1) / workers;
    std::vector<std::thread> pool;
    for (std::size_t lo = 0; lo < count; lo += chunk)
        pool.emplace_back([&body, lo, hi = std::min(count, lo + chunk)] { body(lo, hi); });
    for (auto& t : pool) t.join();
}

// ------------------------------------------------------------------ rsvd API
void set_device(int device) {
    if (device != t_device) t_handle.reset();
    t_device = device;
}

std::size_t RsvdConfig::sketch_width(std::size_t m, std::size_t n) const {
    const rsvd_b200_config c = to_c(*this);
    return rsvd_b200_sketch_width(&c, m, n);
}

double RsvdResult::residual_fro(const DenseMatrix& a) const {
    const std::size_t k = factors.sigma.size();
    if (factors.u.rows() != a.rows() || factors.v.rows() != a.cols())
        throw DimensionError("residual_fro: factors for " +
                             shape_str(factors.u.rows(), factors.v.rows()) + " against input " +
                             shape_str(a.rows(), a.cols()));
    double out = 0.0;
    check(rsvd_b200_residual_fro(handle(), a.data().data(), a.rows(), a.cols(),
                                 factors.u.data().data(), factors.sigma.data(),
                                 factors.v.data().data(), k, &out));
    return out;
}

DenseMatrix gaussian_matrix(GaussianSampler& sampler, std::size_t rows, std::size_t cols) {
    DenseMatrix out(rows, cols);
    detail::SamplerAccess::draw(sampler, rows * cols,
                                [&](std::uint64_t counter, int has_cached, double cached) {
                                    check(rsvd_b200_gaussian_stream(
                                        handle(), sampler.seed(), counter, has_cached, cached,
                                        rows, cols, out.data().data()));
                                });
    return out;
}

DenseMatrix sketch(const DenseMatrix& a, std::size_t s, GaussianSampler& sampler) {
    const std::size_t md = std::min(a.rows(), a.cols());
    if (s < 1 || s > md)
        throw ArgumentError("sketch width " + std::to_string(s) + " outside [1, " +
                            std::to_string(md) + "] for a " + shape_str(a.rows(), a.cols()) +
                            " input");
    DenseMatrix y(a.rows(), s);
    detail::SamplerAccess::draw(sampler, a.cols() * s,
                                [&](std::uint64_t counter, int has_cached, double cached) {
                                    check(rsvd_b200_sketch_stream(
                                        handle(), a.data().data(), a.rows(), a.cols(), s,
                                        sampler.seed(), counter, has_cached, cached,
                                        y.data().data()));
                                });
    return y;
}

DenseMatrix power_iterate(const DenseMatrix& a, const DenseMatrix& y0, std::size_t q) {
    if (y0.rows() != a.rows())
        throw DimensionError("power_iterate: y0 has " + std::to_string(y0.rows()) +
                             " rows, a has " + std::to_string(a.rows()));
    DenseMatrix w(y0.rows(), y0.cols());
    check(rsvd_b200_power_iterate(handle(), a.data().data(), a.rows(), a.cols(),
                                  y0.data().data(), y0.cols(), q, w.data().data()));
    return w;
}

QrFactors householder_qr(const DenseMatrix& a) {
    DenseMatrix q(a.rows(), a.cols()), r(a.cols(), a.cols());
    check(rsvd_b200_householder_qr(handle(), a.data().data(), a.rows(), a.cols(),
                                   q.data().data(), r.data().data()));
    return {std::move(q), std::move(r)};
}

DenseMatrix range_basis(const DenseMatrix& y) {
    std::vector<double> q(y.size());
    std::size_t cols = 0;
    check(rsvd_b200_range_basis(handle(), y.data().data(), y.rows(), y.cols(), q.data(), &cols));
    q.resize(y.rows() * cols);
    return DenseMatrix(y.rows(), cols, std::move(q));
}

RsvdResult project_and_solve(const DenseMatrix& a, const DenseMatrix& qbasis, std::size_t k) {
    if (qbasis.rows() != a.rows())
        throw DimensionError("project_and_solve: basis has " + std::to_string(qbasis.rows()) +
                             " rows, a has " + std::to_string(a.rows()));
    if (k < 1 || k > qbasis.cols())
        throw ArgumentError("rank k=" + std::to_string(k) + " exceeds the basis width " +
                            std::to_string(qbasis.cols()));
    DenseMatrix u(a.rows(), k), v(a.cols(), k);
    std::vector<double> sigma(k);
    std::size_t sw = 0;
    check(rsvd_b200_project_and_solve(handle(), a.data().data(), a.rows(), a.cols(),
                                      qbasis.data().data(), qbasis.cols(), k, u.data().data(),
                                      sigma.data(), v.data().data(), &sw));
    return RsvdResult{SvdFactors{std::move(u), std::move(sigma), std::move(v)}, sw};
}

RsvdResult randomized_ksvd(const DenseMatrix& a, const RsvdConfig& cfg) {
    const rsvd_b200_config c = to_c(cfg);
    const std::size_t k = cfg.k;
    if (k < 1 || k > std::min(a.rows(), a.cols())) {
        check(rsvd_b200_randomized_ksvd(handle(), a.data().data(), a.rows(), a.cols(), &c,
                                        nullptr, nullptr, nullptr, nullptr));
    }
    DenseMatrix u(a.rows(), k), v(a.cols(), k);
    std::vector<double> sigma(k);
    std::size_t sw = 0;
    check(rsvd_b200_randomized_ksvd(handle(), a.data().data(), a.rows(), a.cols(), &c,
                                    u.data().data(), sigma.data(), v.data().data(), &sw));
    return RsvdResult{SvdFactors{std::move(u), std::move(sigma), std::move(v)}, sw};
}

std::vector<double> singular_values_only(const DenseMatrix& a, const RsvdConfig& cfg) {
    const rsvd_b200_config c = to_c(cfg);
    std::vector<double> sigma(std::max<std::size_t>(cfg.k, 1));
    check(rsvd_b200_singular_values_only(handle(), a.data().data(), a.rows(), a.cols(), &c,
                                         sigma.data()));
    sigma.resize(cfg.k);
    return sigma;
}

// ------------------------------------------------------------------ PCA (pca.cpp)
namespace pca {

std::pair<DenseMatrix, std::vector<double>> center_columns(const DenseMatrix& x) {
    const std::size_t n = x.rows(), d = x.cols();
    if (n < 2) throw ArgumentError("center_columns needs at least 2 rows, got " + std::to_string(n));
    std::vector<double> mean(d, 0.0);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < d; ++j) mean[j] += x(i, j);
    for (double& m : mean) m /= static_cast<double>(n);
    DenseMatrix centered(n, d);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < d; ++j) centered(i, j) = x(i, j) - mean[j];
    return {std::move(centered), std::move(mean)};
}

PcaModel fit_pca(const DenseMatrix& x, std::size_t k, const RsvdConfig& cfg) {
    const rsvd_b200_config c = to_c(cfg);
    const std::size_t kk = std::max<std::size_t>(k, 1);
    std::vector<double> mean(x.cols()), var(kk), comp(x.cols() * kk);
    check(rsvd_b200_fit_pca(handle(), x.data().data(), x.rows(), x.cols(), k, &c, mean.data(),
                            comp.data(), var.data()));
    return PcaModel{std::move(mean), DenseMatrix(x.cols(), k, std::move(comp)), std::move(var)};
}

DenseMatrix transform(const PcaModel& model, const DenseMatrix& x) {
    const std::size_t d = model.components.rows(), k = model.components.cols();
    if (x.cols() != d)
        throw DimensionError("transform: data has " + std::to_string(x.cols()) +
                             " features, model has " + std::to_string(d));
    DenseMatrix out(x.rows(), k);
    check(rsvd_b200_pca_transform(handle(), x.data().data(), x.rows(), d, model.mean.data(),
                                  model.components.data().data(), k, out.data().data()));
    return out;
}

}  // namespace pca

}  // namespace randsvd
