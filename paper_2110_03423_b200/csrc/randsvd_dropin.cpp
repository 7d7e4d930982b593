// C++ drop-in for the reference API (include/randsvd/*.hpp) over the C-ABI.
//
// A user of the reference's `randsvd::randomized_ksvd(const DenseMatrix&,
// const RsvdConfig&)` (rsvd.hpp:58) relinks against librsvd_b200.so and keeps
// the same calls, value types, layout and exception types. Each host thread
// lazily owns one rsvd_b200_handle on its selected device.
#include <cmath>
#include <cstdlib>
#include <memory>
#include <string>

#include "../../include/randsvd/pca.hpp"
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
        case RSVD_B200_CONVERGENCE_ERROR: throw ConvergenceError(msg, kSvdMaxSweeps);
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

double frobenius_norm(const DenseMatrix& a) {
    double acc = 0.0;
    for (double x : a.data()) acc += x * x;
    return std::sqrt(acc);
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
    if (sampler.counter() != 0)
        throw ArgumentError("gaussian_matrix on the device needs a fresh sampler (counter 0)");
    DenseMatrix out(rows, cols);
    check(rsvd_b200_gaussian_matrix(handle(), sampler.seed(), rows, cols, out.data().data()));
    sampler.advance(2 * ((rows * cols + 1) / 2));
    return out;
}

DenseMatrix sketch(const DenseMatrix& a, std::size_t s, GaussianSampler& sampler) {
    if (sampler.counter() != 0)
        throw ArgumentError("sketch on the device needs a fresh sampler (counter 0)");
    const std::size_t md = std::min(a.rows(), a.cols());
    if (s < 1 || s > md)
        throw ArgumentError("sketch width " + std::to_string(s) + " outside [1, " +
                            std::to_string(md) + "] for a " + shape_str(a.rows(), a.cols()) +
                            " input");
    DenseMatrix y(a.rows(), s);
    check(rsvd_b200_sketch(handle(), a.data().data(), a.rows(), a.cols(), s, sampler.seed(),
                           y.data().data()));
    sampler.advance(2 * ((a.cols() * s + 1) / 2));
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
