// randsvd_b200 — the reference CLI's hot-path subcommands (cli.cpp:81-221, 251-306) on the
// B200 library, written against the C++ drop-in headers exactly as a reference caller
// would use them (include/randsvd/*.hpp):
//   randsvd_b200 rsvd in.dmat (--k K | --k-frac F) [--oversample P] [--power-q Q]
//                [--epsilon E] [--seed S] [--threads T] [--values-only] --out PFX
//   randsvd_b200 pca in.dmat --k K [--oversample P] [--power-q Q] [--seed S] --out PFX
// Outputs PFX.{u,sigma,v}.dmat (rsvd) / PFX.{components,variance,mean}.dmat (pca) and the
// reference's one-line stderr summary; the timer covers the solve only (cli.cpp:256-266).
// Exit codes as cli.cpp:367-385: usage 1, I/O 2, anything else 3. --threads is accepted
// and ignored (the GPU grid replaces the host thread budget).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <iostream>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "randsvd/dmat.hpp"
#include "randsvd/errors.hpp"
#include "randsvd/pca.hpp"
#include "randsvd/rsvd.hpp"

using namespace randsvd;

namespace {

std::string fmt3(double x) {
    std::ostringstream o;
    o.precision(3);
    o << std::fixed << x;
    return o.str();
}

DenseMatrix column_vector(const std::vector<double>& v) { return DenseMatrix(v.size(), 1, v); }

struct Args {
    std::string cmd, input, out;
    std::optional<std::size_t> k;
    std::optional<double> k_frac, epsilon;
    std::size_t oversample = 10, power_q = 2;
    std::uint64_t seed = 0;
    unsigned threads = 1;
    bool values_only = false;
};

Args parse(int argc, char** argv) {
    if (argc < 2) throw UsageError("expected a subcommand: rsvd | pca");
    Args a;
    a.cmd = argv[1];
    if (a.cmd != "rsvd" && a.cmd != "pca") throw UsageError("unknown subcommand " + a.cmd);
    for (int i = 2; i < argc; ++i) {
        const std::string f = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw UsageError(f + " needs a value");
            return argv[++i];
        };
        try {
            if (f == "--k") a.k = std::stoull(val());
            else if (f == "--k-frac") a.k_frac = std::stod(val());
            else if (f == "--oversample") a.oversample = std::stoull(val());
            else if (f == "--power-q") a.power_q = std::stoull(val());
            else if (f == "--epsilon") a.epsilon = std::stod(val());
            else if (f == "--seed") a.seed = std::stoull(val());
            else if (f == "--threads") a.threads = (unsigned)std::stoul(val());
            else if (f == "--out") a.out = val();
            else if (f == "--values-only" && a.cmd == "rsvd") a.values_only = true;
            else if (!f.empty() && f[0] == '-') throw UsageError("unknown option " + f);
            else if (a.input.empty()) a.input = f;
            else throw UsageError("unexpected argument " + f);
        } catch (const std::invalid_argument&) {
            throw UsageError("bad value for " + f);
        }
    }
    if (a.input.empty() || a.out.empty()) throw UsageError("input and --out are required");
    if (a.k && a.k_frac) throw UsageError("--k excludes --k-frac");
    if (!a.k && !a.k_frac) throw UsageError("--k or --k-frac is required");
    if (a.k && *a.k == 0) throw UsageError("--k must be positive");
    if (a.threads == 0) throw UsageError("--threads must be positive");
    return a;
}

RsvdConfig config(const Args& a, std::size_t cols) {
    RsvdConfig cfg;
    cfg.k = a.k ? *a.k : (std::size_t)std::ceil(*a.k_frac * (double)cols);  // cli.cpp:75-79
    cfg.oversample = a.oversample;
    cfg.power_q = a.power_q;
    cfg.seed = a.seed;
    if (a.epsilon) {
        cfg.epsilon = *a.epsilon;
        cfg.epsilon_mode = true;
    }
    return cfg;
}

double since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int run(const Args& a) {
    const DenseMatrix x = read_dmat(a.input);
    const RsvdConfig cfg = config(a, x.cols());
    if (a.cmd == "pca") {
        const auto t0 = std::chrono::steady_clock::now();
        const pca::PcaModel model = pca::fit_pca(x, cfg.k, cfg);
        const double wall = since(t0);
        write_dmat(a.out + ".components.dmat", model.components);
        write_dmat(a.out + ".variance.dmat", column_vector(model.explained_variance));
        write_dmat(a.out + ".mean.dmat", column_vector(model.mean));
        std::cerr << "pca: shape=" << x.rows() << "x" << x.cols() << " k=" << cfg.k
                  << " wall=" << fmt3(wall) << "s threads=" << a.threads << "\n";
        return 0;
    }
    std::size_t width = cfg.sketch_width(x.rows(), x.cols());
    std::string residual = "n/a";
    const auto t0 = std::chrono::steady_clock::now();
    double wall = 0.0;
    if (a.values_only) {
        const std::vector<double> sigma = singular_values_only(x, cfg);
        wall = since(t0);
        write_dmat(a.out + ".sigma.dmat", column_vector(sigma));
    } else {
        const RsvdResult res = randomized_ksvd(x, cfg);
        wall = since(t0);
        width = res.sketch_width;
        residual = fmt3(res.residual_fro(x));
        write_dmat(a.out + ".u.dmat", res.factors.u);
        write_dmat(a.out + ".sigma.dmat", column_vector(res.factors.sigma));
        write_dmat(a.out + ".v.dmat", res.factors.v);
    }
    std::cerr << "rsvd: shape=" << x.rows() << "x" << x.cols() << " k=" << cfg.k
              << " s=" << width << " q=" << cfg.power_q << " seed=" << cfg.seed
              << " residual=" << residual << " wall=" << fmt3(wall)
              << "s threads=" << a.threads << "\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return run(parse(argc, argv));
    } catch (const UsageError& e) {
        std::cerr << "usage error: " << e.what() << "\n";
        return 1;
    } catch (const IoError& e) {
        std::cerr << "io error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 3;
    }
}
