// Host-side orchestration of the B200 randomized k-SVD and its C-ABI
// (include/rsvd_b200.h). Every arithmetic stage runs in the sm_100a kernels of
// this directory; this file only sequences them on the handle's stream, owns the
// HBM workspace and maps failures to the reference's error contract.
//
// Algorithm 1 exactly as the reference sequences it (rsvd.cpp:126-134):
//   s      = sketch_width(m, n)                                   (rsvd.cpp:28-35)
//   Y0     = A * Omega                                            (rsvd.cpp:51-59)
//   W      = QR(Y0).q;  q x { Z = QR(A^T W).q ; W = QR(A Z).q }   (rsvd.cpp:61-73)
//   Q      = range_basis(W)                                       (rsvd.cpp:75-87)
//   B      = Q^T A; (U_B, sigma, V) = svd(B); U = Q U_B[:, :k]    (rsvd.cpp:89-109)
// with these B200 substitutions:
//   * every product is a TMA-fed FP64 tensor-core GEMM (gemm_f64.cu) reading A
//     in place (no transposed copy); split-K partials are reduced in fixed order.
//     For A with at least 2^26 elements the passes over A run as exact INT8 digit
//     products on tcgen05 (gemm_oz.cu, Ozaki scheme): on the optimistic path from A's
//     digit planes converted once per solve, on the robust rerun with in-kernel digits;
//     FP32 A runs every m-sized product as 3xTF32 on tcgen05 (gemm_tf32.cu);
//   * thin QR is CholeskyQR2 (Gram by the same GEMMs, s x s Cholesky in shared
//     memory, TRSM as a GEMM against R^-1), with a blocked Householder QR
//     (householder.cu, the reference's algorithm in compact-WY panels) as the
//     fallback when a Cholesky pivot signals an ill-conditioned input;
//   * the SVD of the s x n matrix B runs as CholeskyQR2 of B^T = Q_B R_B followed
//     by one-sided Jacobi on the s x s R_B (one CTA, a thread-block cluster, or a
//     cooperative block Jacobi by width; same rotation rule and thresholds as
//     svd.cpp), V = Q_B U_R, U_B = W_R, then the reference's sort and sign convention.
// range_basis inside the pipeline: power_iterate always returns orthonormal
// columns (Householder or CholeskyQR2 Q), whose R factor has |R_jj| = 1 + O(eps),
// so the drop rule |R_jj| <= 1e-13 ||W||_F (<= 1e-13 sqrt(s)) can never fire and
// Q(range_basis(W)) = W up to rounding; the pipeline therefore passes W through
// and sketch_width = s. The standalone rsvd_b200_range_basis implements the full
// rule (Householder R diagonal) for callers that pass arbitrary matrices.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/rsvd_b200.h"
#include "comm.h"
#include "kernels.h"

using namespace rsvdb200;

namespace {

thread_local std::string g_last_error;

struct Failure {
    rsvd_b200_status code;
    std::string msg;
};

[[noreturn]] void fail(rsvd_b200_status code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw Failure{code, buf};
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(RSVD_B200_CUDA_ERROR, "%s: %s", what, cudaGetErrorString(e));
}

template <typename F>
rsvd_b200_status guarded(F&& f) {
    try {
        f();
        return RSVD_B200_OK;
    } catch (const Failure& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return RSVD_B200_ALLOC_ERROR;
    }
}

long round_up(long x, long m) { return (x + m - 1) / m * m; }

// Padded sketch width: multiples of 16 up to 96 (128-row tiles, 4x2 warps),
// multiples of 32 up to 288 (64-row tiles, 2x4 warps).
int pad_np(long s) {
    if (s <= 96) return (int)round_up(std::max(1L, s), 16);
    if (s <= 288) return (int)round_up(s, 32);
    fail(RSVD_B200_ARGUMENT_ERROR, "sketch width %ld exceeds the supported maximum of 288", s);
}

// Split-K count so that tiles * splits fills whole waves of 148 SMs, with at least two
// k-tiles (of 32) per split.
int choose_splits(long tiles, long k_tiles) {
    if (k_tiles <= 1) return 1;
    if (tiles >= 2 * 148) {
        // many tiles: split only to fix a ragged last wave (C5: 512 tiles = 3.46 waves, 86 %
        // busy; 2 splits = 6.92 waves, 99 %); the slabs cost one extra pass over M x NP
        auto eff = [](long ctas) { return (double)ctas / (148.0 * ((ctas + 147) / 148)); };
        int best = 1;
        double best_eff = eff(tiles);
        for (int sp = 2; sp <= 4 && sp <= k_tiles / 64; ++sp)
            if (eff(sp * tiles) > best_eff + 0.03) {
                best_eff = eff(sp * tiles);
                best = sp;
            }
        return best;
    }
    const long cap = std::max(1L, k_tiles / 2);
    int best = 1;
    double best_eff = 0.0;
    for (int w = 1; w <= 16; ++w) {
        const long sp = std::min(cap, std::max(1L, std::lround(148.0 * w / (double)tiles)));
        const long ctas = sp * tiles;
        const double eff = (double)ctas / (148.0 * ((ctas + 147) / 148));
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = (int)sp;
        }
        // long contractions (>= 2048 k-tiles, where a CTA's fixed cost is small) search on to
        // ~99 % busy: the C2 A^T Q passes (32 column tiles) go from 9 splits (288 CTAs, 1.95
        // waves) to 23 (736 CTAs, 4.97 waves; 3.89 -> 3.82 ms); the extra slabs are 60 MB
        if (sp == cap || (eff > (k_tiles >= 2048 ? 0.985 : 0.93) && w >= 2)) break;
    }
    return best;
}

// Bumped by every workspace (re)allocation: a captured solve graph (SolveGraph) holds raw
// workspace pointers and is only replayed while the generation it was captured at is current.
std::atomic<unsigned long> g_ws_gen{0};

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void reserve(size_t b) {
        if (b <= bytes) return;
        g_ws_gen.fetch_add(1);
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        if (cudaMalloc(&p, b) != cudaSuccess)
            fail(RSVD_B200_ALLOC_ERROR, "cudaMalloc of %zu bytes failed", b);
        bytes = b;
    }
    double* d() const { return static_cast<double*>(p); }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

struct StageTimer {
    const char* name;
    cudaEvent_t start, stop;
};

// Everything a captured device-resident solve depends on besides the workspace generation.
struct GraphKey {
    const void* a = nullptr;
    long m = 0, n = 0, lda = 0;
    int s = 0, NP = 0;
    bool f32 = false;
    size_t k = 0, q = 0;
    uint64_t seed = 0;
    const void *u = nullptr, *sigma = nullptr, *v = nullptr;
    long ldu = 0, ldv = 0;
    int profiling = 0;
    unsigned long gen = 0;
    const void* comm = nullptr;  // sharded solves: the communicator the graph's all-reduces use
    int apass = 0;               // A-pass datapath (oz_mode: DMMA / emulated / stored digits)
    bool operator==(const GraphKey& o) const {
        return a == o.a && m == o.m && n == o.n && lda == o.lda && s == o.s && NP == o.NP &&
               f32 == o.f32 && k == o.k && q == o.q && seed == o.seed && u == o.u &&
               sigma == o.sigma && v == o.v && ldu == o.ldu && ldv == o.ldv &&
               profiling == o.profiling && gen == o.gen && comm == o.comm && apass == o.apass;
    }
};

}  // namespace

struct rsvd_b200_handle {
    int device = 0;
    cudaStream_t stream = nullptr;
    // host-buffer solves: A is uploaded in row chunks on copy_stream and the sketch GEMM
    // consumes each chunk as it lands (up_ev[c] recorded after chunk c)
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> up_ev;
    cudaEvent_t up_start = nullptr;
    long up_chunk_rows = 0, up_chunks = 0;
    bool up_active = false;
    // workspace
    DevBuf a_copy, a_t, xt, y, q, part, b, b2, qbt, vbuf, small, flags, u_out, v_out, sig_out,
        hh_work, hh_rows, synth_buf, omega_host_dev, jscratch, cwork, ubt;
    std::unique_ptr<Comm> comm;  // row-sharded solves (comm.h); null = single device
    DevBuf red_scratch;          // TSQR R stack
    DevBuf flag_red;             // the two flags of a sharded run, as doubles, all-reduced
    // the last shard layout that passed the collective check (comm, m_local, m_total, n, s)
    const void* shard_ok_comm = nullptr;
    long shard_ok[4] = {0, 0, 0, 0};
    DevBuf pca_ones, pca_sums, pca_mean, pca_comp;  // PCA (fit_pca / transform)
    DevBuf res_vs, res_part, res_u;                 // residual_fro
    // FP32 path (A stored in FP32, 3xTF32 tensor-core products): tall FP32 buffers
    // (each with its TF32 lo parts: the B operand of a 3xTF32 product needs both)
    DevBuf yf, qf, xtf, rtf, ubtf, af_copy, yf_lo, qf_lo, xtf_lo, rtf_lo, ubtf_lo, tf32_tmp;
    float* basis_f = nullptr;     // Q1 of the current basis in the FP32 path (yf or qf)
    float* basis_f_lo = nullptr;  // its lo parts
    long fallbacks = 0, reruns = 0;
    int last_sweeps = 0;
    bool force_robust = false;
    // the optimistic run's abort flag while one is in flight (else nullptr): the A-pass GEMMs
    // skip themselves once a Cholesky breakdown has doomed the run to a robust rerun
    const int* abort_ptr = nullptr;
    bool c_identity = true;  // the current basis Q = Q1 C has C = I
    double* basis = nullptr;  // Q1 of the current basis (h->y or h->q)
    bool gram_ready = false;  // slot kG holds Y^T Y of the last produced Y
    // host-buffer solves: the first power iteration's A^T Y0 split-K slabs were produced during
    // the chunked upload (sketch_dev); power_iterate_dev only reduces them
    bool aty_pending = false;
    int aty_splits = 0;
    long aty_slab = 0;
    DevBuf pre_part;  // the upload-time (A^T Y0)^T split-K slabs (FP64, or FP32 in the FP32 path)
    long upload_aty = 0;  // splits of the last solve's upload-time A^T Y0 (0: not used)
    DevBuf gpart;             // per-tile Gram partials of the fused epilogue
    // INT8-emulated FP64 passes (gemm_oz.cu): digit planes of the small operand, exponent
    // arrays (A rows, A columns, B columns, scratch) and the scan partials
    DevBuf oz_bdig, oz_ef, oz_part;
    DevBuf oz_adig;  // A's row-scaled digit planes (stored-digit passes)
    bool oz_stored = false;  // this run's passes after the sketch read A's stored digits
    long oz_passes = 0;  // passes over A of the last solve that ran on the INT8 tensor cores
    long oz_stored_passes = 0;  // of those, atx passes from A's stored digits
    int* flags_host = nullptr;
    StreamPos omega_pos;  // sampler state the next sketch's Omega continues (default: fresh)
    std::vector<double> omega_host;  // validation mode (n x s row-major)
    size_t omega_rows = 0, omega_cols = 0;
    int profiling = 0;  // 1: stage events, 2: + per-launch events on the A-pass GEMMs
    std::vector<StageTimer> timers;
    struct KernelEvent {
        const char* tag;
        double flops;
        cudaEvent_t start, stop;
    };
    std::vector<KernelEvent> kevents;
    struct KernelStat {
        long count = 0;
        double ms = 0.0, flops = 0.0;
    };
    std::vector<std::pair<std::string, KernelStat>> kstats;
    std::vector<std::pair<const char*, double>> last_profile;
    long launches = 0;
    // CUDA graphs of the optimistic device-resident pipeline (solve_tall): captured on the
    // first solve of a shape/config/buffer set and replayed while the key still matches,
    // so a repeated solve costs one graph launch instead of ~60-250 kernel launches with
    // their host-side tensor-map encodes. A few keys are kept (LRU) because callers that
    // allocate fresh outputs per solve alternate between buffer sets.
    struct SolveGraph {
        GraphKey key;
        cudaGraphExec_t exec = nullptr;
        long launches = 0;
        unsigned long used = 0;
        void reset() {
            if (exec) cudaGraphExecDestroy(exec);
            exec = nullptr;
        }
    };
    static constexpr int kMaxGraphs = 4;
    SolveGraph graphs[kMaxGraphs];
    unsigned long graph_clock = 0;
    void reset_graphs() {
        for (auto& g : graphs) g.reset();
    }
    bool use_graphs = true;
    long graph_replays = 0;

    // ----------------------------------------------------------------- timing
    void mark(const char* name) {
        if (!profiling) return;
        StageTimer t{name, nullptr, nullptr};
        cudaEventCreate(&t.start);
        cudaEventCreate(&t.stop);
        if (!timers.empty()) cudaEventRecord(timers.back().stop, stream);
        cudaEventRecord(t.start, stream);
        timers.push_back(t);
    }
    void kernel_begin(const char* tag, double flops) {
        if (profiling < 2 || !tag) return;
        KernelEvent e{tag, flops, nullptr, nullptr};
        cudaEventCreate(&e.start);
        cudaEventCreate(&e.stop);
        cudaEventRecord(e.start, stream);
        kevents.push_back(e);
    }
    void kernel_end(const char* tag) {
        if (profiling < 2 || !tag) return;
        cudaEventRecord(kevents.back().stop, stream);
    }
    void finish_kernel_events() {
        if (kevents.empty()) return;
        cudaEventSynchronize(kevents.back().stop);
        for (auto& e : kevents) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e.start, e.stop);
            auto it = std::find_if(kstats.begin(), kstats.end(),
                                   [&](auto& x) { return x.first == e.tag; });
            if (it == kstats.end()) {
                kstats.emplace_back(e.tag, KernelStat{});
                it = kstats.end() - 1;
            }
            it->second.count += 1;
            it->second.ms += ms;
            it->second.flops += e.flops;
            cudaEventDestroy(e.start);
            cudaEventDestroy(e.stop);
        }
        kevents.clear();
    }
    void finish_timers() {
        finish_kernel_events();
        if (!profiling || timers.empty()) return;
        cudaEventRecord(timers.back().stop, stream);
        cudaEventSynchronize(timers.back().stop);
        last_profile.clear();
        for (auto& t : timers) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, t.start, t.stop);
            last_profile.emplace_back(t.name, (double)ms);
            cudaEventDestroy(t.start);
            cudaEventDestroy(t.stop);
        }
        timers.clear();
    }

    static double trace_us() {  // host clock for the trace lines
        using namespace std::chrono;
        static const auto t0 = steady_clock::now();
        return duration<double, std::micro>(steady_clock::now() - t0).count();
    }
    void sync() {
        if (trace) fprintf(stderr, "[rsvd_b200] %12.1f us -- sync\n", trace_us());
        ck(cudaStreamSynchronize(stream), "stream synchronize");
        if (trace) fprintf(stderr, "[rsvd_b200] %12.1f us -- synced\n", trace_us());
    }
    int read_flag(int idx) {
        sync();
        return flags_host[idx];
    }
    void launched(cudaError_t e, const char* what, int count = 1) {
        ck(e, what);
        launches += count;
        if (trace) {
            fprintf(stderr, "[rsvd_b200] %12.1f us %s\n", trace_us(), what);
            if (trace > 1) ck(cudaStreamSynchronize(stream), what);
        }
    }
    // RSVD_B200_TRACE=1 logs every launch, =2 also synchronises after each one
    int trace = 0;
};

namespace {

// Slots in h->flags (device int array, mirrored in pinned flags_host).
enum {
    kFlagNonfinite = 0,  // NaN/Inf seen in A (fused into the first pass)
    kFlagAbort = 1,      // a Cholesky broke down on the optimistic path -> rerun robustly
    kFlagChol = 2,       // status of the last Cholesky (robust path)
    kFlagCholScratch = 3,
    kFlagJacobi = 4,     // sweeps, or -1 if the Jacobi SVD did not converge
    kFlagComplete = 5,   // 1 if the orthonormal completion failed
    kNumFlags = 8
};

// Small s-by-s scratch layout inside h->small (each NP x NP doubles).
enum { kG = 0, kR1 = 1, kR1iT = 2, kR2 = 3, kR2iT = 4, kRB = 5, kUR = 6, kWR = 7, kTmp = 8,
       kSig = 9, kC = 10, kX = 11, kB1 = 12, kB2 = 13, kB3 = 14, kB4 = 15, kB5 = 16,
       kNumSmall = 17 };

struct Plan {
    long m, n;   // tall problem: m >= n (m = this rank's rows when sharded)
    long lda;    // leading dimension of A on device
    int s, NP;   // sketch width and padded width
    long ldn;    // leading dimension of n-length rows (Xt, B, Q_B^T): round_up(n, 2)
    bool sharded = false;  // A row-sharded over h->comm: sums over m are all-reduced
    // FP32 path: A (af, lda floats) in FP32; every product with an m-dimension runs on the
    // tcgen05 3xTF32 kernels with tall operands m x NPf in FP32 (NPf = s rounded up to 16);
    // the s x s and n x s side stays FP64 at width NP.
    bool f32 = false;
    const float* af = nullptr;
    int NPf = 0;
    long ldnf = 0;  // leading dimension of FP32 n-length rows (16-byte multiple)
};

// One pipeline run. `robust`: synchronise after every Cholesky and take the
// Householder fallback on breakdown. Otherwise (the optimistic path) nothing
// synchronises: a breakdown only raises kFlagAbort, later kernels carry on (their
// results are discarded), and the host reruns the solve robustly after the single
// synchronisation at the end.
struct Ctx {
    rsvd_b200_handle* h;
    Plan p;
    bool robust;
    int* flags;
    double* slot(int i) const { return h->small.d() + (size_t)i * p.NP * p.NP; }
    // Sum over the row shards (no-op on a single device): the Gram of a tall QR and the
    // n x s partials of A^T Q / Q^T A are the only cross-rank data of Algorithm 1.
    void allreduce(double* buf, size_t count) const {
        if (!p.sharded) return;
        const std::string err = h->comm->allreduce_sum(buf, count, h->stream);
        if (!err.empty()) fail(RSVD_B200_NCCL_ERROR, "%s", err.c_str());
        h->launches += 1;
    }
};

double* small_slot(rsvd_b200_handle* h, const Plan& p, int slot) {
    return h->small.d() + (size_t)slot * p.NP * p.NP;
}

void download_flags(rsvd_b200_handle* h) {
    ck(cudaMemcpyAsync(h->flags_host, h->flags.p, kNumFlags * sizeof(int), cudaMemcpyDeviceToHost,
                       h->stream),
       "flag download");
}

long ax_tiles(long M, int NP) { return (M + (NP <= 96 ? 127 : 63)) / (NP <= 96 ? 128 : 64); }

// ------------------------------------------------------------ GEMM wrappers
// Y (M x NP) = A (M x K) * X where Xt (NP x K) holds X^T. If `gram_out` is given and the
// launch can fuse it (NP <= 96, no split-K), the Gram Y^T Y is produced by the GEMM's
// epilogue and reduced into gram_out (NP x NP); returns whether that happened.
// cols > 0: Xt's rows >= cols are zero (the sketch width s of an A-pass); lets the kernel
// drop the MMA padding of s (GemmAx::cols).
bool gemm_ax(rsvd_b200_handle* h, const double* A, long M, long K, long lda, const double* Xt,
             long ldx, int NP, double* Y, long ldy, int* flag = nullptr,
             const char* tag = nullptr, double flops = 0.0, double* gram_out = nullptr,
             int cols = 0) {
    GemmAx g{A, M, K, lda, Xt, ldx, NP, Y, ldy};
    g.flag = flag;
    g.cols = cols;
    g.abort = h->abort_ptr;
    const int splits = choose_splits(ax_tiles(M, NP), (K + 31) / 32);
    if (splits == 1) {
        const bool fuse = gram_out && NP <= 96;
        const long tiles = ax_tiles(M, NP);
        if (fuse) {
            if (h->gpart.bytes < (size_t)tiles * NP * NP * sizeof(double))
                fail(RSVD_B200_ALLOC_ERROR, "Gram workspace too small");
            g.gram = h->gpart.d();
        }
        h->kernel_begin(tag, flops);
        h->launched(launch_gemm_ax(g, h->stream), "gemm_ax");
        h->kernel_end(tag);
        if (fuse)
            h->launched(launch_reduce_partials(h->gpart.d(), (long)NP * NP, (int)tiles, gram_out,
                                               (long)NP * NP, h->stream),
                        "reduce_partials");
        return fuse;
    }
    const long slab = M * ldy;
    if (h->part.bytes < (size_t)splits * slab * sizeof(double))
        fail(RSVD_B200_ALLOC_ERROR, "split-K workspace too small");
    g.Y = h->part.d();
    g.splits = splits;
    g.split_stride = slab;
    h->kernel_begin(tag, flops);
    h->launched(launch_gemm_ax(g, h->stream), "gemm_ax(split)");
    h->kernel_end(tag);
    h->launched(launch_reduce_partials(h->part.d(), slab, splits, Y, slab, h->stream),
                "reduce_partials");
    return false;
}

// Y = A X as gemm_ax, over row chunks of A whose upload (solve_host) is still in flight:
// chunk c's launch waits for its copy event, so the sketch runs behind the H2D copy and
// only the last chunk's GEMM is exposed. Chunks are whole 128/64-row tiles, so the fused
// Gram partials line up with the unchunked launch's.
// aty_ldz > 0: also produce the split-K slabs of (A^T Y)^T (the first power iteration's
// A-pass, Y = this sketch, ld aty_ldz) into h->part, each chunk's share right after the chunk
// is sketched. The splits are exactly gemm_atx's (choose_splits, same k-tile ranges, same
// kernel), so the slabs — and the reduced result — are bit-identical to gemm_atx's.
bool gemm_ax_chunked(rsvd_b200_handle* h, const double* A, long M, long K, long lda,
                     const double* Xt, long ldx, int NP, double* Y, long ldy, int* flag,
                     const char* tag, double flops, double* gram_out, int cols,
                     long aty_ldz = 0) {
    int aty_splits = 0;
    long per_rows = 0, slab = 0;
    if (aty_ldz > 0) {
        aty_splits = choose_splits(ax_tiles(K, NP), (M + 31) / 32);
        per_rows = (((M + 31) / 32 + aty_splits - 1) / aty_splits) * 32;
        slab = (long)NP * aty_ldz;
        if (aty_splits < 2)
            aty_splits = 0;  // gemm_atx would not split: leave it to the pass
        else  // own buffer: the tall QR's Gram (when not fused) reuses h->part first
            h->pre_part.reserve((size_t)aty_splits * slab * sizeof(double));
    }
    // the rows [r0, r1) just sketched: each split overlapping them advances by that segment
    // (atx `accumulate` continues the split's partial sum, so a split built from several
    // segments accumulates in exactly the order of one launch over its whole range)
    auto launch_aty = [&](long r0, long r1) {
        for (int j = (int)(r0 / per_rows); j < aty_splits && j * per_rows < r1; ++j) {
            const long s0 = j * per_rows, s1 = std::min(M, s0 + per_rows);
            const long a = std::max(s0, r0), b = std::min(s1, r1);
            if (a >= b) continue;
            GemmAtx g{A + a * lda, b - a, K, lda, Y + a * ldy, ldy, NP,
                      h->pre_part.d() + j * slab, aty_ldz, true};
            g.accumulate = a > s0;
            g.cols = cols;  // the same (tail) kernel as the device pass's gemm_atx
            h->launched(launch_gemm_atx(g, h->stream), "gemm_atx(upload segment)");
        }
    };
    const bool fuse = gram_out && NP <= 96;
    if (fuse && h->gpart.bytes < (size_t)ax_tiles(M, NP) * NP * NP * sizeof(double))
        fail(RSVD_B200_ALLOC_ERROR, "Gram workspace too small");
    long tile0 = 0;
    h->kernel_begin(tag, flops);
    for (long c = 0; c < h->up_chunks; ++c) {
        const long r0 = c * h->up_chunk_rows, r1 = std::min(M, r0 + h->up_chunk_rows);
        ck(cudaStreamWaitEvent(h->stream, h->up_ev[c], 0), "wait for chunk upload");
        GemmAx g{A + r0 * lda, r1 - r0, K, lda, Xt, ldx, NP, Y + r0 * ldy, ldy};
        g.flag = flag;
        g.cols = cols;
        if (fuse) g.gram = h->gpart.d() + tile0 * NP * NP;
        h->launched(launch_gemm_ax(g, h->stream), "gemm_ax(chunk)");
        tile0 += ax_tiles(r1 - r0, NP);
        if (aty_splits > 0) launch_aty(r0, r1);
    }
    h->kernel_end(tag);
    for (int j = 0; j < aty_splits; ++j)  // splits past the last row (rounding): zero slabs
        if (j * per_rows >= M)
            h->launched(launch_fill(h->pre_part.d() + j * slab, slab, 0.0, h->stream), "fill");
    if (aty_splits > 0) {
        h->aty_pending = true;
        h->aty_splits = aty_splits;
        h->aty_slab = slab;
        h->upload_aty = aty_splits;
    }
    if (fuse)
        h->launched(launch_reduce_partials(h->gpart.d(), (long)NP * NP, (int)tile0, gram_out,
                                           (long)NP * NP, h->stream),
                    "reduce_partials");
    return fuse;
}

// Z = A^T W.  A (K x N, lda), W (K x NP, ldw); out_t: Z^T (NP x N, ldz) else Z (N x NP, ldz).
// cols > 0: W's columns >= cols are zero (GemmAtx::cols).
void gemm_atx(rsvd_b200_handle* h, const double* A, long K, long N, long lda, const double* W,
              long ldw, int NP, double* Z, long ldz, bool out_t, const char* tag = nullptr,
              double flops = 0.0, int cols = 0) {
    GemmAtx g{A, K, N, lda, W, ldw, NP, Z, ldz, out_t};
    g.abort = h->abort_ptr;
    g.cols = cols;
    const int splits = choose_splits(ax_tiles(N, NP), (K + 31) / 32);
    if (splits == 1) {
        h->kernel_begin(tag, flops);
        h->launched(launch_gemm_atx(g, h->stream), "gemm_atx");
        h->kernel_end(tag);
        return;
    }
    const long slab = out_t ? (long)NP * ldz : N * ldz;
    if (h->part.bytes < (size_t)splits * slab * sizeof(double))
        fail(RSVD_B200_ALLOC_ERROR, "split-K workspace too small");
    g.Z = h->part.d();
    g.splits = splits;
    g.split_stride = slab;
    h->kernel_begin(tag, flops);
    h->launched(launch_gemm_atx(g, h->stream), "gemm_atx(split)");
    h->kernel_end(tag);
    h->launched(launch_reduce_partials(h->part.d(), slab, splits, Z, slab, h->stream),
                "reduce_partials");
}

// 3xTF32 tensor-core product (gemm_tf32.cu) with split-K over K for FP64 outputs when the
// output tiles alone would not fill the GPU (1 CTA per SM); slabs reduced in fixed order.
// Slab: the out_t rows NP x ldo, else M x ldo.
// The tensor core's FP32 accumulation is biased (it shrinks long sums by ~1e-8 per added
// term), so an FP64-output product never accumulates more than kTf32Chain K-values in
// TMEM: longer contractions are split and the slabs summed in FP64. This keeps the
// relative bias of e.g. B = Q^T A (K = m = 200000) at ~1e-5 instead of ~2e-4.
constexpr long kTf32Chain = 2048;

int tf32_splits(long M, long K) {
    const long tiles = (M + 127) / 128;
    const long k_tiles = (K + 15) / 16;  // tf32 k-tiles of 16
    const int by_chain = (int)((K + kTf32Chain - 1) / kTf32Chain);
    return std::max(choose_splits(tiles, k_tiles), by_chain);
}

void gemm_tf32(rsvd_b200_handle* h, GemmTf32 g, const char* tag = nullptr, double flops = 0.0) {
    g.abort = h->abort_ptr;
    const int splits = g.out64 ? tf32_splits(g.M, g.K) : 1;
    if (splits == 1) {
        h->kernel_begin(tag, flops);
        h->launched(launch_gemm_tf32(g, h->stream), "gemm_tf32");
        h->kernel_end(tag);
        return;
    }
    // the slabs hold the TMEM accumulators, which are FP32: stored as FP32 (exactly), summed
    // in FP64 in a fixed order — half the slab traffic of FP64 slabs, the same result
    // (row-major FP32 stores are float4: FP64 slabs unless every row stays 16-byte aligned)
    const long slab = g.out_t ? (long)g.NP * g.ldo : g.M * g.ldo;
    const bool f32_slabs = g.out_t || (g.ldo % 4 == 0 && slab % 4 == 0);
    if (h->part.bytes < (size_t)splits * slab * (f32_slabs ? sizeof(float) : sizeof(double)))
        fail(RSVD_B200_ALLOC_ERROR, "split-K workspace too small");
    double* out = static_cast<double*>(g.out);
    g.out = h->part.p;
    g.out64 = !f32_slabs;
    g.splits = splits;
    g.split_stride = slab;
    h->kernel_begin(tag, flops);
    h->launched(launch_gemm_tf32(g, h->stream), "gemm_tf32(split)");
    h->kernel_end(tag);
    if (f32_slabs)
        h->launched(launch_reduce_partials_f32(static_cast<const float*>(h->part.p), slab, splits,
                                               out, slab, h->stream),
                    "reduce_partials");
    else
        h->launched(launch_reduce_partials(h->part.d(), slab, splits, out, slab, h->stream),
                    "reduce_partials");
}

// ---------------------------------------------- INT8-emulated FP64 A-passes (gemm_oz.cu)
// The passes over A of an FP64 solve run on the INT8 tensor cores (Ozaki scheme) when A holds
// at least 2^26 elements (below, the scale scan and digit preparation cost more than the
// DMMA passes save, and the FP64 DMMA kernels keep products such as sketch(I) = Omega
// bit-exact). RSVD_B200_GEMM=dmma / =oz forces either path (tests, comparisons).
bool oz_on(const Plan& p) {
    const char* e = getenv("RSVD_B200_GEMM");  // read per solve: tests switch it
    const int mode = (e && std::string(e) == "dmma") ? 0 : (e && std::string(e) == "oz") ? 2 : 1;
    if (mode == 0 || p.f32 || p.NP < 16 || p.NP > 256) return false;
    return mode == 2 || (double)p.m * (double)p.n >= (double)(1L << 26);
}

// Stored digits (default for the emulated path; RSVD_B200_OZ_STORED=0 disables): one fused
// pass over A (oz_scan_convert, per row chunk as it lands) yields the row scales, the NaN/Inf
// check and A's row-scaled digits in the two tiled layouts of gemm_ozd, and every pass over A
// then reads digits instead of FP64 — no conversion inside the GEMMs, none duplicated by the
// column-chunk CTAs (C2: 1.81 / 1.59 ms per ax / atx pass against 2.61 / 2.64 in-kernel; the
// atx passes fold A's row scales into W). Needs oz_ax_bytes + oz_atx_bytes (1.75 x the FP64 A)
// of HBM; without the room the passes stay in-kernel. Accuracy of the atx passes: normwise
// FP64 per column of W' (the row scales folded in), against per column of A in-kernel — so the
// robust rerun (inputs that break CholeskyQR) keeps the in-kernel digits.
bool oz_stored_fits(rsvd_b200_handle* h, const Plan& p) {
    const char* e = getenv("RSVD_B200_OZ_STORED");
    if (e && atoi(e) == 0) return false;
    const size_t need = oz_ax_bytes(p.m, p.n) + oz_atx_bytes(p.m, p.n);
    if (need <= h->oz_adig.bytes) return true;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return false;
    return need + (size_t)(2ull << 30) <= free_b + h->oz_adig.bytes;
}

// 0: DMMA passes, 1: emulated with in-kernel digits, 2: emulated with stored digits
int oz_mode(rsvd_b200_handle* h, const Plan& p) {
    if (!oz_on(p)) return 0;
    return oz_stored_fits(h, p) ? 2 : 1;
}

long oz_tiles(long N, int NP) {
    int nch, nf;
    oz_chunks(NP, &nch, &nf);
    return ((N + 127) / 128) * nch;
}

// split-K of an oz pass: every split within the int32 accumulators' headroom; the atx shape
// (few output tiles, K = m) also splits to fill the waves like choose_splits. The ax shape
// never splits for occupancy, so a row chunk of it (chunked upload) runs exactly the tiles
// of the whole pass.
int oz_splits(long N, int NP, long K, bool fill) {
    const long kt = (K + 31) / 32;
    const int need = (int)((kt + kOzMaxKTiles - 1) / kOzMaxKTiles);
    return fill ? std::max(choose_splits(oz_tiles(N, NP), kt), need) : need;
}

// Largest split-K slab set any GEMM of a plan needs.
size_t partial_doubles(const Plan& p) {
    const long NP = p.NP;
    size_t need = 0;
    auto atx = [&](long K, long N, long ldz, bool out_t) {
        const int sp = choose_splits(ax_tiles(N, p.NP), (K + 31) / 32);
        if (sp > 1) need = std::max(need, (size_t)sp * (out_t ? NP * ldz : N * ldz));
    };
    auto ax = [&](long M, long K, long ldy) {
        const int sp = choose_splits(ax_tiles(M, p.NP), (K + 31) / 32);
        if (sp > 1) need = std::max(need, (size_t)sp * M * ldy);
    };
    atx(p.m, p.n, p.ldn, true);  // A-pass (A^T W)^T, Q^T A
    if (oz_on(p)) {
        const int sa = oz_splits(p.n, NP, p.m, true);
        if (sa > 1) need = std::max(need, (size_t)sa * NP * p.ldn);
        const int sx = oz_splits(p.m, NP, p.n, false);
        if (sx > 1) need = std::max(need, (size_t)sx * p.m * NP);
    }
    atx(p.m, NP, NP, false);     // tall Gram
    atx(NP, p.n, p.ldn, true);   // wide TRSM / C^T correction
    atx(NP, p.n, NP, false);     // V = Q_B U_R
    ax(p.m, p.n, NP);            // A-pass A Z
    ax(p.m, NP, NP);             // tall TRSM, back-projection
    ax(NP, p.n, NP);             // wide Gram
    if (p.f32) {  // 3xTF32: A-pass (A^T Q)^T (NPf x ldn slabs) and the tall Gram (NPf x NP)
        const int sp1 = tf32_splits(p.n, p.m);
        if (sp1 > 1) need = std::max(need, (size_t)sp1 * p.NPf * p.ldn);
        const int sp2 = tf32_splits(p.NPf, p.m);
        if (sp2 > 1) need = std::max(need, (size_t)sp2 * p.NPf * NP);
        const int sp3 = tf32_splits(p.m, p.NPf);  // U = Q (C U_B) (FP64 out, K = NPf)
        if (sp3 > 1) need = std::max(need, (size_t)sp3 * p.m * p.NPf);
    }
    return std::max<size_t>(need, 1);
}

constexpr double kCholTol = 1e-12;  // pivot / max diag: beyond cond ~1e6 use Householder
// FP32 path: Grams carry ~1e-5 relative error (TF32 tensor-core accumulation), so
// CholeskyQR is only trusted up to cond(Y) ~ 300; beyond, the FP64 Householder fallback.
constexpr double kCholTolF32 = 1e-5;

// G = R^T R (R upper, diag > 0) and R^-T of the s x s Gram in slot g_slot. Widths that
// fit one CTA's shared memory run cholesky_kernel directly; wider ones (s > ~150, e.g.
// s = 272) are factored as a 2 x 2 block Cholesky from two in-smem factorisations:
//   R11 = chol(G11), R12 = R11^-T G12, S = G22 - R12^T R12, R22 = chol(S),
//   R^-T = [[R11^-T, 0], [-R22^-T R12^T R11^-T, R22^-T]],
// with both pivot tests judged against the largest diagonal of the whole G.
void cholesky(const Ctx& c, int g_slot, int r_slot, int rit_slot) {
    rsvd_b200_handle* h = c.h;
    cudaStream_t st = h->stream;
    const int NP = c.p.NP, s = c.p.s;
    int* status = c.flags + (c.robust ? kFlagChol : kFlagCholScratch);
    int* abort = c.robust ? nullptr : c.flags + kFlagAbort;
    const double* G = c.slot(g_slot);
    double* R = c.slot(r_slot);
    double* RiT = c.slot(rit_slot);
    static const int chol_max = getenv("RSVD_B200_CHOL_MAX") ? atoi(getenv("RSVD_B200_CHOL_MAX"))
                                                             : cholesky_max_width();
    const double tol = c.p.f32 ? kCholTolF32 : kCholTol;
    if (s <= std::min(chol_max, cholesky_max_width())) {
        h->launched(launch_cholesky(G, NP, s, NP, R, RiT, status, abort, tol, st), "cholesky");
        return;
    }
    // 2 x 2 blocks: the two Cholesky CTAs write their factors straight into R / R^-T (the first
    // one the whole NP x NP region, zeros included; the second only its s2 x s2 block)
    const int s1 = (s + 1) / 2, s2 = s - s1;
    double* S = c.slot(kB3);
    double* R22 = R + (size_t)s1 * NP + s1;
    double* R22iT = RiT + (size_t)s1 * NP + s1;
    h->launched(launch_cholesky(G, NP, s1, NP, R, RiT, status, abort, tol, st, G, NP, s, false),
                "cholesky");
    // R12 = R11^-T G12 -> R[0:s1, s1:s]
    h->launched(launch_small_gemm(s1, s2, s1, 1.0, RiT, NP, false, G + s1, NP, false, 0.0,
                                  nullptr, 0, R + s1, NP, st),
                "small_gemm");
    // S = G22 - R12^T R12
    h->launched(launch_small_gemm(s2, s2, s1, -1.0, R + s1, NP, true, R + s1, NP, false, 1.0,
                                  G + (size_t)s1 * NP + s1, NP, S, NP, st),
                "small_gemm");
    h->launched(launch_cholesky(S, NP, s2, NP, R22, R22iT, status, abort, tol, st, G, NP, s, true,
                                s2),
                "cholesky");
    // T = R12^T R11^-T (s2 x s1) into S; RiT[s1:, 0:s1] = -R22^-T T
    h->launched(launch_small_gemm(s2, s1, s1, 1.0, R + s1, NP, true, RiT, NP, false, 0.0,
                                  nullptr, 0, S, NP, st),
                "small_gemm");
    h->launched(launch_small_gemm(s2, s1, s2, -1.0, R22iT, NP, false, S, NP, false, 0.0, nullptr,
                                  0, RiT + (size_t)s1 * NP, NP, st),
                "small_gemm");
}

bool chol_broke(const Ctx& c) {
    if (!c.robust) return false;
    download_flags(c.h);
    return c.h->read_flag(kFlagChol) != 0;
}

void set_identity(const Ctx& c, int slot) {
    std::vector<double> eye((size_t)c.p.NP * c.p.NP, 0.0);
    for (int i = 0; i < c.p.NP; ++i) eye[(size_t)i * c.p.NP + i] = 1.0;
    ck(cudaMemcpyAsync(c.slot(slot), eye.data(), eye.size() * sizeof(double),
                       cudaMemcpyHostToDevice, c.h->stream),
       "identity upload");
    c.h->sync();  // eye is a stack temporary
}

// Householder fallback of a row-sharded tall QR (TSQR): Y_g = Q_g R_g locally, the
// ranks' R_g (NP x NP blocks, zero padded) are stacked by a sum all-reduce of a
// world*NP x NP buffer in which each rank fills its own block, the stack is factored
// again (replicated, identical on every rank) as Q_s R, and Q_g <- Q_g Q_s[block g].
// R keeps diag >= 0 (the reference's sign fix, qr.cpp:86-93), so for a full-rank Y the
// result is the unique thin QR the unsharded Householder QR produces.
void tsqr(const Ctx& c, double* Y, long M, double* Qout) {
    rsvd_b200_handle* h = c.h;
    const int NP = c.p.NP, s = c.p.s;
    const int world = h->comm->world, rank = h->comm->rank;
    if (M < s)
        fail(RSVD_B200_DIMENSION_ERROR,
             "TSQR fallback needs at least s=%d rows per shard, rank %d has %ld", s, rank, M);
    const long stack_rows = (long)world * NP;
    const size_t stack = (size_t)stack_rows * NP;
    h->red_scratch.reserve((stack * 2 + (size_t)NP * NP) * sizeof(double));
    double* R = h->red_scratch.d();
    double* Qs = R + stack;
    double* Xt = Qs + stack;
    h->hh_work.reserve(householder_work_doubles(std::max(M, stack_rows), NP) * sizeof(double));
    h->launched(launch_fill(R, (long)stack, 0.0, h->stream), "fill");
    h->launched(launch_householder_qr(Y, M, s, NP, Qout, NP, R + (size_t)rank * NP * NP, NP,
                                      h->hh_work.d(), h->stream),
                "householder_qr");
    c.allreduce(R, stack);
    h->launched(launch_householder_qr(R, stack_rows, s, NP, Qs, NP, c.slot(kRB), NP,
                                      h->hh_work.d(), h->stream),
                "householder_qr");
    // Q_g (M x NP) <- Q_g * Q_s[rank block] (NP x NP); ax takes the transposed block
    h->launched(launch_transpose(Qs + (size_t)rank * NP * NP, NP, NP, NP, Xt, NP, h->stream),
                "transpose");
    gemm_ax(h, Qout, M, NP, NP, Xt, NP, NP, Qout, NP);  // in place: K = NP, one k-pass per CTA
}

// ---------------------------------------------------------------- tall QR
// Thin QR of Y (M x NP, ld NP, columns >= s zero) by CholeskyQR, returned in factored
// form Q = Q1 * C with Q1 at h->basis and C in slot kC (h->c_identity when C = I):
//  * passes = 1 (intermediate power-iteration QRs): Q1 = Y itself and C = R1^-1; no
//    pass over Y at all. The next product only needs span(Y R1^-1) and applies R1^-1
//    to its small output (A^T Y R1^-1); the final QR re-orthonormalises.
//  * passes = 2 (CholeskyQR2, the final basis): Q1 = Y R1^-1 is formed by a GEMM whose
//    epilogue also produces G2 = Q1^T Q1, and C = R2^-1 is again left to the
//    consumers (Q = Q1 R2^-1 without the second tall TRSM).
// `gram_ready`: slot kG already holds Y^T Y (fused into the GEMM that produced Y).
// `materialize` forms Q explicitly in `Q1out` (step-function API).
// The Householder fallback (robust path) writes Q itself to Q1out, C = I, R in kRB.
// Returns true if the fallback ran.
bool tall_qr(const Ctx& c, double* Y, long M, double* Q1out, int passes, bool materialize,
             bool gram_ready) {
    rsvd_b200_handle* h = c.h;
    const int NP = c.p.NP, s = c.p.s;
    h->c_identity = true;
    h->basis = Q1out;
    if (!gram_ready) gemm_atx(h, Y, M, NP, NP, Y, NP, NP, c.slot(kG), NP, false);  // G1 = Y^T Y
    c.allreduce(c.slot(kG), (size_t)NP * NP);  // sharded: G1 = sum_g Y_g^T Y_g
    cholesky(c, kG, kR1, kR1iT);
    if (!chol_broke(c)) {
        if (passes == 1 && !materialize) {
            h->basis = Y;
            h->launched(launch_transpose(c.slot(kR1iT), NP, NP, NP, c.slot(kC), NP, h->stream),
                        "transpose");  // C = R1^-1
            h->c_identity = false;
            h->launched(launch_copy2d(c.slot(kR1), NP, c.slot(kRB), NP, NP, NP, h->stream),
                        "copy2d");
            return false;
        }
        // Q1 = Y R1^-1 with G2 = Q1^T Q1 from the same kernel's epilogue
        const bool g2 = gemm_ax(h, Y, M, NP, NP, c.slot(kR1iT), NP, NP, Q1out, NP, nullptr, nullptr,
                                0.0, passes == 2 ? c.slot(kG) : nullptr);
        if (passes == 1) {
            h->launched(launch_copy2d(c.slot(kR1), NP, c.slot(kRB), NP, NP, NP, h->stream),
                        "copy2d");
            return false;
        }
        if (!g2) gemm_atx(h, Q1out, M, NP, NP, Q1out, NP, NP, c.slot(kG), NP, false);
        c.allreduce(c.slot(kG), (size_t)NP * NP);
        cholesky(c, kG, kR2, kR2iT);
        if (!chol_broke(c)) {
            if (materialize) {  // in place: each ax CTA reads exactly the rows it writes
                gemm_ax(h, Q1out, M, NP, NP, c.slot(kR2iT), NP, NP, Q1out, NP);
            } else {
                h->launched(launch_transpose(c.slot(kR2iT), NP, NP, NP, c.slot(kC), NP, h->stream),
                            "transpose");  // C = R2^-1
                h->c_identity = false;
            }
            h->launched(launch_small_matmul(c.slot(kR2), c.slot(kR1), s, NP, c.slot(kRB), false,
                                            h->stream),
                        "small_matmul");  // R = R2 R1
            return false;
        }
    }
    if (c.p.sharded) {
        tsqr(c, Y, M, Q1out);
        h->basis = Q1out;
        h->c_identity = true;
        h->fallbacks += 1;
        return true;
    }
    h->hh_work.reserve(householder_work_doubles(M, NP) * sizeof(double));
    h->launched(launch_householder_qr(Y, M, s, NP, Q1out, NP, c.slot(kRB), NP, h->hh_work.d(),
                                      h->stream),
                "householder_qr");
    h->basis = Q1out;
    h->c_identity = true;
    h->fallbacks += 1;
    return true;
}

// Tall QR of the FP32 path: Y = h->yf (M x NPf, FP32), same factored-basis contract as
// tall_qr (basis h->basis_f = Q1, C in slot kC). Grams G = Y^T Y by the MN-major 3xTF32
// kernel (FP64 out), Q1 = Y R1^-1 by the K-major one. The Householder fallback (and TSQR
// when sharded) runs in FP64 on a converted copy of Y.
bool tall_qr_f32(const Ctx& c, long M, int passes) {
    rsvd_b200_handle* h = c.h;
    cudaStream_t st = h->stream;
    const int NP = c.p.NP, NPf = c.p.NPf, s = c.p.s;
    float* Y = static_cast<float*>(h->yf.p);
    float* Ylo = static_cast<float*>(h->yf_lo.p);
    float* Q1 = static_cast<float*>(h->qf.p);
    float* Q1lo = static_cast<float*>(h->qf_lo.p);
    auto gram = [&](const float* X, const float* Xlo) {
        GemmTf32 g{X, (long)NPf, M, (long)NPf, X, (long)NPf, NPf, c.slot(kG), (long)NP};
        g.Blo = Xlo;
        g.mn = true;
        g.upper = true;  // the Cholesky reads the upper triangle only
        gemm_tf32(h, g);
        c.allreduce(c.slot(kG), (size_t)NP * NP);
    };
    h->c_identity = true;
    h->basis_f = Y;
    h->basis_f_lo = Ylo;
    gram(Y, Ylo);
    cholesky(c, kG, kR1, kR1iT);
    if (!chol_broke(c)) {
        if (passes == 1) {
            h->launched(launch_transpose(c.slot(kR1iT), NP, NP, NP, c.slot(kC), NP, st),
                        "transpose");  // C = R1^-1
            h->c_identity = false;
            h->launched(launch_copy2d(c.slot(kR1), NP, c.slot(kRB), NP, NP, NP, st), "copy2d");
            return false;
        }
        // Q1 = Y R1^-1 (K-major 3xTF32 with Bt = R1^-T in FP32), then its Gram
        h->launched(launch_cvt_f64_f32(c.slot(kR1iT), NP, NPf, NPf, s, s,
                                       static_cast<float*>(h->rtf.p), NPf, st,
                                       static_cast<float*>(h->rtf_lo.p)),
                    "cvt");
        GemmTf32 t{Y, M, (long)NPf, (long)NPf, static_cast<float*>(h->rtf.p), (long)NPf, NPf,
                   Q1, (long)NPf};
        t.Blo = static_cast<float*>(h->rtf_lo.p);
        t.out_lo = Q1lo;
        t.out64 = false;
        gemm_tf32(h, t);
        gram(Q1, Q1lo);
        cholesky(c, kG, kR2, kR2iT);
        if (!chol_broke(c)) {
            h->launched(launch_transpose(c.slot(kR2iT), NP, NP, NP, c.slot(kC), NP, st),
                        "transpose");  // C = R2^-1
            h->c_identity = false;
            h->basis_f = Q1;
            h->basis_f_lo = Q1lo;
            h->launched(launch_small_matmul(c.slot(kR2), c.slot(kR1), s, NP, c.slot(kRB), false, st),
                        "small_matmul");  // R = R2 R1
            return false;
        }
    }
    // FP64 fallback on a converted copy of Y
    h->y.reserve((size_t)M * NP * sizeof(double));
    h->q.reserve((size_t)M * NP * sizeof(double));
    h->launched(launch_fill(h->y.d(), M * NP, 0.0, st), "fill");
    h->launched(launch_cvt_f32_f64(Y, NPf, M, NPf, h->y.d(), NP, st), "cvt");
    if (c.p.sharded) {
        tsqr(c, h->y.d(), M, h->q.d());
    } else {
        h->hh_work.reserve(householder_work_doubles(M, NP) * sizeof(double));
        h->launched(launch_householder_qr(h->y.d(), M, s, NP, h->q.d(), NP, c.slot(kRB), NP,
                                          h->hh_work.d(), st),
                    "householder_qr");
    }
    h->launched(launch_cvt_f64_f32(h->q.d(), NP, M, NPf, M, s, Q1, NPf, st, Q1lo), "cvt");
    h->basis_f = Q1;
    h->basis_f_lo = Q1lo;
    h->c_identity = true;
    h->fallbacks += 1;
    return true;
}

// Thin QR of an N x s matrix held transposed, Zt (NP x N, ld ldz) -> Qt (NP x N, ld ldz),
// R (NP x NP) into slot r_slot. CholeskyQR with `passes` passes (both triangular solves
// applied: these matrices are only n x s); Householder fallback on the robust path.
bool wide_qr(const Ctx& c, const double* Zt, long N, long ldz, double* Qt, int r_slot,
             int passes) {
    rsvd_b200_handle* h = c.h;
    const int NP = c.p.NP, s = c.p.s;
    gemm_ax(h, Zt, NP, N, ldz, Zt, ldz, NP, c.slot(kG), NP);  // G = Zt Zt^T
    cholesky(c, kG, kR1, kR1iT);
    if (!chol_broke(c)) {
        h->launched(launch_transpose(c.slot(kR1iT), NP, NP, NP, c.slot(kTmp), NP, h->stream),
                    "transpose");
        gemm_atx(h, Zt, NP, N, ldz, c.slot(kTmp), NP, NP, Qt, ldz, true);  // Q1^T = R1^-T Zt
        if (passes == 1) {
            h->launched(launch_copy2d(c.slot(kR1), NP, c.slot(r_slot), NP, NP, NP, h->stream),
                        "copy2d");
            return false;
        }
        gemm_ax(h, Qt, NP, N, ldz, Qt, ldz, NP, c.slot(kG), NP);
        cholesky(c, kG, kR2, kR2iT);
        if (!chol_broke(c)) {
            h->launched(launch_transpose(c.slot(kR2iT), NP, NP, NP, c.slot(kTmp), NP, h->stream),
                        "transpose");
            // in place: each atx CTA reads exactly the Qt columns it writes (K = NP rows)
            gemm_atx(h, Qt, NP, N, ldz, c.slot(kTmp), NP, NP, Qt, ldz, true);
            h->launched(launch_small_matmul(c.slot(kR2), c.slot(kR1), s, NP, c.slot(r_slot), false,
                                            h->stream),
                        "small_matmul");
            return false;
        }
    }
    // row-major copies of Z and Q in handle buffers (a per-call allocation would free and
    // re-allocate, i.e. synchronise the device and invalidate the captured solve graphs)
    h->hh_rows.reserve(2 * (size_t)N * NP * sizeof(double));
    double* zrow = h->hh_rows.d();
    double* qrow = zrow + (size_t)N * NP;
    h->launched(launch_transpose(Zt, NP, N, ldz, zrow, NP, h->stream), "transpose");
    h->hh_work.reserve(householder_work_doubles(N, NP) * sizeof(double));
    h->launched(launch_householder_qr(zrow, N, s, NP, qrow, NP, c.slot(r_slot), NP,
                                      h->hh_work.d(), h->stream),
                "householder_qr");
    h->launched(launch_transpose(qrow, N, NP, NP, Qt, ldz, h->stream), "transpose");
    h->fallbacks += 1;
    return true;
}

// (NP x N) = C^T * in: the deferred R2^-1 of a factored basis Q = Q1 C applied to
// (A^T Q1)^T or Q1^T A. Returns `in` unchanged when C = I.
const double* apply_ct(const Ctx& c, const double* in, double* out) {
    if (c.h->c_identity) return in;
    gemm_atx(c.h, in, c.p.NP, c.p.n, c.p.ldn, c.slot(kC), c.p.NP, c.p.NP, out, c.p.ldn, true);
    return out;
}

Plan make_plan(long m, long n, long lda, long s) {
    Plan p;
    p.m = m;
    p.n = n;
    p.lda = lda;
    p.s = (int)s;
    p.NP = pad_np(s);
    p.ldn = round_up(n, 2);
    return p;
}

Ctx begin_run(rsvd_b200_handle* h, const Plan& p, bool robust) {
    const int NP = p.NP;
    h->xt.reserve((size_t)NP * p.ldn * sizeof(double));
    if (p.f32) {
        for (DevBuf* b : {&h->yf, &h->qf, &h->yf_lo, &h->qf_lo})
            b->reserve((size_t)p.m * p.NPf * sizeof(float));
        h->xtf.reserve((size_t)p.NPf * p.ldnf * sizeof(float));
        h->xtf_lo.reserve((size_t)p.NPf * p.ldnf * sizeof(float));
        h->rtf.reserve((size_t)p.NPf * p.NPf * sizeof(float));
        h->rtf_lo.reserve((size_t)p.NPf * p.NPf * sizeof(float));
    } else {
        h->y.reserve((size_t)p.m * NP * sizeof(double));
        h->q.reserve((size_t)p.m * NP * sizeof(double));
    }
    h->b.reserve((size_t)NP * p.ldn * sizeof(double));
    h->b2.reserve((size_t)NP * p.ldn * sizeof(double));
    h->qbt.reserve((size_t)NP * p.ldn * sizeof(double));
    h->vbuf.reserve((size_t)p.n * NP * sizeof(double));
    h->small.reserve((size_t)kNumSmall * NP * NP * sizeof(double));
    h->part.reserve(partial_doubles(p) * sizeof(double));
    if (NP <= 96 && !p.f32) h->gpart.reserve((size_t)ax_tiles(p.m, NP) * NP * NP * sizeof(double));
    h->jscratch.reserve(std::max<size_t>(1, jacobi_global_scratch_doubles(p.s)) * sizeof(double));
    h->cwork.reserve(complete_basis_work_doubles(p.n) * sizeof(double));
    h->oz_passes = 0;
    h->oz_stored_passes = 0;
    h->oz_stored = false;
    if (oz_on(p)) {
        h->oz_ef.reserve((size_t)(p.m + p.n + 2 * NP + 8) * sizeof(int));
        h->oz_bdig.reserve(std::max(oz_digits_bytes(NP, p.n), oz_digits_bytes(NP, p.m)));
        h->oz_part.reserve(oz_scan_part_ints(p.m, p.n) * sizeof(int));
        // optimistic path only: the robust rerun (inputs that break CholeskyQR, i.e. strongly
        // graded spectra) keeps the in-kernel digits, whose per-column scales of A hold the
        // small singular values' relative accuracy better (tools/probe/stored_accuracy.py:
        // 5.4e-11 against 1.8e-10 at sigma ratio 2.5e-8)
        if (!robust && oz_mode(h, p) == 2) {
            h->oz_adig.reserve(oz_ax_bytes(p.m, p.n) + oz_atx_bytes(p.m, p.n));
            h->oz_stored = true;
        }
    }
    ck(cudaMemsetAsync(h->flags.p, 0, kNumFlags * sizeof(int), h->stream), "memset flags");
    h->aty_pending = false;
    h->upload_aty = 0;
    if (p.f32)  // the 3xTF32 A-pass writes rows < NPf of (A^T Q)^T / Q^T A; pad rows stay 0
        ck(cudaMemsetAsync(h->b.p, 0, (size_t)NP * p.ldn * sizeof(double), h->stream), "memset b");
    h->trace = getenv("RSVD_B200_TRACE") ? atoi(getenv("RSVD_B200_TRACE")) : 0;
    if (p.sharded) h->flag_red.reserve(2 * sizeof(double));
    h->abort_ptr = robust ? nullptr : static_cast<int*>(h->flags.p) + kFlagAbort;
    return Ctx{h, p, robust, static_cast<int*>(h->flags.p)};
}

// oz scales of A (row maxima for the ax passes, column maxima for the atx passes) and the
// NaN/Inf scan of validate (rsvd.cpp:144): rows [r0, r0 + rows) of A, the first chunk
// resetting the column maxima.
int* oz_row_ef(const Ctx& c) { return static_cast<int*>(c.h->oz_ef.p); }
int* oz_col_ef(const Ctx& c) { return oz_row_ef(c) + c.p.m; }
int* oz_b_ef(const Ctx& c) { return oz_col_ef(c) + c.p.n; }

void oz_scan(const Ctx& c, const double* A, long r0, long rows, bool first, bool check) {
    rsvd_b200_handle* h = c.h;
    h->launched(launch_oz_scan(A + r0 * c.p.lda, rows, c.p.n, c.p.lda, oz_row_ef(c) + r0,
                               oz_col_ef(c), static_cast<int*>(h->oz_part.p),
                               check ? c.flags + kFlagNonfinite : nullptr, h->stream, !first),
                "oz_scan");
}

// Digits of the n-side operand Xt (NP x ldn; rows >= s zero) for the ax passes.
void oz_digits_xt(const Ctx& c, const double* Xt) {
    int nch, nf;  // the stored-digit GEMM reads the planes tiled per column chunk
    oz_chunks(c.p.NP, &nch, &nf);
    c.h->launched(launch_oz_digits_rows(Xt, c.p.ldn, c.p.NP, c.p.s, c.p.n,
                                        static_cast<uint8_t*>(c.h->oz_bdig.p), oz_b_ef(c),
                                        c.h->stream, c.h->oz_stored ? nf : 0),
                  "oz_digits_rows");
}

// A's stored digits (oz_adig): the ax tiles, then the atx blocks of gemm_ozd
uint8_t* oz_dig_ax(const Ctx& c) { return static_cast<uint8_t*>(c.h->oz_adig.p); }
uint8_t* oz_dig_atx(const Ctx& c) { return oz_dig_ax(c) + oz_ax_bytes(c.p.m, c.p.n); }

// the side stream (copy_stream: host uploads) and `events` chunk events on it
void ensure_side_stream(rsvd_b200_handle* h, long events) {
    if (!h->copy_stream) {
        ck(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking), "stream create");
        ck(cudaEventCreateWithFlags(&h->up_start, cudaEventDisableTiming), "event create");
    }
    while ((long)h->up_ev.size() < events) {
        cudaEvent_t e;
        ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
        h->up_ev.push_back(e);
    }
}

// Y[r0 : r0 + rows] (NP wide) = A[r0 : r0 + rows] X from the stored ax tiles (r0 % 128 == 0),
// Xt's digits prepared tiled (oz_digits_xt).
void ozd_ax(const Ctx& c, long r0, long rows, double* Y, const char* tag, double flops) {
    rsvd_b200_handle* h = c.h;
    const Plan& p = c.p;
    GemmOzd g;
    g.a_inner = (p.n + 31) / 32;
    g.adig = oz_dig_ax(c) + (size_t)(r0 / 128) * g.a_inner * oz_ax_bytes(128, 32);
    g.M = rows, g.K = p.n, g.a_ef = oz_row_ef(c) + r0;
    g.bdig = static_cast<const uint8_t*>(h->oz_bdig.p), g.b_ef = oz_b_ef(c), g.NP = p.NP;
    g.abort = h->abort_ptr;
    const int splits = oz_splits(rows, p.NP, p.n, false);
    if (r0 == 0) {
        h->oz_passes += 1;
        h->oz_stored_passes += 1;
    }
    h->kernel_begin(tag, flops);
    if (splits == 1) {
        g.out = Y + r0 * p.NP, g.ldo = p.NP;
        h->launched(launch_gemm_ozd(g, h->stream), "gemm_ozd");
        h->kernel_end(tag);
        return;
    }
    const long slab = rows * p.NP;
    if (h->part.bytes < (size_t)splits * slab * sizeof(double))
        fail(RSVD_B200_ALLOC_ERROR, "split-K workspace too small");
    g.out = h->part.d(), g.ldo = p.NP, g.splits = splits, g.split_stride = slab;
    h->launched(launch_gemm_ozd(g, h->stream), "gemm_ozd(split)");
    h->kernel_end(tag);
    h->launched(launch_reduce_partials(h->part.d(), slab, splits, Y + r0 * p.NP, slab, h->stream),
                "reduce_partials");
}

// Y (rows x NP) = A[r0 : r0 + rows] X with the digits of Xt already prepared.
void oz_ax(const Ctx& c, const double* A, long r0, long rows, double* Y, const char* tag,
           double flops) {
    rsvd_b200_handle* h = c.h;
    const Plan& p = c.p;
    GemmOz g;
    g.A = A + r0 * p.lda, g.M = rows, g.K = p.n, g.lda = p.lda;
    g.a_ef = oz_row_ef(c) + r0;
    g.bdig = static_cast<const uint8_t*>(h->oz_bdig.p), g.ldb = oz_ldb(p.n), g.b_ef = oz_b_ef(c);
    g.NP = p.NP;
    g.abort = h->abort_ptr;
    const int splits = oz_splits(rows, p.NP, p.n, false);
    if (r0 == 0) h->oz_passes += 1;
    h->kernel_begin(tag, flops);
    if (splits == 1) {
        g.out = Y + r0 * p.NP, g.ldo = p.NP;
        h->launched(launch_gemm_oz(g, h->stream), "gemm_oz");
        h->kernel_end(tag);
        return;
    }
    const long slab = rows * p.NP;
    if (h->part.bytes < (size_t)splits * slab * sizeof(double))
        fail(RSVD_B200_ALLOC_ERROR, "split-K workspace too small");
    g.out = h->part.d(), g.ldo = p.NP, g.splits = splits, g.split_stride = slab;
    h->launched(launch_gemm_oz(g, h->stream), "gemm_oz(split)");
    h->kernel_end(tag);
    h->launched(launch_reduce_partials(h->part.d(), slab, splits, Y + r0 * p.NP, slab, h->stream),
                "reduce_partials");
}

// Zt (NP x ldn) = (A^T W)^T, W (m x NP, columns >= s zero).
void oz_atx(const Ctx& c, const double* A, const double* W, double* Zt, const char* tag,
            double flops) {
    rsvd_b200_handle* h = c.h;
    const Plan& p = c.p;
    int* colmax = oz_b_ef(c) + p.NP;
    if (h->oz_stored) {  // W' = diag(2^(E_row - 53)) W digitised per column, A's stored digits
        int nch, nf;
        oz_chunks(p.NP, &nch, &nf);
        h->launched(launch_oz_digits_cols(W, p.NP, p.NP, p.s, p.m,
                                          static_cast<uint8_t*>(h->oz_bdig.p), oz_b_ef(c),
                                          colmax, h->stream, oz_row_ef(c), nf),
                    "oz_digits_cols");
        GemmOzd g;
        g.mn = true;
        g.adig = oz_dig_atx(c), g.a_inner = (p.n + 127) / 128;
        g.M = p.n, g.K = p.m, g.a_ef = oz_row_ef(c);
        g.bdig = static_cast<const uint8_t*>(h->oz_bdig.p), g.b_ef = oz_b_ef(c), g.NP = p.NP;
        g.out_t = true;
        g.abort = h->abort_ptr;
        const int splits = oz_splits(p.n, p.NP, p.m, true);
        h->oz_passes += 1;
        h->oz_stored_passes += 1;
        h->kernel_begin(tag, flops);
        if (splits == 1) {
            g.out = Zt, g.ldo = p.ldn;
            h->launched(launch_gemm_ozd(g, h->stream), "gemm_ozd");
            h->kernel_end(tag);
            return;
        }
        const long slab = (long)p.NP * p.ldn;
        if (h->part.bytes < (size_t)splits * slab * sizeof(double))
            fail(RSVD_B200_ALLOC_ERROR, "split-K workspace too small");
        g.out = h->part.d(), g.ldo = p.ldn, g.splits = splits, g.split_stride = slab;
        h->launched(launch_gemm_ozd(g, h->stream), "gemm_ozd(split)");
        h->kernel_end(tag);
        h->launched(launch_reduce_partials(h->part.d(), slab, splits, Zt, slab, h->stream),
                    "reduce_partials");
        return;
    }
    h->launched(launch_oz_digits_cols(W, p.NP, p.NP, p.s, p.m,
                                      static_cast<uint8_t*>(h->oz_bdig.p), oz_b_ef(c), colmax,
                                      h->stream),
                "oz_digits_cols");
    GemmOz g;
    g.mn = true;
    g.A = A, g.M = p.n, g.K = p.m, g.lda = p.lda;
    g.a_ef = oz_col_ef(c);
    g.bdig = static_cast<const uint8_t*>(h->oz_bdig.p), g.ldb = oz_ldb(p.m), g.b_ef = oz_b_ef(c);
    g.NP = p.NP;
    g.out_t = true;
    g.abort = h->abort_ptr;
    const int splits = oz_splits(p.n, p.NP, p.m, true);
    h->oz_passes += 1;
    h->kernel_begin(tag, flops);
    if (splits == 1) {
        g.out = Zt, g.ldo = p.ldn;
        h->launched(launch_gemm_oz(g, h->stream), "gemm_oz");
        h->kernel_end(tag);
        return;
    }
    const long slab = (long)p.NP * p.ldn;
    if (h->part.bytes < (size_t)splits * slab * sizeof(double))
        fail(RSVD_B200_ALLOC_ERROR, "split-K workspace too small");
    g.out = h->part.d(), g.ldo = p.ldn, g.splits = splits, g.split_stride = slab;
    h->launched(launch_gemm_oz(g, h->stream), "gemm_oz(split)");
    h->kernel_end(tag);
    h->launched(launch_reduce_partials(h->part.d(), slab, splits, Zt, slab, h->stream),
                "reduce_partials");
}

// FP32 path: the n-side operand of the next A-pass, Xt (NP x ldn, FP64) -> xtf (NPf x ldnf)
void xt_to_f32(const Ctx& c) {
    const Plan& p = c.p;
    c.h->launched(launch_cvt_f64_f32(c.h->xt.d(), p.ldn, p.NPf, p.n, p.s, p.n,
                                     static_cast<float*>(c.h->xtf.p), p.ldnf, c.h->stream,
                                     static_cast<float*>(c.h->xtf_lo.p)),
                  "cvt");
}

// FP32 path A-pass (A^T Q1)^T / Q1^T A into h->b (rows < NPf, FP64).
void atx_a_f32(const Ctx& c) {
    const Plan& p = c.p;
    GemmTf32 g{p.af, p.n, p.m, p.lda, c.h->basis_f, (long)p.NPf, p.NPf, c.h->b.p, p.ldn};
    g.Blo = c.h->basis_f_lo;
    g.mn = true;
    g.out_t = true;
    gemm_tf32(c.h, g, "gemm_A", 2.0 * p.m * p.n * p.s);
}

// ---- sketch (rsvd.cpp:51-59): h->y (m x NP) = A * Omega, Omega from the device
// generator or the validation-mode host Omega; `check` fuses the NaN/Inf scan of A
// (validate, rsvd.cpp:144) into this first pass over A.
// pre_aty: the solve continues with power iterations whose first A^T W reads W = Y0 in
// factored form (tall_qr with one pass) — a chunked upload then also produces its slabs.
void sketch_dev(const Ctx& c, const double* A, uint64_t seed, bool check, bool pre_aty = false) {
    rsvd_b200_handle* h = c.h;
    const Plan& p = c.p;
    cudaStream_t st = h->stream;
    const long n = p.n;
    const int s = p.s, NP = p.NP;
    h->mark("omega");
    if (!h->omega_host.empty()) {
        if (h->omega_rows != (size_t)n || h->omega_cols != (size_t)s)
            fail(RSVD_B200_DIMENSION_ERROR,
                 "validation Omega is %zux%zu, the solve needs %ldx%d", h->omega_rows,
                 h->omega_cols, n, s);
        h->omega_host_dev.reserve((size_t)n * s * sizeof(double));
        ck(cudaMemcpyAsync(h->omega_host_dev.p, h->omega_host.data(), (size_t)n * s * 8,
                           cudaMemcpyHostToDevice, st),
           "omega upload");
        h->launched(launch_fill(h->xt.d(), (long)NP * p.ldn, 0.0, st), "fill");
        h->launched(launch_transpose(h->omega_host_dev.d(), n, s, s, h->xt.d(), p.ldn, st),
                    "transpose");
    } else {
        h->launched(launch_omega(seed, n, s, NP, h->xt.d(), p.ldn, st, h->omega_pos), "omega");
    }
    h->mark("sketch_gemm");
    if (p.f32) {
        xt_to_f32(c);
        const bool chunked = h->up_active && p.af == h->a_copy.p;
        const long rows_per = chunked ? h->up_chunk_rows : p.m;
        const long chunks = chunked ? h->up_chunks : 1;
        h->kernel_begin("gemm_A", 2.0 * p.m * n * s);
        // pre: also the first power iteration's (A^T Y0)^T slabs, chunk by chunk, with
        // atx_a_f32's own split-K partition (whole splits per chunk), into h->pre_part
        bool pre = chunked && pre_aty;
        int pre_splits = 0;
        long pre_per = 0, pre_slab = 0;
        if (pre) {
            pre_splits = tf32_splits(p.n, p.m);
            pre_per = ((p.m + 15) / 16 + pre_splits - 1) / pre_splits;  // k-tiles per split
            pre_slab = (long)p.NPf * p.ldn;
            pre = pre_splits > 1 && rows_per % (pre_per * 16) == 0;
            if (pre) h->pre_part.reserve((size_t)pre_splits * pre_slab * sizeof(float));
        }
        for (long ci = 0; ci < chunks; ++ci) {  // chunks: the sketch consumes the upload
            const long r0 = ci * rows_per, rows = std::min(p.m - r0, rows_per);
            if (chunked)
                ck(cudaStreamWaitEvent(h->stream, h->up_ev[ci], 0), "wait for chunk upload");
            GemmTf32 g{p.af + r0 * p.lda, rows, n, p.lda, static_cast<float*>(h->xtf.p), p.ldnf,
                       p.NPf, static_cast<float*>(h->yf.p) + r0 * p.NPf, (long)p.NPf};
            g.Blo = static_cast<float*>(h->xtf_lo.p);
            g.out_lo = static_cast<float*>(h->yf_lo.p) + r0 * p.NPf;
            g.out64 = false;
            g.flag = check ? c.flags + kFlagNonfinite : nullptr;
            gemm_tf32(h, g);
            if (pre) {
                GemmTf32 a{p.af + r0 * p.lda, p.n, rows, p.lda,
                           static_cast<float*>(h->yf.p) + r0 * p.NPf, (long)p.NPf, p.NPf,
                           static_cast<float*>(h->pre_part.p) + (r0 / (pre_per * 16)) * pre_slab,
                           p.ldn};
                a.Blo = static_cast<float*>(h->yf_lo.p) + r0 * p.NPf;
                a.mn = true;
                a.out_t = true;
                a.out64 = false;
                a.k_per_split = (int)pre_per;
                a.split_stride = pre_slab;
                h->launched(launch_gemm_tf32(a, h->stream), "gemm_tf32(upload split)");
            }
        }
        h->kernel_end("gemm_A");
        if (pre) {
            // splits past the last row (ceil rounding of the partition) got no chunk: their
            // slabs must be zero, not stale, because the reduce sums all pre_splits of them
            const long written = ((p.m + 15) / 16 + pre_per - 1) / pre_per;
            if (written < pre_splits)
                ck(cudaMemsetAsync(static_cast<float*>(h->pre_part.p) + written * pre_slab, 0,
                                   (size_t)(pre_splits - written) * pre_slab * sizeof(float),
                                   h->stream),
                   "zero trailing upload slabs");
            h->aty_pending = true;
            h->aty_splits = pre_splits;
            h->aty_slab = pre_slab;
            h->upload_aty = pre_splits;
        }
        if (chunked) h->up_active = false;
        h->gram_ready = false;
        return;
    }
    if (oz_on(p)) {
        // scales + NaN/Inf scan and the sketch on the INT8 tensor cores; a chunked upload is
        // scanned and sketched chunk by chunk as it lands (row scales are chunk-local). The
        // Gram of Y0 is left to tall_qr (no fused epilogue); no upload-time A^T Y0 (its
        // column scales need all of A).
        oz_digits_xt(c, h->xt.d());
        const bool chunked = h->up_active && A == h->a_copy.d();
        const long rows_per = chunked ? h->up_chunk_rows : p.m;
        const long chunks = chunked ? h->up_chunks : 1;
        for (long ci = 0; ci < chunks; ++ci) {
            const long r0 = ci * rows_per, rows = std::min(p.m - r0, rows_per);
            if (chunked)
                ck(cudaStreamWaitEvent(h->stream, h->up_ev[ci], 0), "wait for chunk upload");
            if (h->oz_stored) {  // row scales, NaN check and both digit layouts
                h->kernel_begin("oz_convert", 0.0);
                if (p.n <= 4608) {  // one pass: the re-read of 4-row groups stays in L2
                    h->launched(launch_oz_scan_convert(A, r0, r0 + rows, p.m, p.n, p.lda,
                                                       oz_dig_ax(c), oz_dig_atx(c), oz_row_ef(c),
                                                       check ? c.flags + kFlagNonfinite : nullptr,
                                                       h->stream),
                                "oz_scan_convert");
                } else {  // wide rows (C3, C5): scan, then the streaming tile conversion
                    oz_scan(c, A, r0, rows, ci == 0, check);
                    h->launched(launch_oz_convert_tiles(A, r0, r0 + rows, p.m, p.n, p.lda,
                                                        oz_dig_ax(c), oz_dig_atx(c), oz_row_ef(c),
                                                        h->stream),
                                "oz_convert_tiles");
                }
                h->kernel_end("oz_convert");
                ozd_ax(c, r0, rows, h->y.d(), "gemm_A", 2.0 * rows * n * s);
            } else {
                oz_scan(c, A, r0, rows, ci == 0, check);
                oz_ax(c, A, r0, rows, h->y.d(), "gemm_A", 2.0 * rows * n * s);
            }
        }
        if (chunked) h->up_active = false;
        h->gram_ready = false;
        return;
    }
    if (h->up_active && A == h->a_copy.d()) {
        h->gram_ready = gemm_ax_chunked(h, A, p.m, n, p.lda, h->xt.d(), p.ldn, NP, h->y.d(), NP,
                                        check ? c.flags + kFlagNonfinite : nullptr, "gemm_A",
                                        2.0 * p.m * n * s, c.slot(kG), s, pre_aty ? p.ldn : 0);
        h->up_active = false;  // every chunk event has been waited on
        return;
    }
    h->gram_ready = gemm_ax(h, A, p.m, n, p.lda, h->xt.d(), p.ldn, NP, h->y.d(), NP,
                            check ? c.flags + kFlagNonfinite : nullptr, "gemm_A",
                            2.0 * p.m * n * s, c.slot(kG), s);
}

// ---- power_iterate (rsvd.cpp:61-73): h->y holds Y0; result W = Q1 C (h->q, slot kC).
void power_iterate_dev(const Ctx& c, const double* A, size_t q, bool materialize) {
    rsvd_b200_handle* h = c.h;
    const Plan& p = c.p;
    if (p.m < p.s)
        fail(RSVD_B200_DIMENSION_ERROR, "householder_qr needs rows >= cols, got %ldx%d", p.m, p.s);
    if (q > 0 && p.n < p.s)
        fail(RSVD_B200_DIMENSION_ERROR, "householder_qr needs rows >= cols, got %ldx%d", p.n, p.s);
    h->mark("qr_tall");
    if (p.f32) {
        tall_qr_f32(c, p.m, q == 0 ? 2 : 1);  // QR(Y0)
        for (size_t round = 0; round < q; ++round) {
            h->mark("power_atx");
            if (round == 0 && h->aty_pending && h->basis_f == h->yf.p) {
                // (A^T Y0)^T: its FP32 split-K slabs were produced during the chunked upload
                h->launched(launch_reduce_partials_f32(static_cast<const float*>(h->pre_part.p),
                                                       h->aty_slab, h->aty_splits, h->b.d(),
                                                       h->aty_slab, h->stream),
                            "reduce_partials");
            } else {
                atx_a_f32(c);  // (A^T Q1)^T
            }
            h->aty_pending = false;
            c.allreduce(h->b.d(), (size_t)p.NP * p.ldn);
            h->mark("qr_wide");
            const double* zt = apply_ct(c, h->b.d(), h->b2.d());
            wide_qr(c, zt, p.n, p.ldn, h->xt.d(), kRB, 1);  // Z^T (FP64)
            h->mark("power_ax");
            xt_to_f32(c);
            GemmTf32 g{p.af, p.m, p.n, p.lda, static_cast<float*>(h->xtf.p), p.ldnf, p.NPf,
                       h->yf.p, (long)p.NPf};
            g.Blo = static_cast<float*>(h->xtf_lo.p);
            g.out_lo = h->yf_lo.p;
            g.out64 = false;
            gemm_tf32(h, g, "gemm_A", 2.0 * p.m * p.n * p.s);  // Y = A Z
            h->mark("qr_tall");
            tall_qr_f32(c, p.m, round + 1 == q ? 2 : 1);
        }
        return;
    }
    tall_qr(c, h->y.d(), p.m, h->q.d(), q == 0 ? 2 : 1, materialize && q == 0,
            h->gram_ready);  // QR(Y0)
    for (size_t round = 0; round < q; ++round) {
        h->mark("power_atx");
        if (round == 0 && h->aty_pending && h->basis == h->y.d()) {
            // (A^T Y0)^T: its split-K slabs were produced during the chunked upload
            h->launched(launch_reduce_partials(h->pre_part.d(), h->aty_slab, h->aty_splits,
                                               h->b.d(), h->aty_slab, h->stream),
                        "reduce_partials");
        } else if (oz_on(p)) {
            oz_atx(c, A, h->basis, h->b.d(), "gemm_A", 2.0 * p.m * p.n * p.s);  // (A^T Q1)^T
        } else {
            gemm_atx(h, A, p.m, p.n, p.lda, h->basis, p.NP, p.NP, h->b.d(), p.ldn, true,
                     "gemm_A", 2.0 * p.m * p.n * p.s, p.s);  // (A^T Q1)^T
        }
        h->aty_pending = false;
        c.allreduce(h->b.d(), (size_t)p.NP * p.ldn);  // sharded: sum_g (A_g^T Q1_g)^T
        h->mark("qr_wide");
        const double* zt = apply_ct(c, h->b.d(), h->b2.d());  // (A^T W)^T, W = Q1 C
        wide_qr(c, zt, p.n, p.ldn, h->xt.d(), kRB, 1);  // Z = QR(A^T W).q, as Z^T
        h->mark("power_ax");
        if (oz_on(p)) {
            oz_digits_xt(c, h->xt.d());
            if (h->oz_stored)
                ozd_ax(c, 0, p.m, h->y.d(), "gemm_A", 2.0 * p.m * p.n * p.s);  // Y = A Z
            else
                oz_ax(c, A, 0, p.m, h->y.d(), "gemm_A", 2.0 * p.m * p.n * p.s);  // Y = A Z
            h->gram_ready = false;
        } else {
            h->gram_ready = gemm_ax(h, A, p.m, p.n, p.lda, h->xt.d(), p.ldn, p.NP, h->y.d(),
                                    p.NP, nullptr, "gemm_A", 2.0 * p.m * p.n * p.s, c.slot(kG),
                                    p.s);  // Y = A Z
        }
        h->mark("qr_tall");
        const bool last = round + 1 == q;
        tall_qr(c, h->y.d(), p.m, h->q.d(), last ? 2 : 1, materialize && last,
                h->gram_ready);  // W = QR(Y).q
    }
}

// ---- project_and_solve (rsvd.cpp:89-109) with basis Q = Q1 C (h->q, slot kC).
// Outputs (device): sigma (k), v (n x k, ldv) and u (m x k, ldu) unless null.
void project_and_solve_dev(const Ctx& c, const double* A, long k, double* u, long ldu,
                           double* sigma, double* v, long ldv) {
    rsvd_b200_handle* h = c.h;
    const Plan& p = c.p;
    cudaStream_t st = h->stream;
    const long m = p.m, n = p.n;
    const int s = p.s, NP = p.NP;
    if (n < s)
        fail(RSVD_B200_DIMENSION_ERROR,
             "project_and_solve: basis width %d exceeds the %ld columns of a", s, n);
    h->mark("project_atx");
    if (p.f32)
        atx_a_f32(c);  // Q1^T A
    else if (oz_on(p))
        oz_atx(c, A, h->basis, h->b.d(), "gemm_A", 2.0 * m * n * s);  // Q1^T A
    else
        gemm_atx(h, A, m, n, p.lda, h->basis, NP, NP, h->b.d(), p.ldn, true, "gemm_A",
                 2.0 * m * n * s, s);  // Q1^T A
    c.allreduce(h->b.d(), (size_t)NP * p.ldn);  // sharded: B = sum_g Q1_g^T A_g
    h->mark("small_svd");
    const double* bq = apply_ct(c, h->b.d(), h->b2.d());  // B = C^T Q1^T A = Q^T A (NP x n)
    wide_qr(c, bq, n, p.ldn, h->qbt.d(), kRB, 2);          // B^T = Q_B R_B
    double* UR = c.slot(kUR);
    double* WR = c.slot(kWR);
    double* sig = c.slot(kSig);
    h->launched(launch_jacobi_svd(c.slot(kRB), s, NP, sig, UR, WR, c.flags + kFlagJacobi,
                                  h->jscratch.d(), c.flags + kFlagAbort, st),
                "jacobi_svd");
    // V = Q_B U_R (n x NP): atx with A = Q_B^T (K = NP, N = n), W = U_R
    gemm_atx(h, h->qbt.d(), NP, n, p.ldn, UR, NP, NP, h->vbuf.d(), NP, false);
    // null columns of B's SVD (svd.cpp:221-234) get the reference's canonical completion;
    // the kernel decides on the device whether there are any
    h->launched(launch_complete_basis(h->vbuf.d(), n, NP, s, sig, std::max<long>(n, s),
                                      h->cwork.d(), c.flags + kFlagComplete, c.flags + kFlagAbort,
                                      st),
                "complete_basis");
    h->launched(launch_sign_fix(h->vbuf.d(), n, NP, s, WR, NP, st), "sign_fix");

    // outputs: sigma[:k], V[:, :k], U = Q U_B[:, :k] = Q1 (C U_B)[:, :k]
    ck(cudaMemcpyAsync(sigma, sig, k * sizeof(double), cudaMemcpyDeviceToDevice, st), "sigma");
    if (v) h->launched(launch_copy2d(h->vbuf.d(), NP, v, ldv, n, k, st), "copy2d");
    if (u) {
        h->mark("backproject");
        const int NPk = pad_np(k);  // Xt for ax = (C U_B)[:, :k]^T, NPk x NP
        const double* cu = WR;
        if (!h->c_identity) {
            h->launched(launch_small_matmul(c.slot(kC), WR, s, NP, c.slot(kX), false, st),
                        "small_matmul");
            cu = c.slot(kX);
        }
        h->ubt.reserve((size_t)NPk * NP * sizeof(double));
        h->launched(launch_fill(h->ubt.d(), (long)NPk * NP, 0.0, st), "fill");
        h->launched(launch_transpose(cu, s, k, NP, h->ubt.d(), NP, st), "transpose");
        if (p.f32) {  // U = Q1 (C U_B)[:, :k] with the K-major 3xTF32 kernel, FP64 out
            const int NPkf = (int)round_up(k, 16);
            h->ubtf.reserve((size_t)NPkf * p.NPf * sizeof(float));
            h->ubtf_lo.reserve((size_t)NPkf * p.NPf * sizeof(float));
            h->launched(launch_cvt_f64_f32(h->ubt.d(), NP, NPkf, p.NPf, k, s,
                                           static_cast<float*>(h->ubtf.p), p.NPf, st,
                                           static_cast<float*>(h->ubtf_lo.p)),
                        "cvt");
            const bool direct = (ldu == NPkf) && ((reinterpret_cast<uintptr_t>(u) & 15) == 0);
            if (!direct) h->y.reserve((size_t)m * NPkf * sizeof(double));
            GemmTf32 g{h->basis_f, m, (long)p.NPf, (long)p.NPf, static_cast<float*>(h->ubtf.p),
                       (long)p.NPf, NPkf, direct ? (void*)u : h->y.p, direct ? ldu : (long)NPkf};
            g.Blo = static_cast<float*>(h->ubtf_lo.p);
            gemm_tf32(h, g);
            if (!direct) h->launched(launch_copy2d(h->y.d(), NPkf, u, ldu, m, k, st), "copy2d");
            return;
        }
        const bool direct = (ldu == NPk) && ((reinterpret_cast<uintptr_t>(u) & 15) == 0);
        if (direct) {
            gemm_ax(h, h->basis, m, NP, NP, h->ubt.d(), NP, NPk, u, ldu);
        } else {
            // h->y is free at this point (power iteration done)
            h->y.reserve((size_t)m * std::max(NP, NPk) * sizeof(double));
            gemm_ax(h, h->basis, m, NP, NP, h->ubt.d(), NP, NPk, h->y.d(), NPk);
            h->launched(launch_copy2d(h->y.d(), NPk, u, ldu, m, k, st), "copy2d");
        }
    }
}

// Sharded runs: NaN/Inf seen in any shard and an abort on any rank become every rank's
// flags, on the device at the end of the pipeline (a sum all-reduce of two doubles between
// a pack and an unpack kernel), so finish_run's one flag download serves sharded runs too
// and the whole pipeline, collectives included, can be one CUDA graph.
void reduce_flags(const Ctx& c) {
    if (!c.p.sharded) return;
    rsvd_b200_handle* h = c.h;
    double* buf = h->flag_red.d();
    h->launched(launch_flags_pack(c.flags, kFlagNonfinite, kFlagAbort, buf, h->stream),
                "flags_pack");
    c.allreduce(buf, 2);
    h->launched(launch_flags_unpack(buf, c.flags, kFlagNonfinite, kFlagAbort, h->stream),
                "flags_unpack");
}

// Status checks after a run (one synchronisation). Returns false if the optimistic run
// must be repeated robustly.
bool finish_run(const Ctx& c, bool checked_nonfinite) {
    download_flags(c.h);
    c.h->sync();
    int* f = c.h->flags_host;  // sharded: NaN/abort already OR-reduced (reduce_flags)
    if (checked_nonfinite && f[kFlagNonfinite])
        fail(RSVD_B200_ARGUMENT_ERROR, "randomized_ksvd input contains NaN or Inf");
    if (f[kFlagAbort]) return false;
    c.h->last_sweeps = f[kFlagJacobi];
    if (f[kFlagJacobi] < 0)
        fail(RSVD_B200_CONVERGENCE_ERROR,
             "one-sided Jacobi SVD did not converge within 30 sweeps");
    if (f[kFlagComplete])
        fail(RSVD_B200_CONVERGENCE_ERROR, "dense_svd could not complete an orthonormal basis");
    return true;
}

// The optimistic pipeline of solve_tall as one CUDA graph. Eligible: single-device
// device-resident solves (no chunked upload in flight, no validation Omega, no forced robust
// path, no launch tracing, no profiling: events recorded by graph nodes cannot be timed). The first solve of a key is captured (relaxed
// mode: a first-time workspace allocation inside the capture is legal, and the key then
// records the generation after it) and launched; later solves with the same key replay it.
// Returns 0 when the solve must take the eager path (not eligible, or the capture failed),
// 1 when the replay produced the result, 2 when it raised the abort flag (a Cholesky
// breakdown): solve_tall then reruns on the robust path as after an eager optimistic attempt.
int solve_tall_graph(rsvd_b200_handle* h, const double* A, const Plan& p,
                      const rsvd_b200_config& cfg, double* u, long ldu, double* sigma, double* v,
                      long ldv) {
    static const bool disabled = getenv("RSVD_B200_NO_GRAPH") != nullptr;
    // sharded solves are captured when their transport is (NCCL's all-reduce is stream
    // capturable; the in-process test group synchronises on the host and is not)
    if (disabled || !h->use_graphs || h->force_robust || (p.sharded && !h->comm->capturable()) ||
        h->up_active || !h->omega_host.empty() || h->profiling != 0 || getenv("RSVD_B200_TRACE"))
        return 0;
    GraphKey key;
    key.a = p.f32 ? static_cast<const void*>(p.af) : A;
    key.m = p.m, key.n = p.n, key.lda = p.lda, key.s = p.s, key.NP = p.NP, key.f32 = p.f32;
    key.k = cfg.k, key.q = cfg.power_q, key.seed = cfg.seed;
    key.u = u, key.sigma = sigma, key.v = v, key.ldu = ldu, key.ldv = ldv;
    key.profiling = h->profiling;
    key.comm = p.sharded ? static_cast<const void*>(h->comm.get()) : nullptr;
    key.gen = g_ws_gen.load();
    key.apass = oz_mode(h, p);
    rsvd_b200_handle::SolveGraph* hit = nullptr;
    rsvd_b200_handle::SolveGraph* lru = &h->graphs[0];
    for (auto& cand : h->graphs) {
        if (cand.exec && cand.key.gen != key.gen) cand.reset();  // stale workspace pointers
        if (cand.exec && cand.key == key) hit = &cand;
        if (!cand.exec || (lru->exec && cand.used < lru->used)) lru = &cand;
    }
    auto& g = hit ? *hit : *lru;
    g.used = ++h->graph_clock;
    if (!hit) {
        g.reset();
        // everything the pipeline allocates is reserved before the capture starts
        begin_run(h, p, false);
        key.gen = g_ws_gen.load();
        const long launches0 = h->launches;
        cudaGraph_t graph = nullptr;
        ck(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeRelaxed), "begin capture");
        bool ok = true;
        std::string why;
        try {
            const Ctx c = begin_run(h, p, false);
            sketch_dev(c, A, cfg.seed, /*check=*/true);
            power_iterate_dev(c, A, cfg.power_q, false);
            project_and_solve_dev(c, A, (long)cfg.k, u, ldu, sigma, v, ldv);
            reduce_flags(c);
        } catch (const Failure& f) {
            ok = false;
            why = f.msg;
        } catch (...) {
            ok = false;
            why = "exception";
        }
        const cudaError_t ec = cudaStreamEndCapture(h->stream, &graph);
        cudaError_t ei = cudaSuccess;
        if (ok && ec == cudaSuccess && graph && g_ws_gen.load() == key.gen)
            ok = (ei = cudaGraphInstantiate(&g.exec, graph, 0)) == cudaSuccess;
        else
            ok = false;
        if (graph) cudaGraphDestroy(graph);
        if (getenv("RSVD_B200_GRAPH_DEBUG"))
            fprintf(stderr,
                    "[rsvd_b200] graph capture %s (end %s, instantiate %s, gen %lu -> %lu, slot "
                    "%ld%s%s)\n",
                    ok ? "ok" : "FAILED", cudaGetErrorString(ec), cudaGetErrorString(ei), key.gen,
                    g_ws_gen.load(), (long)(&g - h->graphs), why.empty() ? "" : ", ",
                    why.c_str());
        if (!ok) {
            cudaGetLastError();  // clear a capture error; the eager path reports real ones
            g.reset();
            h->launches = launches0;
            return 0;
        }
        g.key = key;
        g.launches = h->launches - launches0;
        h->launches = launches0;
    }
    ck(cudaGraphLaunch(g.exec, h->stream), "graph launch");
    h->launches += g.launches;
    h->graph_replays += 1;
    const Ctx c{h, p, false, static_cast<int*>(h->flags.p)};
    return finish_run(c, true) ? 1 : 2;
}

// Tall solve (rsvd.cpp:126-134) on device data. A: m x n (lda), m >= n. The optimistic
// pipeline runs first; a Cholesky breakdown anywhere reruns the whole solve on the robust
// path (Householder fallbacks), which reproduces the reference's QR semantics.
void solve_tall(rsvd_b200_handle* h, const double* A, const Plan& p, const rsvd_b200_config& cfg,
                double* u, long ldu, double* sigma, double* v, long ldv, size_t* sketch_width) {
    struct ClearAbort {  // no GEMM outside a solve may see a stale abort pointer
        rsvd_b200_handle* h;
        ~ClearAbort() { h->abort_ptr = nullptr; }
    } clear_abort{h};
    h->fallbacks = 0;
    h->reruns = 0;
    h->upload_aty = 0;
    const int gr = solve_tall_graph(h, A, p, cfg, u, ldu, sigma, v, ldv);
    if (gr == 1) {
        if (sketch_width) *sketch_width = (size_t)p.s;
        return;
    }
    if (gr == 2) h->reruns = 1;
    for (int attempt = gr == 2 ? 1 : 0; attempt < 2; ++attempt) {
        const Ctx c = begin_run(h, p, /*robust=*/attempt > 0 || h->force_robust);
        sketch_dev(c, A, cfg.seed, /*check=*/true, /*pre_aty=*/cfg.power_q > 0);
        power_iterate_dev(c, A, cfg.power_q, false);
        // range_basis(W) = W in the pipeline (see the header comment); k <= s always,
        // so pad_to_rank (rsvd.cpp:117-124) never widens the result here.
        project_and_solve_dev(c, A, (long)cfg.k, u, ldu, sigma, v, ldv);
        reduce_flags(c);
        h->mark("end");
        const bool ok = finish_run(c, true);
        h->finish_timers();
        if (ok) break;
        if (c.robust) fail(RSVD_B200_CUDA_ERROR, "internal: abort flag on the robust path");
        h->reruns += 1;
    }
    if (sketch_width) *sketch_width = (size_t)p.s;
}

// Device-side entry used by every public solve. Handles orientation (rsvd.cpp:150-156)
// and TMA alignment of A.
void solve_device(rsvd_b200_handle* h, const double* A, long m, long n, long lda,
                  const rsvd_b200_config& cfg, double* u, double* sigma, double* v,
                  size_t* sketch_width) {
    const long md = std::min(m, n);
    if (cfg.k < 1 || (long)cfg.k > md)
        fail(RSVD_B200_ARGUMENT_ERROR, "target rank k=%zu outside [1, %ld] for a %ldx%ld input",
             cfg.k, md, m, n);
    if (!(cfg.epsilon > 0.0 && cfg.epsilon < 1.0))
        fail(RSVD_B200_ARGUMENT_ERROR, "epsilon must lie in (0, 1)");
    const long k = (long)cfg.k;
    if (m >= n) {
        const double* a = A;
        long la = lda;
        if ((lda % 2) || (reinterpret_cast<uintptr_t>(A) & 15)) {  // TMA needs 16-byte rows
            la = round_up(n, 2);
            h->a_copy.reserve((size_t)m * la * sizeof(double));
            h->launched(launch_copy2d(A, lda, h->a_copy.d(), la, m, n, h->stream), "copy2d");
            a = h->a_copy.d();
        }
        const Plan p =
            make_plan(m, n, la, (long)rsvd_b200_sketch_width(&cfg, (size_t)m, (size_t)n));
        solve_tall(h, a, p, cfg, u, k, sigma, v, k, sketch_width);
        return;
    }
    // wide: solve on the materialised transpose, U and V swap roles
    const long lt = round_up(m, 2);
    h->a_t.reserve((size_t)n * lt * sizeof(double));
    h->launched(launch_transpose(A, m, n, lda, h->a_t.d(), lt, h->stream), "transpose");
    const Plan p = make_plan(n, m, lt, (long)rsvd_b200_sketch_width(&cfg, (size_t)n, (size_t)m));
    solve_tall(h, h->a_t.d(), p, cfg, v, k, sigma, u, k, sketch_width);
}

void make_f32(Plan& p, const float* af) {
    p.f32 = true;
    p.af = af;
    p.NPf = (int)round_up(p.s, 16);
    p.ldnf = round_up(p.n, 4);
}

// FP32 input (BASELINE config C4): A m x n FP32 (lda floats); outputs FP64 like every
// other entry point. Orientation handling as solve_device.
void solve_device_f32(rsvd_b200_handle* h, const float* A, long m, long n, long lda,
                      const rsvd_b200_config& cfg, double* u, double* sigma, double* v,
                      size_t* sketch_width) {
    const long md = std::min(m, n);
    if (cfg.k < 1 || (long)cfg.k > md)
        fail(RSVD_B200_ARGUMENT_ERROR, "target rank k=%zu outside [1, %ld] for a %ldx%ld input",
             cfg.k, md, m, n);
    if (!(cfg.epsilon > 0.0 && cfg.epsilon < 1.0))
        fail(RSVD_B200_ARGUMENT_ERROR, "epsilon must lie in (0, 1)");
    const long k = (long)cfg.k;
    if (m >= n) {
        const float* a = A;
        long la = lda;
        if ((lda % 4) || (reinterpret_cast<uintptr_t>(A) & 15)) {  // 16-byte TMA rows
            la = round_up(n, 4);
            h->af_copy.reserve((size_t)m * la * sizeof(float));
            ck(cudaMemcpy2DAsync(h->af_copy.p, la * 4, A, lda * 4, n * 4, m,
                                 cudaMemcpyDeviceToDevice, h->stream),
               "A copy");
            a = static_cast<float*>(h->af_copy.p);
        }
        Plan p = make_plan(m, n, la, (long)rsvd_b200_sketch_width(&cfg, (size_t)m, (size_t)n));
        make_f32(p, a);
        solve_tall(h, nullptr, p, cfg, u, k, sigma, v, k, sketch_width);
        return;
    }
    const long lt = round_up(m, 4);
    h->af_copy.reserve((size_t)n * lt * sizeof(float));
    h->launched(launch_transpose_f32(A, m, n, lda, static_cast<float*>(h->af_copy.p), lt,
                                     h->stream),
                "transpose_f32");
    Plan p = make_plan(n, m, lt, (long)rsvd_b200_sketch_width(&cfg, (size_t)n, (size_t)m));
    make_f32(p, static_cast<float*>(h->af_copy.p));
    solve_tall(h, nullptr, p, cfg, v, k, sigma, u, k, sketch_width);
}

// Row-sharded solve: this rank holds rows [r0, r0 + m_local) of the m_total x n input
// (m_total >= n). Every rank calls it collectively with the same n, m_total and config;
// sigma and V come back replicated, U sharded like A. The shard layout is checked
// collectively first (one tiny all-reduce), so a bad shard fails on every rank alike.
void solve_sharded(rsvd_b200_handle* h, const void* Av, bool f32, long m_local, long m_total,
                   long n, long lda, const rsvd_b200_config& cfg, double* u, double* sigma,
                   double* v, size_t* sketch_width) {
    if (!h->comm) fail(RSVD_B200_ARGUMENT_ERROR, "sharded solve needs a communicator "
                                                 "(rsvd_b200_comm_init_nccl / _local)");
    if (m_total < n)
        fail(RSVD_B200_DIMENSION_ERROR,
             "the row-sharded solve needs a tall input (m_total >= n), got %ldx%ld", m_total, n);
    const long md = std::min(m_total, n);
    if (cfg.k < 1 || (long)cfg.k > md)
        fail(RSVD_B200_ARGUMENT_ERROR, "target rank k=%zu outside [1, %ld] for a %ldx%ld input",
             cfg.k, md, m_total, n);
    if (!(cfg.epsilon > 0.0 && cfg.epsilon < 1.0))
        fail(RSVD_B200_ARGUMENT_ERROR, "epsilon must lie in (0, 1)");
    const long s = (long)rsvd_b200_sketch_width(&cfg, (size_t)m_total, (size_t)n);
    // collective shard check: sum of m_local, count of shards thinner than s — once per
    // layout and communicator (every rank caches the same verdict)
    const long layout[4] = {m_local, m_total, n, s};
    if (h->shard_ok_comm != h->comm.get() || !std::equal(layout, layout + 4, h->shard_ok)) {
        double chk[2] = {(double)m_local, m_local < s ? 1.0 : 0.0};
        h->red_scratch.reserve(2 * sizeof(double));
        ck(cudaMemcpyAsync(h->red_scratch.p, chk, sizeof chk, cudaMemcpyHostToDevice, h->stream),
           "shard check upload");
        const std::string err = h->comm->allreduce_sum(h->red_scratch.d(), 2, h->stream);
        if (!err.empty()) fail(RSVD_B200_NCCL_ERROR, "%s", err.c_str());
        ck(cudaMemcpyAsync(chk, h->red_scratch.p, sizeof chk, cudaMemcpyDeviceToHost, h->stream),
           "shard check download");
        h->sync();
        if ((long)chk[0] != m_total)
            fail(RSVD_B200_DIMENSION_ERROR, "shard rows sum to %ld, m_total is %ld",
                 (long)chk[0], m_total);
        if (chk[1] != 0.0)
            fail(RSVD_B200_DIMENSION_ERROR,
                 "every shard needs at least s=%ld rows (%d shard(s) are thinner)", s,
                 (int)chk[1]);
        h->shard_ok_comm = h->comm.get();
        std::copy(layout, layout + 4, h->shard_ok);
    }
    const long k = (long)cfg.k;
    if (f32) {
        const float* a = static_cast<const float*>(Av);
        long la = lda;
        if ((lda % 4) || (reinterpret_cast<uintptr_t>(a) & 15)) {
            la = round_up(n, 4);
            h->af_copy.reserve((size_t)m_local * la * sizeof(float));
            ck(cudaMemcpy2DAsync(h->af_copy.p, la * 4, a, lda * 4, n * 4, m_local,
                                 cudaMemcpyDeviceToDevice, h->stream),
               "A copy");
            a = static_cast<float*>(h->af_copy.p);
        }
        Plan p = make_plan(m_local, n, la, s);
        p.sharded = true;
        make_f32(p, a);
        solve_tall(h, nullptr, p, cfg, u, k, sigma, v, k, sketch_width);
        return;
    }
    const double* A = static_cast<const double*>(Av);
    const double* a = A;
    long la = lda;
    if ((lda % 2) || (reinterpret_cast<uintptr_t>(A) & 15)) {  // TMA needs 16-byte rows
        la = round_up(n, 2);
        h->a_copy.reserve((size_t)m_local * la * sizeof(double));
        h->launched(launch_copy2d(A, lda, h->a_copy.d(), la, m_local, n, h->stream), "copy2d");
        a = h->a_copy.d();
    }
    Plan p = make_plan(m_local, n, la, s);
    p.sharded = true;
    solve_tall(h, a, p, cfg, u, k, sigma, v, k, sketch_width);
}

}  // namespace

// ||A - U diag(sigma) V^T||_F (RsvdResult::residual_fro, rsvd.cpp:37-49) on the device:
// U diag(sigma) V^T is never formed; each 96-column chunk of it is the accumulator of an
// ax GEMM (K = k) whose epilogue subtracts it from A's chunk and sums the squares per CTA.
// All device pointers; sigma_dev has k entries. Returns the norm (synchronises).
double residual_device(rsvd_b200_handle* h, const double* A, long m, long n, long lda,
                       const double* U, long ldu, const double* sigma_dev, const double* V,
                       long ldv, long k) {
    cudaStream_t st = h->stream;
    const long kp = round_up(k, 2);  // TMA rows of U / Vs: 16-byte multiples
    const double* Ua = U;
    if (ldu != kp || (reinterpret_cast<uintptr_t>(U) & 15)) {
        h->res_u.reserve((size_t)m * kp * sizeof(double));
        h->launched(launch_fill(h->res_u.d(), m * kp, 0.0, st), "fill");
        h->launched(launch_copy2d(U, ldu, h->res_u.d(), kp, m, k, st), "copy2d");
        Ua = h->res_u.d();
    }
    const long chunk = 96, npad = round_up(n, chunk), chunks = npad / chunk;
    h->res_vs.reserve((size_t)npad * kp * sizeof(double));
    h->launched(launch_scale_cols(V, ldv, n, npad, (int)k, sigma_dev, h->res_vs.d(), kp, st),
                "scale_cols");
    const long tiles = (m + 127) / 128;
    h->res_part.reserve((size_t)(chunks * tiles + 1) * sizeof(double));
    double* part = h->res_part.d();
    for (long c = 0; c < chunks; ++c) {
        GemmAx g{Ua, m, kp, kp, h->res_vs.d() + c * chunk * kp, kp, (int)chunk, nullptr, 0};
        g.resid = A + c * chunk;
        g.resid_ld = lda;
        g.resid_cols = (int)std::min(chunk, n - c * chunk);
        g.resid_out = part + c * tiles;
        h->launched(launch_gemm_ax(g, st), "gemm_ax(resid)");
    }
    double* tot = part + chunks * tiles;
    h->launched(launch_reduce_partials(part, 1, (int)(chunks * tiles), tot, 1, st),
                "reduce_partials");
    double r = 0.0;
    ck(cudaMemcpyAsync(&r, tot, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H residual");
    h->sync();
    return std::sqrt(r);
}

// PCA centering on the device (pca.cpp:10-26): column sums of X (N x d, ldx) by the atx
// GEMM against a ones operand (deterministic split-K), then Xc = X - 1 mean^T into
// Xc (ld ldc, may alias X) and mean into h->pca_mean.
void pca_center(rsvd_b200_handle* h, const double* X, long N, long d, long ldx, double* Xc,
                long ldc) {
    cudaStream_t st = h->stream;
    const int NP = 16;
    const long ldd = round_up(d, 2);
    h->pca_ones.reserve((size_t)N * NP * sizeof(double));
    h->pca_sums.reserve((size_t)NP * ldd * sizeof(double));
    h->pca_mean.reserve((size_t)d * sizeof(double));
    h->launched(launch_fill(h->pca_ones.d(), N * NP, 1.0, st), "fill");
    // part must hold the split-K slabs of this product
    const int sp = choose_splits(ax_tiles(d, NP), (N + 31) / 32);
    h->part.reserve((size_t)std::max(1, sp) * NP * ldd * sizeof(double));
    gemm_atx(h, X, N, d, ldx, h->pca_ones.d(), NP, NP, h->pca_sums.d(), ldd, true);
    h->launched(launch_center(X, ldx, N, d, h->pca_sums.d(), nullptr, Xc, ldc, h->pca_mean.d(), st),
                "center");
}

// ====================================================================== C-ABI
extern "C" {

void rsvd_b200_config_default(rsvd_b200_config* cfg) {
    cfg->k = 1;
    cfg->oversample = 10;
    cfg->power_q = 2;
    cfg->seed = 0;
    cfg->epsilon = 0.5;
    cfg->epsilon_mode = 0;
}

size_t rsvd_b200_sketch_width(const rsvd_b200_config* cfg, size_t m, size_t n) {
    const size_t cap = std::min(m, n);
    if (cfg->epsilon_mode) {
        const double raw = std::ceil(static_cast<double>(cfg->k) / cfg->epsilon);
        return std::min<size_t>(static_cast<size_t>(raw), cap);
    }
    return std::min(cfg->k + cfg->oversample, cap);
}

const char* rsvd_b200_last_error(void) { return g_last_error.c_str(); }

const char* rsvd_b200_version(void) { return "rsvd_b200 0.1 (sm_100a, FP64 DMMA)"; }

rsvd_b200_status rsvd_b200_create(int device, rsvd_b200_handle** out) {
    return guarded([&] {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
            fail(RSVD_B200_CUDA_ERROR, "no CUDA device available");
        if (device < 0 || device >= count)
            fail(RSVD_B200_ARGUMENT_ERROR, "device %d outside [0, %d)", device, count);
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major != 10)
            fail(RSVD_B200_CUDA_ERROR, "device %d is sm_%d%d; this library is built for sm_100a",
                 device, prop.major, prop.minor);
        auto* h = new rsvd_b200_handle();
        h->device = device;
        ck(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "stream create");
        h->flags.reserve(kNumFlags * sizeof(int));
        ck(cudaMallocHost(&h->flags_host, kNumFlags * sizeof(int)), "cudaMallocHost");
        *out = h;
    });
}

rsvd_b200_status rsvd_b200_destroy(rsvd_b200_handle* h) {
    if (!h) return RSVD_B200_OK;
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->stream);
    if (h->copy_stream) {
        cudaStreamSynchronize(h->copy_stream);
        cudaStreamDestroy(h->copy_stream);
    }
    for (cudaEvent_t e : h->up_ev) cudaEventDestroy(e);
    if (h->up_start) cudaEventDestroy(h->up_start);
    h->reset_graphs();
    if (h->flags_host) cudaFreeHost(h->flags_host);
    cudaStreamDestroy(h->stream);
    delete h;
    return RSVD_B200_OK;
}

void* rsvd_b200_stream(rsvd_b200_handle* h) { return h->stream; }

rsvd_b200_status rsvd_b200_wait_stream(rsvd_b200_handle* h, void* other) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        cudaEvent_t ev;
        ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event create");
        ck(cudaEventRecord(ev, static_cast<cudaStream_t>(other)), "event record");
        ck(cudaStreamWaitEvent(h->stream, ev, 0), "stream wait");
        cudaEventDestroy(ev);
    });
}

rsvd_b200_status rsvd_b200_set_omega(rsvd_b200_handle* h, const double* omega, size_t rows,
                                     size_t cols) {
    return guarded([&] {
        if (!omega) {
            h->omega_host.clear();
            h->omega_rows = h->omega_cols = 0;
            return;
        }
        h->omega_host.assign(omega, omega + rows * cols);
        h->omega_rows = rows;
        h->omega_cols = cols;
    });
}

void rsvd_b200_set_profiling(rsvd_b200_handle* h, int level) { h->profiling = level; }

int rsvd_b200_kernel_stats(rsvd_b200_handle* h, const char* tag, long* count, double* total_ms,
                           double* total_flops) {
    for (auto& e : h->kstats)
        if (e.first == tag) {
            *count = e.second.count;
            *total_ms = e.second.ms;
            *total_flops = e.second.flops;
            return 1;
        }
    *count = 0;
    *total_ms = *total_flops = 0.0;
    return 0;
}

void rsvd_b200_reset_stats(rsvd_b200_handle* h) { h->kstats.clear(); }

int rsvd_b200_last_profile(rsvd_b200_handle* h, const char** names, double* ms, int max) {
    // merge repeated stage names
    std::vector<std::pair<const char*, double>> merged;
    for (auto& e : h->last_profile) {
        if (!strcmp(e.first, "end")) continue;
        auto it = std::find_if(merged.begin(), merged.end(),
                               [&](auto& x) { return !strcmp(x.first, e.first); });
        if (it == merged.end())
            merged.push_back(e);
        else
            it->second += e.second;
    }
    const int n = std::min<int>(max, (int)merged.size());
    for (int i = 0; i < n; ++i) {
        names[i] = merged[i].first;
        ms[i] = merged[i].second;
    }
    return n;
}

long rsvd_b200_last_launch_count(rsvd_b200_handle* h) { return h->launches; }

rsvd_b200_status rsvd_b200_randomized_ksvd_device(rsvd_b200_handle* h, const double* a_dev,
                                                  size_t m, size_t n, size_t lda,
                                                  const rsvd_b200_config* cfg, double* u_dev,
                                                  double* sigma_dev, double* v_dev,
                                                  size_t* sketch_width) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        h->launches = 0;
        solve_device(h, a_dev, (long)m, (long)n, (long)lda, *cfg, u_dev, sigma_dev, v_dev,
                     sketch_width);
    });
}

// H2D of a host A (m x n) into h->a_copy (lda). Tall inputs large enough to matter go up in
// row chunks on the copy stream (up_ev per chunk) for sketch_dev to consume as they land;
// everything else is one copy on the solve stream.
static void upload_a(rsvd_b200_handle* h, const void* av, long m, long n, long lda,
                     size_t esz = sizeof(double)) {
    const char* a = static_cast<const char*>(av);
    h->a_copy.reserve((size_t)m * lda * esz);
    const long bytes_row = lda * (long)esz;
    const char* mb = getenv("RSVD_B200_UPLOAD_CHUNK_MB");  // tests: force small chunks
    const long chunk_bytes = (mb && atol(mb) > 0 ? atol(mb) : 256l) << 20;
    const long chunk_rows = round_up(std::max<long>(128, chunk_bytes / bytes_row), 128);
    if (m < n || m < 2 * chunk_rows) {
        ck(cudaMemcpy2DAsync(h->a_copy.p, bytes_row, a, n * esz, n * esz, m,
                             cudaMemcpyHostToDevice, h->stream),
           "H2D of A");
        return;
    }
    const long chunks = (m + chunk_rows - 1) / chunk_rows;
    ensure_side_stream(h, chunks);
    // the copies must not overtake earlier work on the solve stream that reads a_copy
    ck(cudaEventRecord(h->up_start, h->stream), "event record");
    ck(cudaStreamWaitEvent(h->copy_stream, h->up_start, 0), "stream wait");
    for (long c = 0; c < chunks; ++c) {
        const long r0 = c * chunk_rows, rows = std::min(m - r0, chunk_rows);
        ck(cudaMemcpy2DAsync(static_cast<char*>(h->a_copy.p) + r0 * bytes_row, bytes_row,
                             a + r0 * n * esz, n * esz, n * esz, rows, cudaMemcpyHostToDevice,
                             h->copy_stream),
           "H2D of A");
        ck(cudaEventRecord(h->up_ev[c], h->copy_stream), "event record");
    }
    h->up_chunk_rows = chunk_rows;
    h->up_chunks = chunks;
    h->up_active = true;
}

// Whatever path the solve took (or if it failed early), the solve stream ends up ordered
// after the whole upload.
struct UploadFence {
    rsvd_b200_handle* h;
    ~UploadFence() {
        if (h->up_active) {
            cudaStreamWaitEvent(h->stream, h->up_ev[h->up_chunks - 1], 0);
            h->up_active = false;
        }
    }
};

static void solve_host(rsvd_b200_handle* h, const double* a, size_t m, size_t n,
                       const rsvd_b200_config* cfg, double* u, double* sigma, double* v,
                       size_t* sketch_width) {
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    h->launches = 0;
    const long lda = round_up((long)n, 2);
    UploadFence fence{h};
    upload_a(h, a, (long)m, (long)n, lda);
    const size_t k = cfg->k;
    h->sig_out.reserve(std::max<size_t>(k, 1) * sizeof(double));
    if (u) h->u_out.reserve(std::max<size_t>(m * k, 1) * sizeof(double));
    if (v) h->v_out.reserve(std::max<size_t>(n * k, 1) * sizeof(double));
    solve_device(h, h->a_copy.d(), (long)m, (long)n, lda, *cfg, u ? h->u_out.d() : nullptr,
                 h->sig_out.d(), v ? h->v_out.d() : nullptr, sketch_width);
    ck(cudaMemcpyAsync(sigma, h->sig_out.p, k * sizeof(double), cudaMemcpyDeviceToHost, h->stream),
       "D2H sigma");
    if (u)
        ck(cudaMemcpyAsync(u, h->u_out.p, m * k * sizeof(double), cudaMemcpyDeviceToHost,
                           h->stream),
           "D2H u");
    if (v)
        ck(cudaMemcpyAsync(v, h->v_out.p, n * k * sizeof(double), cudaMemcpyDeviceToHost,
                           h->stream),
           "D2H v");
    h->sync();
}

// ------------------------------------------------------------ row-sharded solves
struct rsvd_b200_local_group {
    explicit rsvd_b200_local_group(int w) : g(w) {}
    LocalGroup g;
};

rsvd_b200_status rsvd_b200_nccl_unique_id(unsigned char* out) {
    return guarded([&] {
        const std::string err = nccl_unique_id(out);
        if (!err.empty()) fail(RSVD_B200_NCCL_ERROR, "%s", err.c_str());
    });
}

rsvd_b200_status rsvd_b200_comm_init_nccl(rsvd_b200_handle* h, const unsigned char* id, int rank,
                                          int world) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world)
            fail(RSVD_B200_ARGUMENT_ERROR, "rank %d outside [0, %d)", rank, world);
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        std::unique_ptr<Comm> c;
        const std::string err = make_nccl_comm(id, rank, world, &c);
        if (!err.empty()) fail(RSVD_B200_NCCL_ERROR, "%s", err.c_str());
        h->comm = std::move(c);
    });
}

rsvd_b200_status rsvd_b200_local_group_create(int world, rsvd_b200_local_group** out) {
    return guarded([&] {
        if (world < 1 || world > 16)
            fail(RSVD_B200_ARGUMENT_ERROR, "local group size %d outside [1, 16]", world);
        *out = new rsvd_b200_local_group(world);
    });
}

void rsvd_b200_local_group_destroy(rsvd_b200_local_group* g) { delete g; }

rsvd_b200_status rsvd_b200_comm_init_local(rsvd_b200_handle* h, rsvd_b200_local_group* g,
                                           int rank) {
    return guarded([&] {
        if (!g || rank < 0 || rank >= g->g.world)
            fail(RSVD_B200_ARGUMENT_ERROR, "rank %d outside the local group", rank);
        h->comm = make_local_comm(&g->g, rank);
    });
}

rsvd_b200_status rsvd_b200_comm_info(rsvd_b200_handle* h, int* rank, int* world) {
    *rank = h->comm ? h->comm->rank : 0;
    *world = h->comm ? h->comm->world : 1;
    return RSVD_B200_OK;
}

void rsvd_b200_comm_free(rsvd_b200_handle* h) {
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->stream);
    h->comm.reset();
}

rsvd_b200_status rsvd_b200_randomized_ksvd_sharded_device(
    rsvd_b200_handle* h, const double* a_dev, size_t m_local, size_t m_total, size_t n,
    size_t lda, const rsvd_b200_config* cfg, double* u_dev, double* sigma_dev, double* v_dev,
    size_t* sketch_width) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        h->launches = 0;
        solve_sharded(h, a_dev, false, (long)m_local, (long)m_total, (long)n, (long)lda, *cfg,
                      u_dev, sigma_dev, v_dev, sketch_width);
    });
}

rsvd_b200_status rsvd_b200_randomized_ksvd_sharded(rsvd_b200_handle* h, const double* a,
                                                   size_t m_local, size_t m_total, size_t n,
                                                   const rsvd_b200_config* cfg, double* u,
                                                   double* sigma, double* v,
                                                   size_t* sketch_width) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        h->launches = 0;
        const long lda = round_up((long)n, 2);
        UploadFence fence{h};
        // chunked when tall: the sketch consumes the shard's rows as they land, as unsharded
        upload_a(h, a, (long)m_local, (long)n, lda);
        const size_t k = cfg->k;
        h->sig_out.reserve(std::max<size_t>(k, 1) * sizeof(double));
        if (u) h->u_out.reserve(std::max<size_t>(m_local * k, 1) * sizeof(double));
        if (v) h->v_out.reserve(std::max<size_t>(n * k, 1) * sizeof(double));
        solve_sharded(h, h->a_copy.d(), false, (long)m_local, (long)m_total, (long)n, lda, *cfg,
                      u ? h->u_out.d() : nullptr, h->sig_out.d(), v ? h->v_out.d() : nullptr,
                      sketch_width);
        ck(cudaMemcpyAsync(sigma, h->sig_out.p, k * sizeof(double), cudaMemcpyDeviceToHost,
                           h->stream),
           "D2H sigma");
        if (u)
            ck(cudaMemcpyAsync(u, h->u_out.p, m_local * k * sizeof(double),
                               cudaMemcpyDeviceToHost, h->stream),
               "D2H u");
        if (v)
            ck(cudaMemcpyAsync(v, h->v_out.p, n * k * sizeof(double), cudaMemcpyDeviceToHost,
                               h->stream),
               "D2H v");
        h->sync();
    });
}

rsvd_b200_status rsvd_b200_randomized_ksvd(rsvd_b200_handle* h, const double* a, size_t m,
                                           size_t n, const rsvd_b200_config* cfg, double* u,
                                           double* sigma, double* v, size_t* sketch_width) {
    return guarded([&] { solve_host(h, a, m, n, cfg, u, sigma, v, sketch_width); });
}

rsvd_b200_status rsvd_b200_singular_values_only(rsvd_b200_handle* h, const double* a, size_t m,
                                                size_t n, const rsvd_b200_config* cfg,
                                                double* sigma) {
    return guarded([&] { solve_host(h, a, m, n, cfg, nullptr, sigma, nullptr, nullptr); });
}

// ---------------------------------------------------------------- FP32 input
rsvd_b200_status rsvd_b200_randomized_ksvd_f32_device(rsvd_b200_handle* h, const float* a_dev,
                                                      size_t m, size_t n, size_t lda,
                                                      const rsvd_b200_config* cfg, double* u_dev,
                                                      double* sigma_dev, double* v_dev,
                                                      size_t* sketch_width) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        h->launches = 0;
        solve_device_f32(h, a_dev, (long)m, (long)n, (long)lda, *cfg, u_dev, sigma_dev, v_dev,
                         sketch_width);
    });
}

// Host-buffer FP32 solve (and, with world > 1 communicators, the sharded one): A goes to
// h->a_copy (raw bytes), outputs come back from the handle's FP64 output buffers.
static void solve_host_f32(rsvd_b200_handle* h, const float* a, size_t m_local, size_t m_total,
                           size_t n, bool sharded, const rsvd_b200_config* cfg, double* u,
                           double* sigma, double* v, size_t* sketch_width) {
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    h->launches = 0;
    const long lda = round_up((long)n, 4);
    UploadFence fence{h};
    upload_a(h, a, (long)m_local, (long)n, lda, sizeof(float));  // chunked when tall
    const size_t k = cfg->k;
    h->sig_out.reserve(std::max<size_t>(k, 1) * sizeof(double));
    if (u) h->u_out.reserve(std::max<size_t>(m_local * k, 1) * sizeof(double));
    if (v) h->v_out.reserve(std::max<size_t>(n * k, 1) * sizeof(double));
    const float* ad = static_cast<const float*>(h->a_copy.p);
    if (sharded)
        solve_sharded(h, ad, true, (long)m_local, (long)m_total, (long)n, lda, *cfg,
                      u ? h->u_out.d() : nullptr, h->sig_out.d(), v ? h->v_out.d() : nullptr,
                      sketch_width);
    else
        solve_device_f32(h, ad, (long)m_local, (long)n, lda, *cfg, u ? h->u_out.d() : nullptr,
                         h->sig_out.d(), v ? h->v_out.d() : nullptr, sketch_width);
    ck(cudaMemcpyAsync(sigma, h->sig_out.p, k * sizeof(double), cudaMemcpyDeviceToHost, h->stream),
       "D2H sigma");
    const size_t urows = sharded || m_local >= n ? m_local : m_local;
    if (u)
        ck(cudaMemcpyAsync(u, h->u_out.p, urows * k * sizeof(double), cudaMemcpyDeviceToHost,
                           h->stream),
           "D2H u");
    if (v)
        ck(cudaMemcpyAsync(v, h->v_out.p, n * k * sizeof(double), cudaMemcpyDeviceToHost,
                           h->stream),
           "D2H v");
    h->sync();
}

rsvd_b200_status rsvd_b200_randomized_ksvd_f32(rsvd_b200_handle* h, const float* a, size_t m,
                                               size_t n, const rsvd_b200_config* cfg, double* u,
                                               double* sigma, double* v, size_t* sketch_width) {
    return guarded([&] { solve_host_f32(h, a, m, m, n, false, cfg, u, sigma, v, sketch_width); });
}

rsvd_b200_status rsvd_b200_randomized_ksvd_sharded_f32(rsvd_b200_handle* h, const float* a,
                                                       size_t m_local, size_t m_total, size_t n,
                                                       const rsvd_b200_config* cfg, double* u,
                                                       double* sigma, double* v,
                                                       size_t* sketch_width) {
    return guarded(
        [&] { solve_host_f32(h, a, m_local, m_total, n, true, cfg, u, sigma, v, sketch_width); });
}

rsvd_b200_status rsvd_b200_randomized_ksvd_sharded_f32_device(
    rsvd_b200_handle* h, const float* a_dev, size_t m_local, size_t m_total, size_t n,
    size_t lda, const rsvd_b200_config* cfg, double* u_dev, double* sigma_dev, double* v_dev,
    size_t* sketch_width) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        h->launches = 0;
        solve_sharded(h, a_dev, true, (long)m_local, (long)m_total, (long)n, (long)lda, *cfg,
                      u_dev, sigma_dev, v_dev, sketch_width);
    });
}

rsvd_b200_status rsvd_b200_gaussian_matrix(rsvd_b200_handle* h, uint64_t seed, size_t rows,
                                           size_t cols, double* out) {
    return rsvd_b200_gaussian_stream(h, seed, 0, 0, 0.0, rows, cols, out);
}

rsvd_b200_status rsvd_b200_gaussian_stream(rsvd_b200_handle* h, uint64_t seed, uint64_t counter,
                                           int has_cached, double cached, size_t rows,
                                           size_t cols, double* out) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        DevBuf d;
        d.reserve(std::max<size_t>(rows * cols, 1) * sizeof(double));
        const StreamPos pos{counter, has_cached ? 1 : 0, cached};
        h->launched(launch_gaussian_rowmajor(seed, (long)rows, (long)cols, d.d(), h->stream, pos),
                    "gaussian");
        ck(cudaMemcpyAsync(out, d.p, rows * cols * sizeof(double), cudaMemcpyDeviceToHost,
                           h->stream),
           "D2H");
        h->sync();
    });
}

rsvd_b200_status rsvd_b200_splitmix_words(rsvd_b200_handle* h, uint64_t seed,
                                          uint64_t first_counter, size_t count, uint64_t* out) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        DevBuf d;
        d.reserve(std::max<size_t>(count, 1) * sizeof(uint64_t));
        h->launched(launch_splitmix_words(seed, first_counter, (long)count,
                                          static_cast<uint64_t*>(d.p), h->stream),
                    "words");
        ck(cudaMemcpyAsync(out, d.p, count * sizeof(uint64_t), cudaMemcpyDeviceToHost, h->stream),
           "D2H");
        h->sync();
    });
}

rsvd_b200_status rsvd_b200_uniforms(rsvd_b200_handle* h, uint64_t seed, uint64_t first_counter,
                                    size_t count, double* out) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        DevBuf d;
        d.reserve(std::max<size_t>(count, 1) * sizeof(double));
        h->launched(launch_uniforms(seed, first_counter, (long)count, d.d(), h->stream),
                    "uniforms");
        ck(cudaMemcpyAsync(out, d.p, count * sizeof(double), cudaMemcpyDeviceToHost, h->stream),
           "D2H");
        h->sync();
    });
}

}  // extern "C"

// ============================================================ step functions
namespace {

// Upload a host row-major matrix into `buf` with an even leading dimension (TMA rows
// must be 16-byte multiples); returns the leading dimension.
long upload(rsvd_b200_handle* h, DevBuf& buf, const double* src, long rows, long cols, long ld) {
    buf.reserve((size_t)std::max(1L, rows * ld) * sizeof(double));
    if (ld > cols) ck(cudaMemsetAsync(buf.p, 0, (size_t)rows * ld * sizeof(double), h->stream), "memset");
    ck(cudaMemcpy2DAsync(buf.p, ld * sizeof(double), src, cols * sizeof(double),
                         cols * sizeof(double), rows, cudaMemcpyHostToDevice, h->stream),
       "H2D");
    return ld;
}

void download(rsvd_b200_handle* h, double* dst, const double* src, long rows, long cols, long ld) {
    ck(cudaMemcpy2DAsync(dst, cols * sizeof(double), src, ld * sizeof(double),
                         cols * sizeof(double), rows, cudaMemcpyDeviceToHost, h->stream),
       "D2H");
    h->sync();
}

void check_shape(long rows, long cols, const char* what) {
    if (rows < 1 || cols < 1)
        fail(RSVD_B200_DIMENSION_ERROR, "%s requires rows >= 1 and cols >= 1, got %ldx%ld", what,
             rows, cols);
}

}  // namespace

extern "C" {

rsvd_b200_status rsvd_b200_sketch(rsvd_b200_handle* h, const double* a, size_t m, size_t n,
                                  size_t s, uint64_t seed, double* y0) {
    return rsvd_b200_sketch_stream(h, a, m, n, s, seed, 0, 0, 0.0, y0);
}

rsvd_b200_status rsvd_b200_sketch_stream(rsvd_b200_handle* h, const double* a, size_t m,
                                         size_t n, size_t s, uint64_t seed, uint64_t counter,
                                         int has_cached, double cached, double* y0) {
    struct PosGuard {  // the solve pipelines always start from a fresh sampler
        rsvd_b200_handle* h;
        ~PosGuard() { h->omega_pos = StreamPos{}; }
    } guard{h};
    h->omega_pos = StreamPos{counter, has_cached ? 1 : 0, cached};
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        check_shape((long)m, (long)n, "sketch");
        const size_t md = std::min(m, n);
        if (s < 1 || s > md)
            fail(RSVD_B200_ARGUMENT_ERROR, "sketch width %zu outside [1, %zu] for a %zux%zu input",
                 s, md, m, n);
        const long lda = upload(h, h->a_copy, a, (long)m, (long)n, round_up((long)n, 2));
        const Ctx c = begin_run(h, make_plan((long)m, (long)n, lda, (long)s), true);
        sketch_dev(c, h->a_copy.d(), seed, false);
        download(h, y0, h->y.d(), (long)m, (long)s, c.p.NP);
    });
}

rsvd_b200_status rsvd_b200_power_iterate(rsvd_b200_handle* h, const double* a, size_t m, size_t n,
                                         const double* y0, size_t s, size_t q, double* w) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        check_shape((long)m, (long)n, "power_iterate");
        check_shape((long)m, (long)s, "power_iterate y0");
        const long lda = upload(h, h->a_copy, a, (long)m, (long)n, round_up((long)n, 2));
        const Ctx c = begin_run(h, make_plan((long)m, (long)n, lda, (long)s), true);
        upload(h, h->y, y0, (long)m, (long)s, c.p.NP);
        h->gram_ready = false;
        power_iterate_dev(c, h->a_copy.d(), q, /*materialize=*/true);
        download(h, w, h->basis, (long)m, (long)s, c.p.NP);
    });
}

// Householder thin QR (qr.cpp:27-102) on the device: the blocked compact-WY kernel of
// householder.cu. a (m x n, lda) may be host or device memory per `on_device`; q (m x n,
// ldq) and r (n x n, ldr) likewise.
void householder_qr_impl(rsvd_b200_handle* h, const double* a, long lda, long m, long n,
                         double* q, long ldq, double* r, long ldr, bool on_device) {
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    check_shape(m, n, "householder_qr");
    if (m < n)
        fail(RSVD_B200_DIMENSION_ERROR,
             "householder_qr needs rows >= cols, got %ldx%ld; transpose the input first", m, n);
    const int NP = (int)(n <= 288 ? pad_np(n) : round_up(n, 8));
    h->y.reserve((size_t)m * NP * sizeof(double));
    h->q.reserve((size_t)m * NP * sizeof(double));
    h->hh_rows.reserve((size_t)NP * NP * sizeof(double));
    h->hh_work.reserve(householder_work_doubles(m, NP) * sizeof(double));
    ck(cudaMemcpy2DAsync(h->y.p, NP * sizeof(double), a, lda * sizeof(double), n * sizeof(double),
                         m, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                         h->stream),
       "copy a");
    double* R = h->hh_rows.d();
    h->launched(launch_householder_qr(h->y.d(), m, (int)n, NP, h->q.d(), NP, R, NP,
                                      h->hh_work.d(), h->stream),
                "householder_qr");
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    ck(cudaMemcpy2DAsync(q, ldq * sizeof(double), h->q.p, NP * sizeof(double), n * sizeof(double),
                         m, kind, h->stream),
       "copy q");
    ck(cudaMemcpy2DAsync(r, ldr * sizeof(double), R, NP * sizeof(double), n * sizeof(double), n,
                         kind, h->stream),
       "copy r");
    if (!on_device) h->sync();
}

// synth_matrix (synth.cpp:58-71) on the device: the reference's construction step for step
// — one GaussianSampler(seed) stream (the device generator, bit-identical to the
// reference's) filled row-major into the rows x cols and then the cols x cols Gaussian
// draws, Haar factors as their Householder Q (householder.cu; diag R >= 0 is the Haar sign
// fix), U's columns scaled by sigma_j = spectrum_value(kind, j + 1) (evaluated on the host
// with the same libm calls as the reference), A = U V^T by the DMMA GEMM in column blocks.
void synth_matrix_impl(rsvd_b200_handle* h, long rows, long cols, int kind, double beta,
                       uint64_t seed, double* out, long ldo, bool on_device) {
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    if (rows < cols || cols < 1)
        fail(RSVD_B200_ARGUMENT_ERROR, "synth_matrix needs rows >= cols >= 1, got %ldx%ld", rows,
             cols);
    if (kind < 0 || kind > 2) fail(RSVD_B200_ARGUMENT_ERROR, "synth_matrix: unknown spectrum kind %d", kind);
    if (kind == 1 && !(beta > 0.0))
        fail(RSVD_B200_ARGUMENT_ERROR, "sharp decay requires beta > 0, got %g", beta);
    std::vector<double> sig((size_t)cols);
    for (long j = 0; j < cols; ++j) {  // synth.cpp:28-40, 1-based index
        const double x = (double)(j + 1);
        sig[j] = kind == 0 ? 1.0 / (x * x)
                 : kind == 1 ? 0.0001 + 1.0 / (1.0 + std::exp(x + 1.0 - beta))
                             : 1.0 / std::pow(x, 0.1);
    }
    const long NP = cols <= 288 ? pad_np(cols) : round_up(cols, 8);
    constexpr long kBlk = 96;                        // output columns per GEMM
    const long vrows = round_up(cols, kBlk);         // V padded (zero rows) for the last block
    const size_t g_n = (size_t)rows * cols + (size_t)cols * cols;
    // workspace: Gaussian draws | U (rows x NP) | V (vrows x NP) | sigma | GEMM tile
    const size_t need = g_n + (size_t)rows * NP + (size_t)vrows * NP + NP +
                        (size_t)rows * kBlk;
    h->synth_buf.reserve(need * sizeof(double));
    double* g = h->synth_buf.d();
    double* u = g + g_n;
    double* v = u + (size_t)rows * NP;
    double* sg = v + (size_t)vrows * NP;
    double* tile = sg + NP;
    h->hh_rows.reserve((size_t)NP * NP * sizeof(double));
    h->hh_work.reserve(householder_work_doubles(rows, NP) * sizeof(double));
    h->launched(launch_gaussian_rowmajor(seed, 1, (long)g_n, g, h->stream), "gaussian");
    h->launched(launch_fill(v, vrows * NP, 0.0, h->stream), "fill");
    h->launched(launch_householder_qr(g, rows, (int)cols, cols, u, NP, h->hh_rows.d(), (int)NP,
                                      h->hh_work.d(), h->stream),
                "householder_qr");
    h->launched(launch_householder_qr(g + (size_t)rows * cols, cols, (int)cols, cols, v, NP,
                                      h->hh_rows.d(), (int)NP, h->hh_work.d(), h->stream),
                "householder_qr");
    ck(cudaMemcpyAsync(sg, sig.data(), cols * sizeof(double), cudaMemcpyHostToDevice, h->stream),
       "sigma upload");
    // U <- U diag(sigma) in place (columns >= cols stay zero)
    h->launched(launch_scale_cols(u, NP, rows, rows, (int)cols, sg, u, NP, h->stream), "scale_cols");
    const cudaMemcpyKind kind_out = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    const int splits = choose_splits(ax_tiles(rows, (int)kBlk), (NP + 31) / 32);
    if (splits > 1) h->part.reserve((size_t)splits * rows * kBlk * sizeof(double));
    for (long j0 = 0; j0 < cols; j0 += kBlk) {  // A[:, j0:j0+96] = U (V[j0:j0+96, :])^T
        const long nb = std::min(kBlk, cols - j0);
        gemm_ax(h, u, rows, NP, NP, v + (size_t)j0 * NP, NP, (int)kBlk, tile, kBlk);
        ck(cudaMemcpy2DAsync(out + j0, ldo * sizeof(double), tile, kBlk * sizeof(double),
                             nb * sizeof(double), rows, kind_out, h->stream),
           "copy a");
    }
    h->sync();  // the host-side sigma vector's lifetime
}

rsvd_b200_status rsvd_b200_synth_matrix(rsvd_b200_handle* h, size_t rows, size_t cols, int kind,
                                        double beta, uint64_t seed, double* out) {
    return guarded([&] {
        synth_matrix_impl(h, (long)rows, (long)cols, kind, beta, seed, out, (long)cols, false);
    });
}

rsvd_b200_status rsvd_b200_synth_matrix_device(rsvd_b200_handle* h, size_t rows, size_t cols,
                                               int kind, double beta, uint64_t seed, double* out,
                                               size_t ld) {
    return guarded([&] {
        synth_matrix_impl(h, (long)rows, (long)cols, kind, beta, seed, out, (long)ld, true);
    });
}

rsvd_b200_status rsvd_b200_householder_qr(rsvd_b200_handle* h, const double* a, size_t m,
                                          size_t n, double* q, double* r) {
    return guarded([&] {
        householder_qr_impl(h, a, (long)n, (long)m, (long)n, q, (long)n, r, (long)n, false);
    });
}

rsvd_b200_status rsvd_b200_householder_qr_device(rsvd_b200_handle* h, const double* a, size_t lda,
                                                 size_t m, size_t n, double* q, size_t ldq,
                                                 double* r, size_t ldr) {
    return guarded([&] {
        householder_qr_impl(h, a, (long)lda, (long)m, (long)n, q, (long)ldq, r, (long)ldr, true);
    });
}

rsvd_b200_status rsvd_b200_range_basis(rsvd_b200_handle* h, const double* y, size_t m, size_t s,
                                       double* qout, size_t* cols_out) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        check_shape((long)m, (long)s, "range_basis");
        if (m < s)
            fail(RSVD_B200_DIMENSION_ERROR, "householder_qr needs rows >= cols, got %zux%zu", m, s);
        const Ctx c = begin_run(h, make_plan((long)m, (long)s, (long)s, (long)s), true);
        const int NP = c.p.NP;
        upload(h, h->y, y, (long)m, (long)s, NP);
        // ||y||_F^2 = trace(Y^T Y)
        gemm_atx(h, h->y.d(), (long)m, NP, NP, h->y.d(), NP, NP, c.slot(kG), NP, false);
        std::vector<double> g((size_t)NP * NP);
        download(h, g.data(), c.slot(kG), NP, NP, NP);
        double fro2 = 0.0;
        for (size_t j = 0; j < s; ++j) fro2 += g[j * NP + j];
        const bool fallback = tall_qr(c, h->y.d(), (long)m, h->q.d(), 2, /*materialize=*/true,
                                      /*gram_ready=*/false);
        std::vector<double> qh((size_t)m * s);
        download(h, qh.data(), h->q.d(), (long)m, (long)s, NP);
        std::vector<size_t> keep;
        if (fallback) {  // drop rule on the Householder R (rsvd.cpp:77-86)
            std::vector<double> r((size_t)NP * NP);
            download(h, r.data(), c.slot(kRB), NP, NP, NP);
            const double drop = 1e-13 * std::sqrt(fro2);
            for (size_t j = 0; j < s; ++j)
                if (std::fabs(r[j * NP + j]) > drop) keep.push_back(j);
            if (keep.empty()) keep.push_back(0);
        } else {  // CholeskyQR2 succeeded: every |R_jj| >= 1e-6 max||y_j|| > the drop bound
            for (size_t j = 0; j < s; ++j) keep.push_back(j);
        }
        for (size_t i = 0; i < m; ++i)
            for (size_t j = 0; j < keep.size(); ++j) qout[i * keep.size() + j] = qh[i * s + keep[j]];
        *cols_out = keep.size();
    });
}

rsvd_b200_status rsvd_b200_project_and_solve(rsvd_b200_handle* h, const double* a, size_t m,
                                             size_t n, const double* qb, size_t sq, size_t k,
                                             double* u, double* sigma, double* v,
                                             size_t* sketch_width) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        check_shape((long)m, (long)n, "project_and_solve");
        check_shape((long)m, (long)sq, "project_and_solve basis");
        if (k < 1 || k > sq)
            fail(RSVD_B200_ARGUMENT_ERROR, "rank k=%zu exceeds the basis width %zu", k, sq);
        const long lda = upload(h, h->a_copy, a, (long)m, (long)n, round_up((long)n, 2));
        const Ctx c = begin_run(h, make_plan((long)m, (long)n, lda, (long)sq), true);
        upload(h, h->q, qb, (long)m, (long)sq, c.p.NP);
        h->c_identity = true;
        h->basis = h->q.d();
        h->sig_out.reserve(k * sizeof(double));
        h->u_out.reserve((size_t)m * k * sizeof(double));
        h->v_out.reserve((size_t)n * k * sizeof(double));
        project_and_solve_dev(c, h->a_copy.d(), (long)k, h->u_out.d(), (long)k, h->sig_out.d(),
                              h->v_out.d(), (long)k);
        finish_run(c, false);
        download(h, sigma, h->sig_out.d(), 1, (long)k, (long)k);
        download(h, u, h->u_out.d(), (long)m, (long)k, (long)k);
        download(h, v, h->v_out.d(), (long)n, (long)k, (long)k);
        if (sketch_width) *sketch_width = sq;
    });
}

long rsvd_b200_last_info(rsvd_b200_handle* h, const char* key) {
    if (!strcmp(key, "jacobi_sweeps")) return h->last_sweeps;
    if (!strcmp(key, "householder_fallbacks")) return h->fallbacks;
    if (!strcmp(key, "robust_reruns")) return h->reruns;
    if (!strcmp(key, "launches")) return h->launches;
    if (!strcmp(key, "graph_launches")) return h->graph_replays;
    if (!strcmp(key, "upload_aty_splits")) return h->upload_aty;
    if (!strcmp(key, "oz_passes")) return h->oz_passes;
    if (!strcmp(key, "oz_stored_passes")) return h->oz_stored_passes;
    return -1;
}

void rsvd_b200_set_robust(rsvd_b200_handle* h, int on) { h->force_robust = on != 0; }

void rsvd_b200_set_graphs(rsvd_b200_handle* h, int on) {
    h->use_graphs = on != 0;
    if (!h->use_graphs) h->reset_graphs();
}

rsvd_b200_status rsvd_b200_debug_cholesky(rsvd_b200_handle* h, const double* G, int s, int NP,
                                         double* R, double* RinvT, double tol, int* status) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        if (s < 1 || s > cholesky_max_width() || NP < s)
            fail(RSVD_B200_ARGUMENT_ERROR, "debug_cholesky: s=%d outside [1, %d] or NP < s", s,
                 cholesky_max_width());
        h->red_scratch.reserve(4 * sizeof(double));
        int* st = reinterpret_cast<int*>(h->red_scratch.p);
        h->launched(launch_cholesky(G, NP, s, NP, R, RinvT, st, nullptr, tol, h->stream),
                    "cholesky");
        ck(cudaMemcpyAsync(status, st, sizeof(int), cudaMemcpyDeviceToHost, h->stream),
           "D2H status");
        h->sync();
    });
}

rsvd_b200_status rsvd_b200_debug_jacobi(rsvd_b200_handle* h, const double* R, int s, int NP,
                                       double* sigma, double* U, double* W, int* sweeps) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        if (s < 1 || s > (int)jacobi_max_width() || NP < s)
            fail(RSVD_B200_ARGUMENT_ERROR, "debug_jacobi: s=%d outside [1, %zu] or NP < s", s,
                 jacobi_max_width());
        h->jscratch.reserve(std::max<size_t>(1, jacobi_global_scratch_doubles(s)) * sizeof(double));
        h->red_scratch.reserve(4 * sizeof(double));
        int* st = reinterpret_cast<int*>(h->red_scratch.p);
        h->launched(launch_jacobi_svd(R, s, NP, sigma, U, W, st, h->jscratch.d(), nullptr,
                                      h->stream),
                    "jacobi_svd");
        ck(cudaMemcpyAsync(sweeps, st, sizeof(int), cudaMemcpyDeviceToHost, h->stream),
           "D2H sweeps");
        h->sync();
    });
}

rsvd_b200_status rsvd_b200_debug_gemm_tf32(rsvd_b200_handle* h, int mn, const float* A, long M,
                                          long K, long lda, const float* B, long ldb, int NP,
                                          void* out, long ldo, int out64, int out_t, int splits) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        GemmTf32 g{A, M, K, lda, B, ldb, NP, out, ldo};
        const long brows = mn ? K : NP, bcols = mn ? NP : K;
        h->tf32_tmp.reserve((size_t)std::max(1L, brows * ldb) * sizeof(float));
        h->launched(launch_split_lo(B, brows, bcols, ldb, static_cast<float*>(h->tf32_tmp.p),
                                    h->stream),
                    "split_lo");
        g.Blo = static_cast<float*>(h->tf32_tmp.p);
        g.mn = mn != 0;
        g.out64 = out64 != 0;
        g.out_t = out_t != 0;
        if (splits > 1) {
            const long slab = out_t ? (long)NP * ldo : M * ldo;
            h->part.reserve((size_t)splits * slab * sizeof(double));
            g.out = h->part.p;
            g.splits = splits;
            g.split_stride = slab;
            h->launched(launch_gemm_tf32(g, h->stream), "gemm_tf32(split)");
            h->launched(launch_reduce_partials(h->part.d(), slab, splits, (double*)out, slab,
                                               h->stream),
                        "reduce_partials");
        } else {
            h->launched(launch_gemm_tf32(g, h->stream), "gemm_tf32");
        }
        h->sync();
    });
}

rsvd_b200_status rsvd_b200_debug_gemm_oz(rsvd_b200_handle* h, int mn, const double* A, long M,
                                        long K, long lda, const double* B, long ldb, int NP,
                                        int cols, double* out, long ldo, int out_t, int splits) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        // A's scales: per row (ax, A is M x K) or per column (atx, A is K x M)
        const long arows = mn ? K : M, acols = mn ? M : K;
        h->oz_ef.reserve((size_t)(arows + acols + 2 * NP + 8) * sizeof(int));
        int* row_ef = static_cast<int*>(h->oz_ef.p);
        int* col_ef = row_ef + arows;
        int* b_ef = col_ef + acols;
        int* scratch = b_ef + NP;
        h->oz_part.reserve(oz_scan_part_ints(arows, acols) * sizeof(int));
        h->launched(launch_oz_scan(A, arows, acols, lda, row_ef, col_ef,
                                   static_cast<int*>(h->oz_part.p), nullptr, h->stream),
                    "oz_scan");
        h->oz_bdig.reserve(oz_digits_bytes(NP, K));
        uint8_t* dig = static_cast<uint8_t*>(h->oz_bdig.p);
        if (mn)
            h->launched(launch_oz_digits_cols(B, ldb, NP, cols, K, dig, b_ef, scratch, h->stream),
                        "oz_digits_cols");
        else
            h->launched(launch_oz_digits_rows(B, ldb, NP, cols, K, dig, b_ef, h->stream),
                        "oz_digits_rows");
        GemmOz g;
        g.mn = mn != 0;
        g.A = A, g.M = M, g.K = K, g.lda = lda;
        g.a_ef = mn ? col_ef : row_ef;
        g.bdig = dig, g.ldb = oz_ldb(K), g.b_ef = b_ef, g.NP = NP;
        g.out = out, g.ldo = ldo, g.out_t = out_t != 0;
        if (splits > 1) {
            const long slab = out_t ? (long)NP * ldo : M * ldo;
            h->part.reserve((size_t)splits * slab * sizeof(double));
            g.out = h->part.d();
            g.splits = splits;
            g.split_stride = slab;
            h->launched(launch_gemm_oz(g, h->stream), "gemm_oz(split)");
            h->launched(launch_reduce_partials(h->part.d(), slab, splits, out, slab, h->stream),
                        "reduce_partials");
        } else {
            h->launched(launch_gemm_oz(g, h->stream), "gemm_oz");
        }
        h->sync();
    });
}

rsvd_b200_status rsvd_b200_debug_gemm_ozd(rsvd_b200_handle* h, int mn, const double* A, long M,
                                         long K, long lda, const double* B, long ldb, int NP,
                                         int cols, double* out, long ldo, int out_t, int splits) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        // A as stored: arows x acols (ax: M x K; atx: K x M), row-scaled digit planes
        const long arows = mn ? K : M, acols = mn ? M : K;
        const size_t tb = oz_tiled_bytes(arows, acols);
        h->oz_adig.reserve(2 * tb);
        h->oz_ef.reserve((size_t)(arows + acols + 2 * NP + 8) * sizeof(int));
        int* row_ef = static_cast<int*>(h->oz_ef.p);
        int* col_ef = row_ef + arows;
        int* b_ef = col_ef + acols;
        int* scratch = b_ef + NP;
        uint8_t* dax = static_cast<uint8_t*>(h->oz_adig.p);
        uint8_t* datx = dax + tb;
        h->oz_part.reserve(oz_scan_part_ints(arows, acols) * sizeof(int));
        h->launched(launch_oz_scan(A, arows, acols, lda, row_ef, col_ef,
                                   static_cast<int*>(h->oz_part.p), nullptr, h->stream, false),
                    "oz_scan");
        h->launched(launch_oz_convert_tiles(A, 0, arows, arows, acols, lda, dax, datx, row_ef,
                                            h->stream),
                    "oz_convert_tiles");
        int nch, nf;
        oz_chunks(NP, &nch, &nf);
        h->oz_bdig.reserve(oz_digits_bytes(NP, K));
        uint8_t* dig = static_cast<uint8_t*>(h->oz_bdig.p);
        if (mn)
            h->launched(launch_oz_digits_cols(B, ldb, NP, cols, K, dig, b_ef, scratch, h->stream,
                                              row_ef, nf),
                        "oz_digits_cols");
        else
            h->launched(launch_oz_digits_rows(B, ldb, NP, cols, K, dig, b_ef, h->stream, nf),
                        "oz_digits_rows");
        GemmOzd g;
        g.mn = mn != 0;
        g.adig = mn ? datx : dax;
        g.a_inner = mn ? (acols + 127) / 128 : (acols + 31) / 32;
        g.M = M, g.K = K;
        g.a_ef = row_ef;
        g.bdig = dig, g.b_ef = b_ef, g.NP = NP;
        g.out = out, g.ldo = ldo, g.out_t = out_t != 0;
        if (splits > 1) {
            const long slab = out_t ? (long)NP * ldo : M * ldo;
            h->part.reserve((size_t)splits * slab * sizeof(double));
            g.out = h->part.d();
            g.splits = splits;
            g.split_stride = slab;
            h->launched(launch_gemm_ozd(g, h->stream), "gemm_ozd(split)");
            h->launched(launch_reduce_partials(h->part.d(), slab, splits, out, slab, h->stream),
                        "reduce_partials");
        } else {
            h->launched(launch_gemm_ozd(g, h->stream), "gemm_ozd");
        }
        h->sync();
    });
}

rsvd_b200_status rsvd_b200_residual_fro_device(rsvd_b200_handle* h, const double* a_dev,
                                              size_t m, size_t n, size_t lda,
                                              const double* u_dev, const double* sigma_dev,
                                              const double* v_dev, size_t k, double* out) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        if (m < 1 || n < 1 || k < 1)
            fail(RSVD_B200_DIMENSION_ERROR, "residual_fro: empty operands");
        // A is read with plain loads in the epilogue: any lda works
        *out = residual_device(h, a_dev, (long)m, (long)n, (long)lda, u_dev, (long)k, sigma_dev,
                               v_dev, (long)k, (long)k);
    });
}

rsvd_b200_status rsvd_b200_residual_fro(rsvd_b200_handle* h, const double* a, size_t m, size_t n,
                                       const double* u, const double* sigma, const double* v,
                                       size_t k, double* out) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        if (m < 1 || n < 1 || k < 1)
            fail(RSVD_B200_DIMENSION_ERROR, "residual_fro: empty operands");
        h->a_copy.reserve(m * n * sizeof(double));
        ck(cudaMemcpyAsync(h->a_copy.p, a, m * n * sizeof(double), cudaMemcpyHostToDevice,
                           h->stream),
           "H2D of A");
        h->u_out.reserve(m * k * sizeof(double));
        h->v_out.reserve(n * k * sizeof(double));
        h->sig_out.reserve(k * sizeof(double));
        ck(cudaMemcpyAsync(h->u_out.p, u, m * k * sizeof(double), cudaMemcpyHostToDevice,
                           h->stream),
           "H2D of U");
        ck(cudaMemcpyAsync(h->v_out.p, v, n * k * sizeof(double), cudaMemcpyHostToDevice,
                           h->stream),
           "H2D of V");
        ck(cudaMemcpyAsync(h->sig_out.p, sigma, k * sizeof(double), cudaMemcpyHostToDevice,
                           h->stream),
           "H2D of sigma");
        *out = residual_device(h, h->a_copy.d(), (long)m, (long)n, (long)n, h->u_out.d(),
                               (long)k, h->sig_out.d(), h->v_out.d(), (long)k, (long)k);
    });
}

// ------------------------------------------------------------------- PCA (§8f)
rsvd_b200_status rsvd_b200_fit_pca(rsvd_b200_handle* h, const double* x, size_t N, size_t d,
                                   size_t k, const rsvd_b200_config* cfg, double* mean,
                                   double* components, double* explained_variance) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        h->launches = 0;
        if (N < 2) fail(RSVD_B200_ARGUMENT_ERROR, "center_columns needs at least 2 rows, got %zu", N);
        if (k < 1 || k > std::min(N, d))
            fail(RSVD_B200_ARGUMENT_ERROR, "fit_pca k=%zu outside [1, %zu]", k, std::min(N, d));
        const long ld = round_up((long)d, 2);
        h->a_copy.reserve((size_t)N * ld * sizeof(double));
        ck(cudaMemcpy2DAsync(h->a_copy.p, ld * sizeof(double), x, d * sizeof(double),
                             d * sizeof(double), N, cudaMemcpyHostToDevice, h->stream),
           "H2D of X");
        pca_center(h, h->a_copy.d(), (long)N, (long)d, ld, h->a_copy.d(), ld);
        rsvd_b200_config c = *cfg;
        c.k = k;
        h->sig_out.reserve(k * sizeof(double));
        h->v_out.reserve((size_t)d * k * sizeof(double));
        solve_device(h, h->a_copy.d(), (long)N, (long)d, ld, c, nullptr, h->sig_out.d(),
                     h->v_out.d(), nullptr);
        std::vector<double> sig(k);
        ck(cudaMemcpyAsync(sig.data(), h->sig_out.p, k * sizeof(double), cudaMemcpyDeviceToHost,
                           h->stream),
           "D2H sigma");
        ck(cudaMemcpyAsync(components, h->v_out.p, d * k * sizeof(double),
                           cudaMemcpyDeviceToHost, h->stream),
           "D2H components");
        ck(cudaMemcpyAsync(mean, h->pca_mean.p, d * sizeof(double), cudaMemcpyDeviceToHost,
                           h->stream),
           "D2H mean");
        h->sync();
        const double denom = (double)(N - 1);  // pca.cpp:36-38
        for (size_t i = 0; i < k; ++i) explained_variance[i] = sig[i] * sig[i] / denom;
    });
}

rsvd_b200_status rsvd_b200_pca_transform(rsvd_b200_handle* h, const double* x, size_t N,
                                         size_t d, const double* mean, const double* components,
                                         size_t k, double* out) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        if (N < 1 || d < 1 || k < 1 || k > d)
            fail(RSVD_B200_DIMENSION_ERROR, "transform: %zu components for %zu features", k, d);
        cudaStream_t st = h->stream;
        const long ld = round_up((long)d, 2);
        h->a_copy.reserve((size_t)N * ld * sizeof(double));
        ck(cudaMemcpy2DAsync(h->a_copy.p, ld * sizeof(double), x, d * sizeof(double),
                             d * sizeof(double), N, cudaMemcpyHostToDevice, st),
           "H2D of X");
        h->pca_mean.reserve(d * sizeof(double));
        h->pca_comp.reserve((size_t)d * k * sizeof(double));
        ck(cudaMemcpyAsync(h->pca_mean.p, mean, d * sizeof(double), cudaMemcpyHostToDevice, st),
           "H2D mean");
        ck(cudaMemcpyAsync(h->pca_comp.p, components, d * k * sizeof(double),
                           cudaMemcpyHostToDevice, st),
           "H2D components");
        h->launched(launch_center(h->a_copy.d(), ld, (long)N, (long)d, nullptr, h->pca_mean.d(),
                                  h->a_copy.d(), ld, nullptr, st),
                    "center");
        // (X - mean) components: ax with Xt = components^T (NPk x d, zero padded)
        const int NPk = pad_np((long)k);
        h->ubt.reserve((size_t)NPk * ld * sizeof(double));
        h->launched(launch_fill(h->ubt.d(), (long)NPk * ld, 0.0, st), "fill");
        h->launched(launch_transpose(h->pca_comp.d(), (long)d, (long)k, (long)k, h->ubt.d(), ld, st),
                    "transpose");
        const long tiles = ax_tiles((long)N, NPk);
        const int sp = choose_splits(tiles, (ld + 31) / 32);
        h->part.reserve((size_t)std::max(1, sp) * N * NPk * sizeof(double));
        h->y.reserve((size_t)N * NPk * sizeof(double));
        gemm_ax(h, h->a_copy.d(), (long)N, (long)d, ld, h->ubt.d(), ld, NPk, h->y.d(), NPk);
        ck(cudaMemcpy2DAsync(out, k * sizeof(double), h->y.p, NPk * sizeof(double),
                             k * sizeof(double), N, cudaMemcpyDeviceToHost, st),
           "D2H projection");
        h->sync();
    });
}

rsvd_b200_status rsvd_b200_dmma_peak(rsvd_b200_handle* h, double* tflops) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        ck(measure_dmma_peak(h->stream, tflops), "DMMA peak probe");
    });
}

rsvd_b200_status rsvd_b200_imma_peak(rsvd_b200_handle* h, double* tops) {
    return guarded([&] {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        ck(measure_imma_peak(h->stream, tops), "INT8 tensor peak probe");
    });
}

}  // extern "C"
