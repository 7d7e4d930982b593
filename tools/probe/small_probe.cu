// Microbenchmark of the single-CTA small-side kernels (not part of the library):
// per-phase clock64 trace of the Cholesky kernel and event timings.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DCHOL_TRACE \
//        -I paper_2110_03423_b200/csrc tools/probe/small_probe.cu -o /tmp/small_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "../../paper_2110_03423_b200/csrc/linalg_small.cu"
#include "../../paper_2110_03423_b200/csrc/linalg_blocked.cu"

using namespace rsvdb200;

// R = triangular factor of U diag(sigma) V^T (U, V Haar via modified Gram-Schmidt), sigma_i =
// exp(-i / tau): the shape of the R_B the pipeline hands to the Jacobi SVD.
static std::vector<double> graded_r(int s, double tau) {
    std::vector<double> U(s * s), V(s * s), A(s * s, 0.0);
    auto haar = [&](std::vector<double>& Q) {
        for (auto& v : Q) {
            double u1 = (rand() + 1.0) / (RAND_MAX + 2.0), u2 = rand() / (RAND_MAX + 1.0);
            v = sqrt(-2 * log(u1)) * cos(6.283185307179586 * u2);
        }
        for (int j = 0; j < s; ++j) {  // columns j orthonormal
            for (int k = 0; k < j; ++k) {
                double d = 0;
                for (int i = 0; i < s; ++i) d += Q[i * s + j] * Q[i * s + k];
                for (int i = 0; i < s; ++i) Q[i * s + j] -= d * Q[i * s + k];
            }
            double n = 0;
            for (int i = 0; i < s; ++i) n += Q[i * s + j] * Q[i * s + j];
            n = sqrt(n);
            for (int i = 0; i < s; ++i) Q[i * s + j] /= n;
        }
    };
    haar(U);
    haar(V);
    for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j)
            for (int k = 0; k < s; ++k) A[i * s + j] += U[i * s + k] * exp(-k / tau) * V[j * s + k];
    // R from modified Gram-Schmidt QR of A (columns)
    std::vector<double> R(s * s, 0.0);
    for (int j = 0; j < s; ++j) {
        for (int k = 0; k < j; ++k) {
            double d = 0;
            for (int i = 0; i < s; ++i) d += A[i * s + j] * A[i * s + k];
            R[k * s + j] = d;
            for (int i = 0; i < s; ++i) A[i * s + j] -= d * A[i * s + k];
        }
        double n = 0;
        for (int i = 0; i < s; ++i) n += A[i * s + j] * A[i * s + j];
        n = sqrt(n);
        R[j * s + j] = n;
        for (int i = 0; i < s; ++i) A[i * s + j] /= n;
    }
    return R;
}

static void jacobi_probe(int s, bool transposed) {
    const int NP = (s + 15) / 16 * 16;
    srand(7);
    std::vector<double> R = graded_r(s, s / 8.0), Rp(NP * NP, 0.0);
    for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j) Rp[i * NP + j] = transposed ? R[j * s + i] : R[i * s + j];
    double *dR, *sig, *U, *W, *scr;
    int* st;
    cudaMalloc(&dR, NP * NP * 8);
    cudaMalloc(&sig, NP * 8);
    cudaMalloc(&U, NP * NP * 8);
    cudaMalloc(&W, NP * NP * 8);
    cudaMalloc(&scr, jacobi_global_scratch_doubles(s) * 8);
    cudaMalloc(&st, 16);
    cudaMemcpy(dR, Rp.data(), NP * NP * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch_jacobi_svd(dR, s, NP, sig, U, W, st, scr, nullptr, 0);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int i = 0; i < reps; ++i) launch_jacobi_svd(dR, s, NP, sig, U, W, st, scr, nullptr, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int sweeps;
    cudaMemcpy(&sweeps, st, 4, cudaMemcpyDeviceToHost);
    std::vector<double> sg(NP);
    cudaMemcpy(sg.data(), sig, NP * 8, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < s; ++i) err = fmax(err, fabs(sg[i] - exp(-i / (s / 8.0))) / exp(-i / (s / 8.0)));
    const int rounds = ((s + 1) & ~1) - 1;
#ifdef JAC_TRACE
    if (s <= 112) {
        int zero = 0, nt = 0;
        long long tr[1024];
        cudaMemcpyToSymbol(g_jac_ntrace, &zero, 4);
        launch_jacobi_svd(dR, s, NP, sig, U, W, st, scr, nullptr, 0);
        cudaDeviceSynchronize();
        cudaMemcpyFromSymbol(&nt, g_jac_ntrace, 4);
        cudaMemcpyFromSymbol(tr, g_jac_trace, sizeof(tr));
        long long sums[8] = {}, cnt[8] = {};
        for (int i = 1; i < nt; ++i) {
            sums[tr[2 * i]] += tr[2 * i + 1] - tr[2 * i - 1];
            cnt[tr[2 * i]] += 1;
        }
        const char* nm[] = {"sync->next", "load+dots", "shuffles", "rotation|send", "update|wait", "rot", "sync"};
        for (int t = 0; t < 7; ++t)
            if (cnt[t]) printf("   %-12s %8lld cycles avg over %lld\n", nm[t], sums[t] / cnt[t], cnt[t]);
    }
#endif
#ifdef BJ_TRACE
    {
        int zero = 0, nt = 0;
        long long tr[512];
        cudaMemcpyToSymbol(g_bj_ntrace, &zero, 4);
        launch_jacobi_svd(dR, s, NP, sig, U, W, st, scr, nullptr, 0);
        cudaDeviceSynchronize();
        cudaMemcpyFromSymbol(&nt, g_bj_ntrace, 4);
        cudaMemcpyFromSymbol(tr, g_bj_trace, sizeof(tr));
        long long sums[8] = {}, cnt[8] = {};
        for (int i = 1; i < nt; ++i) {
            sums[tr[2 * i]] += tr[2 * i + 1] - tr[2 * i - 1];
            cnt[tr[2 * i]] += 1;
        }
        const char* nm[] = {"sync->setup", "load", "inner", "store+or", "grid.sync"};
        for (int t = 0; t < 5; ++t)
            if (cnt[t]) printf("   %-12s %8lld cycles avg over %lld\n", nm[t], sums[t] / cnt[t], cnt[t]);
    }
#endif
    printf("jacobi%s s=%d: %.1f us, %d sweeps, %.0f cycles/round (at 1.9 GHz), max rel sigma err %.1e\n",
           transposed ? "(R^T)" : "", s, ms * 1000 / reps, sweeps, ms * 1e-3 / reps * 1.9e9 / (sweeps * rounds), err);
}

int main(int argc, char** argv) {
    if (argc > 1) {
        for (int i = 1; i < argc; ++i) {
            jacobi_probe(atoi(argv[i]), false);
            jacobi_probe(atoi(argv[i]), true);
        }
        return 0;
    }
    const int sizes[] = {74, 136, 148};
    for (int s : sizes) {
        const int NP = (s + 15) / 16 * 16;
        // SPD: G = M^T M + s I
        std::vector<double> M(s * s), G(NP * NP, 0.0);
        srand(1);
        for (auto& v : M) v = rand() / (double)RAND_MAX - 0.5;
        for (int i = 0; i < s; ++i)
            for (int j = 0; j < s; ++j) {
                double acc = (i == j) ? s : 0.0;
                for (int k = 0; k < s; ++k) acc += M[k * s + i] * M[k * s + j];
                G[i * NP + j] = acc;
            }
        double *dG, *dR, *dRi;
        int* dst;
        cudaMalloc(&dG, NP * NP * 8);
        cudaMalloc(&dR, NP * NP * 8);
        cudaMalloc(&dRi, NP * NP * 8);
        cudaMalloc(&dst, 16);
        cudaMemcpy(dG, G.data(), NP * NP * 8, cudaMemcpyHostToDevice);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int it = 0; it < 3; ++it)
            launch_cholesky(dG, NP, s, NP, dR, dRi, dst, nullptr, 1e-14, 0);
        const int reps = 20;
        cudaEventRecord(e0);
        for (int it = 0; it < reps; ++it)
            launch_cholesky(dG, NP, s, NP, dR, dRi, dst, nullptr, 1e-14, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        int n = 0;
        long long tr[256] = {};
#ifdef CHOL_TRACE
        int zero = 0;
        cudaMemcpyToSymbol(g_chol_ntrace, &zero, 4);
        launch_cholesky(dG, NP, s, NP, dR, dRi, dst, nullptr, 1e-14, 0);
        cudaDeviceSynchronize();
        cudaMemcpyFromSymbol(&n, g_chol_ntrace, 4);
        cudaMemcpyFromSymbol(tr, g_chol_trace, sizeof(tr));
#endif
        // check: R^T R = G, R * RinvT^T = I
        std::vector<double> R(NP * NP), Ri(NP * NP);
        cudaMemcpy(R.data(), dR, NP * NP * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(Ri.data(), dRi, NP * NP * 8, cudaMemcpyDeviceToHost);
        double e1m = 0, e2m = 0;
        for (int i = 0; i < s; ++i)
            for (int j = 0; j < s; ++j) {
                double a = 0, b = 0;
                for (int k = 0; k < s; ++k) {
                    a += R[k * NP + i] * R[k * NP + j];
                    b += R[i * NP + k] * Ri[j * NP + k];
                }
                e1m = fmax(e1m, fabs(a - G[i * NP + j]) / G[0]);
                e2m = fmax(e2m, fabs(b - (i == j)));
            }
        printf("s=%d  %.2f us/launch  |RtR-G|/G00=%.2e |R Rinv - I|=%.2e\n", s, ms * 1000 / reps,
               e1m, e2m);
        const char* names[] = {"load", "-", "trsm", "diag+syrk", "-", "inv_diag", "inv_upd",
                               "out", "dg_load", "dg_pivots", "dg_tail"};
        long long prev = tr[1];
        long long sums[16] = {};
        for (int i = 1; i < n; ++i) {
            sums[tr[2 * i]] += tr[2 * i + 1] - prev;
            prev = tr[2 * i + 1];
        }
        for (int t = 1; t < 11; ++t) printf("   %-9s %8lld cycles\n", names[t], sums[t]);
        printf("   total    %8lld cycles (from load end)\n", prev - tr[1]);
        cudaFree(dG);
        cudaFree(dR);
        cudaFree(dRi);
        cudaFree(dst);
    }
    return 0;
}
