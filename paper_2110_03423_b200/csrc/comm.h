// Reduction transport of the row-sharded rSVD.
//
// A is row-sharded across the ranks; the only data that crosses ranks are the
// natural sums of Algorithm 1 over the row dimension m:
//   * the s x s Gram Y_g^T Y_g of every CholeskyQR pass,
//   * the n x s partials (A_g^T Q_g)^T of the power iteration and Q_g^T A_g of B,
//   * the stacked R factors of the TSQR Householder fallback,
//   * the status flags (NaN/Inf seen in any shard, abort) at the end of a solve.
// All of them are in-place sum all-reduces of FP64 device buffers enqueued on the
// solver's stream. Two transports implement it:
//   * NcclComm      — NCCL (dlopen'ed: the libnccl.so.2 already in the process,
//                     e.g. torch's, else the system one) over NVLink / NVSwitch;
//   * LocalGroupComm — an in-process group of handles (threads) whose buffers are
//                     mutually addressable (same device or P2P); it sums the ranks'
//                     buffers in fixed rank order with a device kernel. It makes the
//                     sharded pipeline testable on one GPU.
// Both give every rank bit-identical sums, so the replicated small factorisations
// (Cholesky, Jacobi) take identical branches on every rank.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include <atomic>
#include <barrier>
#include <memory>
#include <string>
#include <vector>

namespace rsvdb200 {

class Comm {
   public:
    virtual ~Comm() = default;
    // In-place sum over ranks of `count` doubles at device pointer `buf`, ordered on
    // `st`. Returns an empty string on success, else the error text.
    virtual std::string allreduce_sum(double* buf, size_t count, cudaStream_t st) = 0;
    virtual const char* kind() const = 0;
    // allreduce_sum may be recorded into a CUDA graph (stream capture)
    virtual bool capturable() const { return false; }
    int rank = 0, world = 1;
};

// NCCL unique id (128 bytes) for rank 0 to broadcast out of band.
std::string nccl_unique_id(unsigned char out[128]);
// Communicator on the current device; "" on success.
std::string make_nccl_comm(const unsigned char id[128], int rank, int world,
                           std::unique_ptr<Comm>* out);

struct LocalGroup {
    explicit LocalGroup(int w) : world(w), bar(w), ptrs(w, nullptr), failed(0) {}
    int world;
    std::barrier<> bar;
    std::vector<double*> ptrs;
    std::atomic<int> failed;  // ranks whose local step failed in the current all-reduce
};

std::unique_ptr<Comm> make_local_comm(LocalGroup* g, int rank);

// Sharded status flags: out[0..1] = (double)flags[i0], (double)flags[i1]; and back,
// flags[i] = (in[.] != 0) after the sum all-reduce (an OR over the ranks).
cudaError_t launch_flags_pack(const int* flags, int i0, int i1, double* out, cudaStream_t st);
cudaError_t launch_flags_unpack(const double* in, int* flags, int i0, int i1, cudaStream_t st);

// out[e] = sum_{r < nbuf} bufs[r][e], fixed order (up to 16 buffers).
cudaError_t launch_sum_buffers(const double* const* bufs, int nbuf, size_t count, double* out,
                               cudaStream_t st);

}  // namespace rsvdb200
