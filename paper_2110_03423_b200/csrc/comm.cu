// Reduction transports of the row-sharded rSVD (see comm.h).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "comm.h"

namespace rsvdb200 {

// ------------------------------------------------------------ local group
struct BufList {
    const double* p[16];
};

__global__ void sum_buffers_kernel(BufList bl, int nbuf, size_t count, double* __restrict__ out) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count;
         e += (size_t)gridDim.x * blockDim.x) {
        double acc = bl.p[0][e];
        for (int r = 1; r < nbuf; ++r) acc += bl.p[r][e];
        out[e] = acc;
    }
}

cudaError_t launch_sum_buffers(const double* const* bufs, int nbuf, size_t count, double* out,
                               cudaStream_t st) {
    if (nbuf < 1 || nbuf > 16) return cudaErrorInvalidValue;
    BufList bl{};
    for (int r = 0; r < nbuf; ++r) bl.p[r] = bufs[r];
    size_t blocks = (count + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    sum_buffers_kernel<<<(unsigned)blocks, 256, 0, st>>>(bl, nbuf, count, out);
    return cudaGetLastError();
}

__global__ void flags_pack_kernel(const int* flags, int i0, int i1, double* out) {
    if (threadIdx.x == 0) {
        out[0] = (double)flags[i0];
        out[1] = (double)flags[i1];
    }
}

__global__ void flags_unpack_kernel(const double* in, int* flags, int i0, int i1) {
    if (threadIdx.x == 0) {
        flags[i0] = in[0] != 0.0;
        flags[i1] = in[1] != 0.0;
    }
}

cudaError_t launch_flags_pack(const int* flags, int i0, int i1, double* out, cudaStream_t st) {
    flags_pack_kernel<<<1, 32, 0, st>>>(flags, i0, i1, out);
    return cudaGetLastError();
}

cudaError_t launch_flags_unpack(const double* in, int* flags, int i0, int i1, cudaStream_t st) {
    flags_unpack_kernel<<<1, 32, 0, st>>>(in, flags, i0, i1);
    return cudaGetLastError();
}

namespace {

std::string cuda_msg(cudaError_t e, const char* what) {
    return std::string(what) + ": " + cudaGetErrorString(e);
}

// Every rank publishes its buffer, sums all ranks' buffers (rank order) into its own
// scratch, and copies the sum back once every rank has finished reading.
class LocalGroupComm final : public Comm {
   public:
    LocalGroupComm(LocalGroup* g, int r) : g_(g) {
        rank = r;
        world = g->world;
    }
    ~LocalGroupComm() override {
        if (scratch_) cudaFree(scratch_);
    }
    const char* kind() const override { return "local"; }

    std::string allreduce_sum(double* buf, size_t count, cudaStream_t st) override {
        if (count == 0) return "";
        // Every rank takes part in both barriers whatever happens locally (a rank that
        // returned early would leave the others blocked forever); failures are published in
        // the group and every rank reports the collective as failed after the barrier.
        std::string err;
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) err = cuda_msg(e, "local allreduce: stream sync");
        if (err.empty() && count > cap_) {
            if (scratch_) cudaFree(scratch_);
            scratch_ = nullptr;
            cap_ = 0;
            e = cudaMalloc(&scratch_, count * sizeof(double));
            if (e != cudaSuccess) err = cuda_msg(e, "local allreduce: scratch");
            else cap_ = count;
        }
        if (!err.empty()) g_->failed.fetch_add(1);
        g_->ptrs[rank] = buf;
        g_->bar.arrive_and_wait();  // every buffer is complete and published (or a rank failed)
        const bool group_ok = g_->failed.load() == 0;
        if (group_ok) {
            e = launch_sum_buffers(g_->ptrs.data(), world, count, scratch_, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) err = cuda_msg(e, "local allreduce: sum");
        }
        g_->bar.arrive_and_wait();  // every rank has read every buffer
        if (!group_ok) {
            if (rank == 0) g_->failed.store(0);  // reset for the next call (all ranks read it)
            g_->bar.arrive_and_wait();
            return err.empty() ? "local allreduce: another rank of the group failed" : err;
        }
        if (!err.empty()) return err;
        e = cudaMemcpyAsync(buf, scratch_, count * sizeof(double), cudaMemcpyDeviceToDevice, st);
        return e == cudaSuccess ? "" : cuda_msg(e, "local allreduce: copy back");
    }

   private:
    LocalGroup* g_;
    double* scratch_ = nullptr;
    size_t cap_ = 0;
};

// ------------------------------------------------------------------- NCCL
// Resolved from the libnccl.so.2 already loaded in the process (torch's), else the
// system library, so one NCCL serves both torch.distributed and the solver.
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                               ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*comm_async_error)(ncclComm_t, ncclResult_t*) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.error = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
        api.comm_init_rank =
            reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
        api.comm_async_error =
            reinterpret_cast<decltype(api.comm_async_error)>(sym("ncclCommGetAsyncError"));
        api.error_string =
            reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
        if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy ||
            !api.error_string)
            api.error = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

std::string nccl_msg(ncclResult_t r, const char* what) {
    return std::string(what) + ": " + nccl().error_string(r);
}

class NcclComm final : public Comm {
   public:
    NcclComm(ncclComm_t c, int r, int w) : comm_(c) {
        rank = r;
        world = w;
    }
    ~NcclComm() override {
        if (comm_) nccl().comm_destroy(comm_);
    }
    const char* kind() const override { return "nccl"; }
    bool capturable() const override { return true; }
    std::string allreduce_sum(double* buf, size_t count, cudaStream_t st) override {
        if (count == 0) return "";
        const ncclResult_t r =
            nccl().all_reduce(buf, buf, count, ncclFloat64, ncclSum, comm_, st);
        return r == ncclSuccess ? "" : nccl_msg(r, "ncclAllReduce");
    }

   private:
    ncclComm_t comm_ = nullptr;
};

}  // namespace

std::unique_ptr<Comm> make_local_comm(LocalGroup* g, int rank) {
    return std::make_unique<LocalGroupComm>(g, rank);
}

std::string nccl_unique_id(unsigned char out[128]) {
    const NcclApi& api = nccl();
    if (!api.error.empty()) return api.error;
    ncclUniqueId id;
    const ncclResult_t r = api.get_unique_id(&id);
    if (r != ncclSuccess) return nccl_msg(r, "ncclGetUniqueId");
    std::memcpy(out, id.internal, 128);
    return "";
}

std::string make_nccl_comm(const unsigned char id[128], int rank, int world,
                           std::unique_ptr<Comm>* out) {
    const NcclApi& api = nccl();
    if (!api.error.empty()) return api.error;
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, 128);
    ncclComm_t c = nullptr;
    const ncclResult_t r = api.comm_init_rank(&c, world, uid, rank);
    if (r != ncclSuccess) return nccl_msg(r, "ncclCommInitRank");
    *out = std::make_unique<NcclComm>(c, rank, world);
    return "";
}

}  // namespace rsvdb200
