// DMAT interchange files (reference: include/randsvd/dmat.hpp:10-19, src/dmat.cpp:17-99):
// "DMAT1\n", rows and cols as u64 little-endian, then rows*cols binary64 little-endian
// values in row-major order, nothing else.
//
//  * randsvd::read_dmat / write_dmat — the drop-in API (same errors: IoError with the
//    byte offset of the failure), reading the payload straight into the DenseMatrix
//    storage instead of through a second raw copy (dmat.cpp:54-55 holds 2x the matrix).
//  * rsvd_b200_load_dmat_device — the B200 loader: a row range of the file (one rank's
//    shard) is streamed into HBM through two pinned staging buffers, the file read of one
//    chunk overlapping the host-to-device copy of the previous one, so loading runs at
//    min(disk, PCIe) bandwidth without ever holding the matrix in pageable memory.
#include <cuda_runtime.h>

#include <bit>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "../../include/randsvd/dmat.hpp"
#include "../../include/randsvd/errors.hpp"
#include "../../include/rsvd_b200.h"

static_assert(std::endian::native == std::endian::little, "DMAT payloads are little-endian");

namespace randsvd {

namespace {

constexpr char kMagic[6] = {'D', 'M', 'A', 'T', '1', '\n'};

std::uint64_t get_u64_le(const char* buf) {
    std::uint64_t v = 0;
    for (int i = 0; i < 8; ++i)
        v |= static_cast<std::uint64_t>(static_cast<unsigned char>(buf[i])) << (8 * i);
    return v;
}

void put_u64_le(std::ostream& out, std::uint64_t v) {
    char buf[8];
    for (int i = 0; i < 8; ++i) buf[i] = static_cast<char>((v >> (8 * i)) & 0xFF);
    out.write(buf, 8);
}

// Header check shared by the stream reader and the device loader (dmat.cpp:36-52).
void read_header(std::istream& in, const std::string& name, std::uint64_t& rows,
                 std::uint64_t& cols) {
    char magic[6];
    in.read(magic, 6);
    if (in.gcount() != 6 || std::memcmp(magic, kMagic, 6) != 0)
        throw IoError("bad DMAT magic in " + name + " at byte offset 0", name, 0);
    char header[16];
    in.read(header, 16);
    if (in.gcount() != 16)
        throw IoError("truncated DMAT header in " + name + " at byte offset " +
                          std::to_string(6 + in.gcount()),
                      name, 6 + static_cast<std::uint64_t>(in.gcount()));
    rows = get_u64_le(header);
    cols = get_u64_le(header + 8);
    if (rows == 0 || cols == 0 || rows > (1ULL << 32) || cols > (1ULL << 32))
        throw IoError("implausible DMAT dimensions " + std::to_string(rows) + "x" +
                          std::to_string(cols) + " in " + name,
                      name, 6);
}

}  // namespace

DenseMatrix read_dmat(std::istream& in, const std::string& name) {
    std::uint64_t rows = 0, cols = 0;
    read_header(in, name, rows, cols);
    std::vector<double> data(rows * cols);
    const std::uint64_t bytes = rows * cols * 8;
    in.read(reinterpret_cast<char*>(data.data()), static_cast<std::streamsize>(bytes));
    if (static_cast<std::uint64_t>(in.gcount()) != bytes) {
        const std::uint64_t off = 22 + static_cast<std::uint64_t>(in.gcount());
        throw IoError("truncated DMAT payload in " + name + " at byte offset " +
                          std::to_string(off) + " (expected " + std::to_string(22 + bytes) +
                          " bytes total)",
                      name, off);
    }
    if (in.peek() != std::char_traits<char>::eof())
        throw IoError("trailing bytes in " + name + " after byte offset " +
                          std::to_string(22 + bytes),
                      name, 22 + bytes);
    return DenseMatrix(rows, cols, std::move(data));
}

void write_dmat(std::ostream& out, const DenseMatrix& m, const std::string& name) {
    out.write(kMagic, 6);
    put_u64_le(out, m.rows());
    put_u64_le(out, m.cols());
    out.write(reinterpret_cast<const char*>(m.data().data()),
              static_cast<std::streamsize>(m.size() * 8));
    if (!out) throw IoError("write failure on " + name, name, 0);
}

DenseMatrix read_dmat(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path, path, 0);
    return read_dmat(in, path);
}

void write_dmat(const std::string& path, const DenseMatrix& m) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw IoError("cannot create " + path, path, 0);
    write_dmat(out, m, path);
}

}  // namespace randsvd

// ================================================================== C-ABI loader
namespace {
thread_local std::string g_dmat_error;
}

extern "C" {

const char* rsvd_b200_dmat_last_error(void) { return g_dmat_error.c_str(); }

int rsvd_b200_dmat_shape(const char* path, uint64_t* rows, uint64_t* cols) {
    try {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw randsvd::IoError(std::string("cannot open ") + path, path, 0);
        randsvd::read_header(in, path, *rows, *cols);
        return 0;
    } catch (const std::exception& e) {
        g_dmat_error = e.what();
        return 7;
    }
}

int rsvd_b200_load_dmat_device(rsvd_b200_handle* h, const char* path, uint64_t row0,
                               uint64_t nrows, double* a_dev, size_t lda) {
    try {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw randsvd::IoError(std::string("cannot open ") + path, path, 0);
        uint64_t rows = 0, cols = 0;
        randsvd::read_header(in, path, rows, cols);
        if (row0 + nrows > rows || lda < cols)
            throw randsvd::IoError(std::string("row range outside ") + path, path, 22);
        in.seekg(22 + row0 * cols * 8);
        cudaStream_t st = static_cast<cudaStream_t>(rsvd_b200_stream(h));
        const uint64_t row_bytes = cols * 8;
        const uint64_t chunk_rows = std::max<uint64_t>(1, (64ull << 20) / row_bytes);
        void* stage[2] = {nullptr, nullptr};
        cudaEvent_t done[2] = {nullptr, nullptr};
        auto cleanup = [&] {
            for (int i = 0; i < 2; ++i) {
                if (done[i]) cudaEventDestroy(done[i]);
                if (stage[i]) cudaFreeHost(stage[i]);
            }
        };
        for (int i = 0; i < 2; ++i)
            if (cudaMallocHost(&stage[i], chunk_rows * row_bytes) != cudaSuccess ||
                cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) != cudaSuccess) {
                cleanup();
                throw std::runtime_error("pinned staging allocation failed");
            }
        uint64_t r = 0;
        int buf = 0;
        while (r < nrows) {
            const uint64_t nr = std::min(chunk_rows, nrows - r);
            cudaEventSynchronize(done[buf]);  // the copy that last used this buffer is done
            in.read(static_cast<char*>(stage[buf]), static_cast<std::streamsize>(nr * row_bytes));
            if (static_cast<uint64_t>(in.gcount()) != nr * row_bytes) {
                cudaStreamSynchronize(st);
                cleanup();
                const uint64_t off = 22 + (row0 + r) * row_bytes + in.gcount();
                throw randsvd::IoError("truncated DMAT payload in " + std::string(path) +
                                           " at byte offset " + std::to_string(off),
                                       path, off);
            }
            if (cudaMemcpy2DAsync(a_dev + r * lda, lda * 8, stage[buf], row_bytes, row_bytes, nr,
                                  cudaMemcpyHostToDevice, st) != cudaSuccess ||
                cudaEventRecord(done[buf], st) != cudaSuccess) {
                cudaStreamSynchronize(st);
                cleanup();
                throw std::runtime_error("H2D of a DMAT chunk failed");
            }
            r += nr;
            buf ^= 1;
        }
        cudaStreamSynchronize(st);
        cleanup();
        return 0;
    } catch (const std::exception& e) {
        g_dmat_error = e.what();
        return 7;
    }
}

}  // extern "C"
