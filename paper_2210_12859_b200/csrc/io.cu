// io.cu — FKDT / FKDX binary files.
//
// Format (include/flatkd/io.hpp:10-18, src/io.cpp:50-99): 4-byte magic
// ("FKDT" points, "FKDX" level-order tree), u32 version = 1, u32 k (dim),
// u64 count, then count*k little-endian f32, row major — a 20-byte header,
// as the reference's writer (encode_binary, io.cpp:50-63) produces.  (The
// reference's reader, decode_binary io.cpp:83-90, takes the payload at
// offset 16 and so rejects its own writer's files; we follow the documented
// layout and the writer.)
//
// Differences from the reference, both deliberate:
//   * the payload streams from the file into DEVICE memory through a pinned
//     double buffer (no full host copy), and finiteness is checked on the
//     device;
//   * the reference rejects count*k > INT_MAX floats (io.cpp:80-83), which
//     rules out a 1B-query 3-D file; here point files may hold up to 2^40
//     points (trees stay < 2^31 nodes: node ids are int32).
// Error texts follow the reference's ("<what>: bad magic", "... file has
// magic FKDX, expected FKDT", "unsupported version", payload mismatch,
// "<what>: non-finite coordinate in point i").
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fkd_b200.h"
#include "order.cuh"

namespace fkd {
const char* set_host_error(const std::string& msg);
}

namespace {

constexpr char kPts[4] = {'F', 'K', 'D', 'T'};
constexpr char kTree[4] = {'F', 'K', 'D', 'X'};

uint32_t get_u32(const unsigned char* p) { return p[0] | (p[1] << 8) | (p[2] << 16) | (uint32_t(p[3]) << 24); }
uint64_t get_u64(const unsigned char* p) { return uint64_t(get_u32(p)) | (uint64_t(get_u32(p + 4)) << 32); }

fkd_status err(fkd_status s, const std::string& m) {
    fkd::set_host_error(m);
    return s;
}

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

// Reads and validates the header; `kind` 0 = points, 1 = tree.
fkd_status read_header(File& file, const char* path, int kind, int64_t* count, int32_t* dim,
                       std::string* what) {
    *what = std::string(kind ? "tree file " : "points file ") + path;
    file.f = std::fopen(path, "rb");
    if (!file.f) return err(FKD_DATA_ERROR, "cannot open " + std::string(path));
    unsigned char h[20];
    if (std::fread(h, 1, 20, file.f) != 20) return err(FKD_DATA_ERROR, *what + ": truncated header");
    const char* want = kind ? kTree : kPts;
    const char* other = kind ? kPts : kTree;
    if (std::memcmp(h, want, 4) != 0) {
        if (std::memcmp(h, other, 4) == 0)
            return err(FKD_DATA_ERROR, *what + ": file has magic " + std::string(other, 4) + ", expected " +
                                           std::string(want, 4));
        return err(FKD_DATA_ERROR, *what + ": bad magic");
    }
    const uint32_t version = get_u32(h + 4);
    if (version != 1) return err(FKD_DATA_ERROR, *what + ": unsupported version " + std::to_string(version));
    const uint32_t k = get_u32(h + 8);
    const uint64_t n = get_u64(h + 12);
    if (n > 0 && k == 0) return err(FKD_DATA_ERROR, *what + ": zero dimension with nonzero count");
    const uint64_t limit = kind ? uint64_t(0x7fffffff) : (uint64_t(1) << 40);
    if (n > limit) return err(FKD_DATA_ERROR, *what + ": point count too large");
    if (k > 4096) return err(FKD_DATA_ERROR, *what + ": dimension too large");
    std::fseek(file.f, 0, SEEK_END);
    const long long size = std::ftell(file.f);
    std::fseek(file.f, 20, SEEK_SET);
    const unsigned long long floats = n * k;
    if (size < 20 || (unsigned long long)(size - 20) != floats * 4ull)
        return err(FKD_DATA_ERROR, *what + ": payload size does not match header (" +
                                       std::to_string(size - 20) + " bytes for " + std::to_string(floats) +
                                       " floats)");
    *count = int64_t(n);
    *dim = int32_t(k);
    return FKD_OK;
}

}  // namespace

extern "C" {

fkd_status fkd_file_info(const char* path, int32_t kind, int64_t* count, int32_t* dim) {
    File f;
    std::string what;
    return read_header(f, path, kind, count, dim, &what);
}

fkd_status fkd_read_file_device(const char* path, int32_t kind, float* d_out, int64_t capacity_points,
                                int64_t* count, int32_t* dim, void* stream) {
    File f;
    std::string what;
    fkd_status s = read_header(f, path, kind, count, dim, &what);
    if (s != FKD_OK) return s;
    if (*count > capacity_points) return err(FKD_INVALID_ARGUMENT, what + ": buffer too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t total = size_t(*count) * size_t(*dim) * sizeof(float);
    const size_t chunk = size_t(32) << 20;
    char* pinned = nullptr;
    if (cudaMallocHost(&pinned, 2 * chunk) != cudaSuccess) return err(FKD_CUDA_ERROR, "pinned staging");
    cudaEvent_t done[2];
    cudaEventCreate(&done[0]);
    cudaEventCreate(&done[1]);
    size_t off = 0;
    int b = 0;
    while (s == FKD_OK && off < total) {
        const size_t len = std::min(chunk, total - off);
        cudaEventSynchronize(done[b]);  // the previous copy out of this half finished
        if (std::fread(pinned + b * chunk, 1, len, f.f) != len) {
            s = err(FKD_DATA_ERROR, what + ": short read");
            break;
        }
        if (cudaMemcpyAsync(reinterpret_cast<char*>(d_out) + off, pinned + b * chunk, len,
                            cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaEventRecord(done[b], st) != cudaSuccess)
            s = err(FKD_CUDA_ERROR, "upload failed");
        off += len;
        b ^= 1;
    }
    cudaStreamSynchronize(st);
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
    cudaFreeHost(pinned);
    if (s != FKD_OK || *count == 0) return s;
    // require_finite(pts, what) (io.cpp:97), on the device
    unsigned* d_lohi = nullptr;
    unsigned long long* d_bad = nullptr;
    unsigned long long bad = ~0ull;
    if (cudaMalloc(&d_lohi, 16 * sizeof(unsigned)) != cudaSuccess ||
        cudaMalloc(&d_bad, sizeof(unsigned long long)) != cudaSuccess)
        return err(FKD_CUDA_ERROR, "scratch");
    cudaMemsetAsync(d_bad, 0xFF, sizeof(unsigned long long), st);
    cudaMemsetAsync(d_lohi, 0, 16 * sizeof(unsigned), st);
    fkd::tree_scan(d_out, *count, *dim, d_lohi, d_bad, st);
    cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(d_lohi);
    cudaFree(d_bad);
    if (e != cudaSuccess) return err(FKD_CUDA_ERROR, std::string("finite check: ") + cudaGetErrorString(e));
    if (bad != ~0ull) return err(FKD_DATA_ERROR, what + ": non-finite coordinate in point " + std::to_string(bad));
    return FKD_OK;
}

fkd_status fkd_write_file(const char* path, int32_t kind, const float* data, int64_t count, int32_t dim) {
    FILE* f = std::fopen(path, "wb");
    if (!f) return err(FKD_DATA_ERROR, "cannot create " + std::string(path));
    unsigned char h[20];
    std::memcpy(h, kind ? kTree : kPts, 4);
    const uint32_t v = 1, k = uint32_t(dim);
    const uint64_t n = uint64_t(count);
    for (int i = 0; i < 4; ++i) {
        h[4 + i] = (v >> (8 * i)) & 0xff;
        h[8 + i] = (k >> (8 * i)) & 0xff;
    }
    for (int i = 0; i < 8; ++i) h[12 + i] = (n >> (8 * i)) & 0xff;
    bool ok = std::fwrite(h, 1, 20, f) == 20;
    const size_t bytes = size_t(count) * size_t(dim) * sizeof(float);
    if (ok && bytes) ok = std::fwrite(data, 1, bytes, f) == bytes;
    ok = (std::fclose(f) == 0) && ok;
    return ok ? FKD_OK : err(FKD_DATA_ERROR, "write failed on " + std::string(path));
}

fkd_status fkd_tree_load(const char* path, const int32_t* devices, int32_t ndev, fkd_tree** out) {
    if (!out) return err(FKD_INVALID_ARGUMENT, "null output");
    *out = nullptr;
    int64_t n = 0;
    int32_t dim = 0;
    fkd_status s = fkd_file_info(path, 1, &n, &dim);
    if (s != FKD_OK) return s;
    int dev = 0;
    if (devices && ndev > 0) dev = devices[0]; else cudaGetDevice(&dev);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
    float* d = nullptr;
    if (n > 0 && cudaMalloc(&d, size_t(n) * dim * sizeof(float)) != cudaSuccess) {
        cudaSetDevice(prev);
        return err(FKD_CUDA_ERROR, "tree buffer");
    }
    s = fkd_read_file_device(path, 1, d, n, &n, &dim, nullptr);
    if (s == FKD_OK) s = fkd_tree_create_device(d, n, dim, nullptr, out);
    cudaFree(d);
    cudaSetDevice(prev);
    // the other devices get their replicas device to device from the first
    // (fkd_tree_add_replicas: pipelined fan-out), not from the file again
    if (s == FKD_OK && devices && ndev > 1) {
        s = fkd_tree_add_replicas(*out, devices + 1, ndev - 1);
        if (s != FKD_OK) {
            fkd_tree_destroy(*out);
            *out = nullptr;
        }
    }
    return s;
}

}  // extern "C"
