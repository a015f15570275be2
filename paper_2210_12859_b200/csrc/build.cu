// build.cu — GPU builder for the left-balanced level-order k-d tree
// (SURVEY.md §8 row f1), byte-identical to flatkd::build_tree
// (src/tree.cpp:55-89).
//
// Reference: build_range() places, at each slot, the element of rank
// left_subtree_size(n) (tree.cpp:10-18) of its range under RankOrder
// (tree.cpp:40-53: split coordinate, then the whole tuple left to right,
// then the original index; floats compared with == / <, so -0 == +0), and
// recurses on the two sides.  RankOrder is a strict total order, so every
// range's membership and every placed element are unique: any algorithm
// that selects by the same order produces the same array.
//
// Here, level-synchronously (every slot of one depth at once):
//   1. ranks: for each dim d, the global position of every point under
//      RankOrder_d — one lexicographic "base" order (stable LSD radix sorts
//      over coords D-1..0, starting from index order), then one more stable
//      sort by coord d per dim.  RankOrder_d == compare rank_d.
//   2. levels: each point carries the slot of the subtree it is in; one
//      radix sort by (slot, rank_{depth % D}) makes every subtree a
//      contiguous run in RankOrder; the run's element at position
//      left_subtree_size(run length) goes to the slot, the rest move to
//      2*slot+1 / 2*slot+2.  Placed points sort to the end.
// Cost: 2D small sorts + one sort per level, O(N log N) on the device.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdint>
#include <string>

#include "build.cuh"

namespace fkd {
namespace {

__device__ __forceinline__ uint32_t orderable(float x) {
    const uint32_t u = __float_as_uint(__fadd_rn(x, 0.0f));  // -0 -> +0 (RankOrder's ==)
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void iota_kernel(uint32_t* out, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = uint32_t(i);
}

__global__ void gather_key_kernel(const float* __restrict__ pts, int dim, int c,
                                  const uint32_t* __restrict__ ids, uint32_t* __restrict__ keys,
                                  int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = orderable(pts[int64_t(ids[i]) * dim + c]);
}

__global__ void scatter_rank_kernel(const uint32_t* __restrict__ ids, uint32_t* __restrict__ rank,
                                    int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) rank[ids[i]] = uint32_t(i);
}

// nodes in the subtree rooted at `slot` of a dense level-order tree of n
__device__ __forceinline__ int64_t subtree_size(int64_t slot, int64_t n) {
    int64_t first = slot, width = 1, total = 0;
    while (first < n) {
        const int64_t last = first + width;  // exclusive
        total += (last < n ? last : n) - first;
        first = 2 * first + 1;
        width *= 2;
    }
    return total;
}

// tree.cpp:10-18
__device__ __forceinline__ int64_t left_subtree_size(int64_t n) {
    if (n <= 1) return 0;
    const int h = 63 - __clzll(n);
    const int64_t full = (int64_t(1) << h) - 1;
    const int64_t last = n - full;
    const int64_t half = int64_t(1) << (h - 1);
    return (half - 1) + (last < half ? last : half);
}

// keys for level L: (slot - first slot of the level) << rbits | rank, placed
// points get the bit above every live key so they sort last.
__global__ void level_keys_kernel(const uint32_t* __restrict__ tag, const uint32_t* __restrict__ rank,
                                  const uint32_t* __restrict__ ids, uint64_t* __restrict__ keys,
                                  int64_t n, uint32_t level_first, int rbits, int done_bit) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t p = ids[i];
    const uint32_t t = tag[p];
    keys[i] = t == 0xFFFFFFFFu ? (uint64_t(1) << done_bit)
                               : (uint64_t(t - level_first) << rbits) | rank[p];
}

// head flags -> segment start via max-scan input
__global__ void heads_kernel(const uint64_t* __restrict__ keys, int64_t n, int rbits,
                             int64_t* __restrict__ start) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool head = i == 0 || (keys[i] >> rbits) != (keys[i - 1] >> rbits);
    start[i] = head ? i : 0;
}

struct MaxOp {
    __device__ __forceinline__ int64_t operator()(int64_t a, int64_t b) const { return a > b ? a : b; }
};

__global__ void place_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ ids,
                             const int64_t* __restrict__ start, int64_t live, int64_t n, int dim,
                             uint32_t level_first, int rbits, const float* __restrict__ pts,
                             uint32_t* __restrict__ tag, float* __restrict__ out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= live) return;
    const uint32_t p = ids[i];
    const int64_t slot = int64_t(keys[i] >> rbits) + level_first;
    const int64_t pos = i - start[i];
    const int64_t r = left_subtree_size(subtree_size(slot, n));
    if (pos == r) {
        for (int c = 0; c < dim; ++c) out[slot * dim + c] = pts[int64_t(p) * dim + c];
        tag[p] = 0xFFFFFFFFu;
    } else {
        tag[p] = uint32_t(pos < r ? 2 * slot + 1 : 2 * slot + 2);
    }
}

inline unsigned blocks(int64_t n) { return unsigned((n + 255) / 256); }

}  // namespace

BuildStatus build_tree_device(const float* d_pts, int64_t n, int dim, float* d_out, cudaStream_t st) {
    BuildStatus bs;
    if (n == 0) return bs;
    auto ck = [&](cudaError_t e, const char* what) {
        if (e != cudaSuccess && bs.err == cudaSuccess) {
            bs.err = e;
            bs.what = what;
        }
        return e == cudaSuccess;
    };
    const int rbits = std::max(1, 64 - __builtin_clzll(uint64_t(n - 1) | 1));
    uint32_t *ids = nullptr, *ids2 = nullptr, *k32 = nullptr, *k32b = nullptr, *rank = nullptr,
             *tag = nullptr;
    uint64_t *k64 = nullptr, *k64b = nullptr;
    int64_t* start = nullptr;
    int64_t* start2 = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    {
        size_t b1 = 0, b2 = 0, b3 = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, b1, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                        (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 32, st);
        cub::DeviceRadixSort::SortPairs(nullptr, b2, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                        (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 64, st);
        cub::DeviceScan::InclusiveScan(nullptr, b3, (int64_t*)nullptr, (int64_t*)nullptr, MaxOp(),
                                       (int)n, st);
        tmp_bytes = std::max(b1, std::max(b2, b3));
    }
    const size_t N = size_t(n);
    if (!ck(cudaMalloc(&ids, N * 4), "alloc") || !ck(cudaMalloc(&ids2, N * 4), "alloc") ||
        !ck(cudaMalloc(&k32, N * 4), "alloc") || !ck(cudaMalloc(&k32b, N * 4), "alloc") ||
        !ck(cudaMalloc(&rank, N * 4 * size_t(dim)), "alloc") || !ck(cudaMalloc(&tag, N * 4), "alloc") ||
        !ck(cudaMalloc(&k64, N * 8), "alloc") || !ck(cudaMalloc(&k64b, N * 8), "alloc") ||
        !ck(cudaMalloc(&start, N * 8), "alloc") || !ck(cudaMalloc(&start2, N * 8), "alloc") ||
        !ck(cudaMalloc(&tmp, tmp_bytes), "alloc")) {
    } else {
        // ---- 1. base lexicographic order (coords 0..D-1, then index)
        iota_kernel<<<blocks(n), 256, 0, st>>>(ids, n);
        ++bs.launches;
        for (int c = dim - 1; c >= 0 && bs.err == cudaSuccess; --c) {
            gather_key_kernel<<<blocks(n), 256, 0, st>>>(d_pts, dim, c, ids, k32, n);
            ++bs.launches;
            size_t b = tmp_bytes;
            ck(cub::DeviceRadixSort::SortPairs(tmp, b, k32, k32b, ids, ids2, (int)n, 0, 32, st), "sort");
            std::swap(ids, ids2);
        }
        // ---- rank_d: stable sort of the base order by coord d
        uint32_t *base = nullptr;
        if (ck(cudaMalloc(&base, N * 4), "alloc")) {
            ck(cudaMemcpyAsync(base, ids, N * 4, cudaMemcpyDeviceToDevice, st), "copy");
            for (int d = 0; d < dim && bs.err == cudaSuccess; ++d) {
                gather_key_kernel<<<blocks(n), 256, 0, st>>>(d_pts, dim, d, base, k32, n);
                size_t b = tmp_bytes;
                ck(cub::DeviceRadixSort::SortPairs(tmp, b, k32, k32b, base, ids2, (int)n, 0, 32, st), "sort");
                scatter_rank_kernel<<<blocks(n), 256, 0, st>>>(ids2, rank + size_t(d) * N, n);
                bs.launches += 2;
            }
            cudaFree(base);
        }
        // ---- 2. levels
        ck(cudaMemsetAsync(tag, 0, N * 4, st), "memset");
        iota_kernel<<<blocks(n), 256, 0, st>>>(ids, n);
        ++bs.launches;
        int64_t placed = 0;
        for (int level = 0; placed < n && bs.err == cudaSuccess; ++level) {
            const uint32_t first = (1u << level) - 1u;
            const int64_t width = std::min<int64_t>(int64_t(1) << level, n - int64_t(first));
            const int64_t live = n - placed;
            const int done_bit = level + rbits;
            level_keys_kernel<<<blocks(n), 256, 0, st>>>(tag, rank + size_t(level % dim) * N, ids, k64, n,
                                                         first, rbits, done_bit);
            size_t b = tmp_bytes;
            ck(cub::DeviceRadixSort::SortPairs(tmp, b, k64, k64b, ids, ids2, (int)n, 0, done_bit + 1, st),
               "sort");
            std::swap(ids, ids2);
            heads_kernel<<<blocks(live), 256, 0, st>>>(k64b, live, rbits, start);
            b = tmp_bytes;
            ck(cub::DeviceScan::InclusiveScan(tmp, b, start, start2, MaxOp(), (int)live, st), "scan");
            place_kernel<<<blocks(live), 256, 0, st>>>(k64b, ids, start2, live, n, dim, first, rbits, d_pts,
                                                       tag, d_out);
            bs.launches += 3;
            ck(cudaGetLastError(), "launch");
            placed += width;
        }
    }
    cudaFree(ids);
    cudaFree(ids2);
    cudaFree(k32);
    cudaFree(k32b);
    cudaFree(rank);
    cudaFree(tag);
    cudaFree(k64);
    cudaFree(k64b);
    cudaFree(start);
    cudaFree(start2);
    cudaFree(tmp);
    return bs;
}

}  // namespace fkd
