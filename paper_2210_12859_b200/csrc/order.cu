// order.cu — Morton ordering of a query batch and the
// small tree-store kernels.
//
// Keys: each coordinate is quantised to b bits over the TREE's bounding box
// (computed once at tree creation, so no per-batch reduction pass), clamped,
// and the D*b <= 24 bits interleaved into a key.  order[] (walk position ->
// query id) groups equal keys in key order, built one of two ways:
//   * counting sort (large batches): one pass computes the key and takes a
//     rank inside its bin with an atomic, an exclusive scan over the 2^(D*b)
//     bins gives bin offsets, one pass scatters id -> offset + rank.  Two
//     reads of the batch instead of the onesweep's three digit passes; the
//     order inside a bin is arbitrary (C3's fullest 24-bit bin holds 140 of
//     10M queries, so the atomics barely contend);
//   * CUB onesweep radix sort of (key, id) over D*b bits (small batches,
//     where scanning 2^24 bins would dominate).  The walk kernel gathers queries through order[] and scatters
// results to their own slots, so no permute / un-permute passes exist.
// Ordering never changes results (every query is independent); it only makes
// the 32 lanes of a warp walk neighbouring paths.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include <cstdint>
#include <cstring>

#include "order.cuh"

namespace fkd {

int morton_bits_per_dim(int dim) {
    if (dim <= 0) return 0;
    int b = 24 / dim;  // 24-bit keys: three 8-bit onesweep passes (measured: no walk cost vs 30 bits)
    if (b > 16) b = 16;
    if (b < 1) b = 1;
    return b;
}

// The key pass reads every query once, so it also performs the reference's
// require_finite(queries, "queries") (batch.cpp:79): the first non-finite
// query id goes to *bad (atomicMin), and the walk kernels that follow exit
// at entry when *bad is set, so no result slot is written for a rejected
// batch (the reference throws before its BatchResult exists, :82-86).
// D axes of a query stored qs floats apart (qs = D, or the query dimension
// from 9-D up, where the key covers the first 8 axes and a scan checks the rest)
template <int D>
__device__ __forceinline__ uint32_t morton_key(const float* __restrict__ q, int64_t i, int qs, const MortonFrame& f,
                                               unsigned long long* bad, int64_t id_base) {
    const int b = f.bits;
    const float top = float((1u << b) - 1u);
    uint32_t c[D];
    bool finite = true;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const float v = __ldg(q + i * qs + d);
        finite &= isfinite(v);
        float t = (v - f.lo[d]) * f.scale[d];
        t = fminf(fmaxf(t, 0.0f), top);  // NaN -> 0 (the batch is rejected anyway)
        c[d] = uint32_t(t);
    }
    if (!finite) atomicMin(bad, (unsigned long long)(id_base + i));
    uint32_t key = 0;
    for (int bit = b - 1; bit >= 0; --bit) {
#pragma unroll
        for (int d = 0; d < D; ++d) key = (key << 1) | ((c[d] >> bit) & 1u);
    }
    return key;
}

// counting sort, pass 1: key + rank inside the key's bin
template <int D>
__global__ void __launch_bounds__(256)
    morton_rank_kernel(const float* __restrict__ q, int64_t m, int qs, MortonFrame f, uint32_t* __restrict__ bins,
                       uint32_t* __restrict__ keys, uint32_t* __restrict__ ranks, unsigned long long* bad,
                       int64_t id_base) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t key = morton_key<D>(q, i, qs, f, bad, id_base);
    keys[i] = key;
    ranks[i] = atomicAdd(bins + key, 1u);
}

// counting sort, pass 2: id -> its bin's offset + its rank
__global__ void __launch_bounds__(256)
    morton_scatter_kernel(int64_t m, const uint32_t* __restrict__ offs, const uint32_t* __restrict__ keys,
                          const uint32_t* __restrict__ ranks, uint32_t* __restrict__ ids) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    ids[__ldg(offs + __ldg(keys + i)) + __ldg(ranks + i)] = uint32_t(i);
}

namespace {
constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
int key_axes(int dim) { return dim < 8 ? dim : 8; }
int64_t key_bins(int dim) { return int64_t(1) << (morton_bits_per_dim(key_axes(dim)) * key_axes(dim)); }
// Counting sort from 2^20 (below, scanning the bins dominates) to 2^25
// queries (above, the rank atomics are L2-atomic-throughput bound: 1B
// uniform queries order in 68 ms this way against 32 ms for the onesweep).
#ifndef FKD_COUNT_SORT_MIN
#define FKD_COUNT_SORT_MIN (int64_t(1) << 20)
#endif
#ifndef FKD_COUNT_SORT_MAX
#define FKD_COUNT_SORT_MAX (int64_t(1) << 25)
#endif
bool use_counting(int64_t m, int dim) {
    return m >= FKD_COUNT_SORT_MIN && m <= FKD_COUNT_SORT_MAX && dim >= 1 && dim <= 16;
}
size_t scan_bytes(int64_t bins) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)bins);
    return bytes;
}
}  // namespace

// radix path: keys + ids for the onesweep
template <int D>
__global__ void __launch_bounds__(256)
    morton_keys_kernel(const float* __restrict__ q, int64_t m, int qs, MortonFrame f,
                       uint32_t* __restrict__ keys, uint32_t* __restrict__ ids, unsigned long long* bad,
                       int64_t id_base) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    keys[i] = morton_key<D>(q, i, qs, f, bad, id_base);
    ids[i] = uint32_t(i);
}

// keys only (full frame resolution, no sort): the multi-GPU Morton-range
// partition (paper_2210_12859_b200/shard.py) splits a batch by these keys
template <int D>
__global__ void __launch_bounds__(256)
    morton_keys_only_kernel(const float* __restrict__ q, int64_t m, int qs, MortonFrame f, uint32_t* __restrict__ keys,
                            unsigned long long* bad) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    keys[i] = morton_key<D>(q, i, qs, f, bad, 0);
}

int morton_keys(const float* d_queries, int64_t m, int dim, const MortonFrame& f, uint32_t* keys,
                unsigned long long* bad, cudaStream_t st) {
    if (m <= 0) return 0;
    const unsigned grid = unsigned((m + 255) / 256);
    switch (key_axes(dim)) {
#define FKD_KEYS(D) case D: morton_keys_only_kernel<D><<<grid, 256, 0, st>>>(d_queries, m, dim, f, keys, bad); break;
        FKD_KEYS(1) FKD_KEYS(2) FKD_KEYS(3) FKD_KEYS(4) FKD_KEYS(5) FKD_KEYS(6) FKD_KEYS(7) FKD_KEYS(8)
#undef FKD_KEYS
        default: return -1;
    }
    return 1;
}

size_t morton_temp_bytes(int64_t m, int dim) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)m, 0, 32);
    if (use_counting(m, dim)) {
        const int64_t bins = key_bins(dim);
        bytes = std::max(bytes, 2 * align_up(size_t(bins) * sizeof(uint32_t)) + scan_bytes(bins));
    }
    return bytes;
}

int morton_order(const float* d_queries, int64_t m, int dim, const MortonFrame& frame,
                 uint32_t* keys_in, uint32_t* keys_out, uint32_t* ids_in, uint32_t* ids_out,
                 void* temp, size_t temp_bytes, unsigned long long* bad, int64_t id_base, cudaStream_t st) {
    const unsigned grid = unsigned((m + 255) / 256);
    // Resolution follows the batch: about 1.7 cells per query (C3, clustered:
    // 10M queries -> 8 bits per axis, a 1.25M host-path chunk -> 7, where 8
    // costs 0.092 vs 0.055 ms of ordering for the same walk time).
    MortonFrame f = frame;
    const int qs = dim;
    const bool counting = use_counting(m, dim);
    dim = key_axes(dim);  // from here on: the key's axes
    if (dim >= 1 && m > 0) {
        const int fit = int(std::floor(std::log2(double(m) * 1.7) / dim));
        const int b = std::max(1, std::min(frame.bits, fit));
        if (b < frame.bits) {
            const float ratio = float((1u << b) - 1u) / float((1u << frame.bits) - 1u);
            for (int d = 0; d < dim; ++d) f.scale[d] = frame.scale[d] * ratio;
            f.bits = b;
        }
    }
    if (counting) {
        const int64_t bins = int64_t(1) << (f.bits * dim);  // <= key_bins(dim), which sized temp
        uint32_t* cnt = static_cast<uint32_t*>(temp);
        uint32_t* offs = reinterpret_cast<uint32_t*>(static_cast<char*>(temp) + align_up(size_t(bins) * 4));
        void* stmp = static_cast<char*>(temp) + 2 * align_up(size_t(bins) * 4);
        size_t sbytes = scan_bytes(bins);
        if (2 * align_up(size_t(bins) * 4) + sbytes > temp_bytes) return -1;
        if (cudaMemsetAsync(cnt, 0, size_t(bins) * 4, st) != cudaSuccess) return -1;
        uint32_t* ranks = keys_out;
        switch (dim) {
#define FKD_RANK(D) case D: morton_rank_kernel<D><<<grid, 256, 0, st>>>(d_queries, m, qs, f, cnt, keys_in, ranks, bad, id_base); break;
            FKD_RANK(1) FKD_RANK(2) FKD_RANK(3) FKD_RANK(4) FKD_RANK(5) FKD_RANK(6) FKD_RANK(7) FKD_RANK(8)
#undef FKD_RANK
            default: return -1;
        }
        if (cub::DeviceScan::ExclusiveSum(stmp, sbytes, cnt, offs, (int)bins, st) != cudaSuccess) return -1;
        morton_scatter_kernel<<<grid, 256, 0, st>>>(m, offs, keys_in, ranks, ids_out);
        return 2;  // our own launches (the scan is a library launch)
    }
    switch (dim) {
        case 1: morton_keys_kernel<1><<<grid, 256, 0, st>>>(d_queries, m, qs, f, keys_in, ids_in, bad, id_base); break;
        case 2: morton_keys_kernel<2><<<grid, 256, 0, st>>>(d_queries, m, qs, f, keys_in, ids_in, bad, id_base); break;
        case 3: morton_keys_kernel<3><<<grid, 256, 0, st>>>(d_queries, m, qs, f, keys_in, ids_in, bad, id_base); break;
        case 4: morton_keys_kernel<4><<<grid, 256, 0, st>>>(d_queries, m, qs, f, keys_in, ids_in, bad, id_base); break;
        case 5: morton_keys_kernel<5><<<grid, 256, 0, st>>>(d_queries, m, qs, f, keys_in, ids_in, bad, id_base); break;
        case 6: morton_keys_kernel<6><<<grid, 256, 0, st>>>(d_queries, m, qs, f, keys_in, ids_in, bad, id_base); break;
        case 7: morton_keys_kernel<7><<<grid, 256, 0, st>>>(d_queries, m, qs, f, keys_in, ids_in, bad, id_base); break;
        case 8: morton_keys_kernel<8><<<grid, 256, 0, st>>>(d_queries, m, qs, f, keys_in, ids_in, bad, id_base); break;
        default: return -1;
    }
    size_t bytes = temp_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, bytes, keys_in, keys_out, ids_in, ids_out,
                                                    (int)m, 0, f.bits * dim, st);
    if (e != cudaSuccess) return -1;
    return 1;  // our own launches (the CUB sort kernels are library launches)
}

// require_finite(queries, "queries") (batch.cpp:79) for batches walked
// without the key pass: first non-finite query id -> *bad.
__global__ void __launch_bounds__(256)
    scan_queries_kernel(const float* __restrict__ q, int64_t m, int dim, unsigned long long* bad, int64_t id_base) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m * dim; i += stride)
        if (!isfinite(__ldg(q + i))) atomicMin(bad, (unsigned long long)(id_base + i / dim));
}

int scan_queries(const float* d_queries, int64_t m, int dim, unsigned long long* bad, int64_t id_base,
                 cudaStream_t st) {
    if (m <= 0 || dim <= 0) return 0;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (m * dim + 255) / 256;
    const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(sms) * 8)));
    scan_queries_kernel<<<grid, 256, 0, st>>>(d_queries, m, dim, bad, id_base);
    return 1;
}

// Sets *flag when some counts[i] != want.  The host pipeline writes the
// counts of an unbounded-radius batch itself (every query then has exactly
// min(k, n) hits: trees and queries are finite, so every distance passes
// d2 <= inf) and copies only the hits; this pass proves the device agreed.
__global__ void __launch_bounds__(256)
    count_check_kernel(const int32_t* __restrict__ c, int64_t m, int32_t want, unsigned long long* flag) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    bool diff = false;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride)
        diff |= __ldcs(c + i) != want;
    if (__syncthreads_or(diff) && threadIdx.x == 0) atomicOr(flag, 1ull);
}

int check_counts(const int32_t* d_counts, int64_t m, int32_t want, unsigned long long* flag, cudaStream_t st) {
    if (m <= 0) return 0;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t blocks = (m + 255) / 256;
    const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>(blocks, int64_t(sms) * 4)));
    count_check_kernel<<<grid, 256, 0, st>>>(d_counts, m, want, flag);
    return 1;
}

// ---- tree store ----

// level-order row-major [n x dim] -> padded [n x stride].  When the padding
// has room (stride > dim) its last float repeats the node's split coordinate
// (coord[depth % dim], tree.hpp:27-29), so the walk reads the plane from a
// fixed lane of the vector load instead of selecting it by split dimension.
__global__ void pack_nodes_kernel(const float* __restrict__ src, int64_t n, int dim, int stride,
                                  float* __restrict__ dst) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n * stride) return;
    const int64_t node = i / stride;
    const int c = int(i - node * stride);
    float v = 0.0f;
    if (c < dim) {
        v = src[node * dim + c];
    } else if (c == stride - 1) {
        const int depth = 31 - __clz(int(node) + 1);
        v = src[node * dim + depth % dim];
    }
    dst[i] = v;
}

__device__ __forceinline__ unsigned ordered_bits(float x) {
    const unsigned u = __float_as_uint(x);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// min/max per dim (ordered-int atomics) + first non-finite node index
__global__ void tree_scan_kernel(const float* __restrict__ src, int64_t n, int dim,
                                 unsigned* __restrict__ lohi, unsigned long long* __restrict__ bad) {
    const int64_t node = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (int d = 0; d < dim && d < 8; ++d) {
        unsigned lo = 0xffffffffu, hi = 0u;
        if (node < n) {
            const float v = src[node * dim + d];
            if (isfinite(v)) lo = hi = ordered_bits(v);
        }
        for (int off = 16; off > 0; off >>= 1) {
            lo = min(lo, __shfl_down_sync(0xffffffffu, lo, off));
            hi = max(hi, __shfl_down_sync(0xffffffffu, hi, off));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(lohi + 2 * d, lo);
            atomicMax(lohi + 2 * d + 1, hi);
        }
    }
    if (node < n) {
        bool finite = true;
        for (int d = 0; d < dim; ++d) finite &= isfinite(src[node * dim + d]);
        if (!finite) atomicMin(bad, (unsigned long long)node);
    }
}

int pack_nodes(const float* d_src, int64_t n, int dim, int stride, float* d_dst, cudaStream_t st) {
    const int64_t total = n * stride;
    if (total == 0) return 0;
    pack_nodes_kernel<<<unsigned((total + 255) / 256), 256, 0, st>>>(d_src, n, dim, stride, d_dst);
    return 1;
}

int tree_scan(const float* d_src, int64_t n, int dim, unsigned* d_lohi, unsigned long long* d_bad,
              cudaStream_t st) {
    if (n == 0) return 0;
    tree_scan_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(d_src, n, dim, d_lohi, d_bad);
    return 1;
}

__global__ void fill_empty_kernel(int32_t* __restrict__ counts, int2* __restrict__ hits, int64_t m,
                                  int k) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m * k) return;
    hits[i] = make_int2(-1, 0x7f800000);  // Hit{} = {-1, +inf} (traverse.hpp:70-73)
    if (i < m) counts[i] = 0;
}

int fill_empty(int32_t* d_counts, fkd_hit* d_hits, int64_t m, int k, cudaStream_t st) {
    const int64_t total = m * k;
    if (total == 0) return 0;
    fill_empty_kernel<<<unsigned((total + 255) / 256), 256, 0, st>>>(
        d_counts, reinterpret_cast<int2*>(d_hits), m, k);
    return 1;
}

float ordered_to_float(unsigned u) {
    unsigned v = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    float f;
    memcpy(&f, &v, 4);
    return f;
}

}  // namespace fkd
