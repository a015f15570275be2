// order.cu — Morton ordering of a query batch and the
// small tree-store kernels.
//
// Keys: each coordinate is quantised to b bits over the TREE's bounding box
// (computed once at tree creation, so no per-batch reduction pass), clamped,
// and the D*b bits interleaved into a 32-bit key.  A CUB onesweep radix sort
// of (key, query id) over exactly D*b bits yields order[]: walk position ->
// query id.  The walk kernel gathers queries through order[] and scatters
// results to their own slots, so no permute / un-permute passes exist.
// Ordering never changes results (every query is independent); it only makes
// the 32 lanes of a warp walk neighbouring paths.
#include <cub/device/device_radix_sort.cuh>

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

template <int D>
__global__ void __launch_bounds__(256)
    morton_keys_kernel(const float* __restrict__ q, int64_t m, MortonFrame f,
                       uint32_t* __restrict__ keys, uint32_t* __restrict__ ids) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int b = f.bits;
    const float top = float((1u << b) - 1u);
    uint32_t c[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        float t = (__ldg(q + i * D + d) - f.lo[d]) * f.scale[d];
        t = fminf(fmaxf(t, 0.0f), top);  // NaN -> 0 (non-finite is reported by the walk)
        c[d] = uint32_t(t);
    }
    uint32_t key = 0;
    for (int bit = b - 1; bit >= 0; --bit) {
#pragma unroll
        for (int d = 0; d < D; ++d) key = (key << 1) | ((c[d] >> bit) & 1u);
    }
    keys[i] = key;
    ids[i] = uint32_t(i);
}

size_t morton_temp_bytes(int64_t m) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)m, 0, 32);
    return bytes;
}

int morton_order(const float* d_queries, int64_t m, int dim, const MortonFrame& f,
                 uint32_t* keys_in, uint32_t* keys_out, uint32_t* ids_in, uint32_t* ids_out,
                 void* temp, size_t temp_bytes, cudaStream_t st) {
    const unsigned grid = unsigned((m + 255) / 256);
    switch (dim) {
        case 1: morton_keys_kernel<1><<<grid, 256, 0, st>>>(d_queries, m, f, keys_in, ids_in); break;
        case 2: morton_keys_kernel<2><<<grid, 256, 0, st>>>(d_queries, m, f, keys_in, ids_in); break;
        case 3: morton_keys_kernel<3><<<grid, 256, 0, st>>>(d_queries, m, f, keys_in, ids_in); break;
        case 4: morton_keys_kernel<4><<<grid, 256, 0, st>>>(d_queries, m, f, keys_in, ids_in); break;
        case 5: morton_keys_kernel<5><<<grid, 256, 0, st>>>(d_queries, m, f, keys_in, ids_in); break;
        case 6: morton_keys_kernel<6><<<grid, 256, 0, st>>>(d_queries, m, f, keys_in, ids_in); break;
        case 7: morton_keys_kernel<7><<<grid, 256, 0, st>>>(d_queries, m, f, keys_in, ids_in); break;
        case 8: morton_keys_kernel<8><<<grid, 256, 0, st>>>(d_queries, m, f, keys_in, ids_in); break;
        default: return -1;
    }
    size_t bytes = temp_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, bytes, keys_in, keys_out, ids_in, ids_out,
                                                    (int)m, 0, f.bits * dim, st);
    if (e != cudaSuccess) return -1;
    return 1;  // our own launches (the CUB sort kernels are library launches)
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
