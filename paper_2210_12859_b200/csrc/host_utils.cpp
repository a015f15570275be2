// host_utils.cpp — host-side pieces of the C ABI that surround the GPU path:
// the level-order builder, the seeded generators and the result hash.
// None of these answer queries; the query path is walk.cuh only.
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <future>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "fkd_b200.h"

namespace fkd {
const char* set_host_error(const std::string& msg);
}

namespace {

// src/tree.cpp:10-18: nodes in the left subtree of a dense level-order tree.
int64_t left_subtree_size(int64_t n) {
    if (n <= 1) return 0;
    const int h = std::bit_width(static_cast<uint64_t>(n)) - 1;
    const int64_t full = (int64_t(1) << h) - 1;
    const int64_t last = n - full;
    const int64_t half = int64_t(1) << (h - 1);
    return (half - 1) + std::min(last, half);
}

struct Builder {
    const float* pts;
    int dim;
    float* out;

    // RankOrder (src/tree.cpp:40-53): a strict total order, so the element of
    // each rank and every sub-range's membership are unique — any selection
    // algorithm yields the reference's array byte for byte.
    bool less(int d, int a, int b) const {
        const float* pa = pts + size_t(a) * dim;
        const float* pb = pts + size_t(b) * dim;
        if (pa[d] != pb[d]) return pa[d] < pb[d];
        for (int i = 0; i < dim; ++i)
            if (pa[i] != pb[i]) return pa[i] < pb[i];
        return a < b;
    }

    // src/tree.cpp:55-67, with the two halves built concurrently near the root
    void build(int* ord, int64_t n, int64_t slot, int depth, int spawn_levels) {
        while (n > 0) {
            const int d = depth % dim;  // slot depth == recursion depth
            const int64_t rank = left_subtree_size(n);
            std::nth_element(ord, ord + rank, ord + n,
                             [this, d](int a, int b) { return less(d, a, b); });
            std::memcpy(out + size_t(slot) * dim, pts + size_t(ord[rank]) * dim,
                        sizeof(float) * size_t(dim));
            int* right = ord + rank + 1;
            const int64_t nr = n - rank - 1;
            if (spawn_levels > 0 && n > 32768) {
                auto fut = std::async(std::launch::async, [=, this] {
                    build(ord, rank, 2 * slot + 1, depth + 1, spawn_levels - 1);
                });
                build(right, nr, 2 * slot + 2, depth + 1, spawn_levels - 1);
                fut.get();
                return;
            }
            build(ord, rank, 2 * slot + 1, depth + 1, 0);
            ord = right;
            n = nr;
            slot = 2 * slot + 2;
            depth = depth + 1;
        }
    }
};

// rng.hpp:11-29
uint64_t splitmix64(uint64_t& s) {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t stream_seed(uint64_t master, uint64_t stream) {
    uint64_t x = master ^ (stream * 0x9E3779B97F4A7C15ull);
    return splitmix64(x);
}

// rng.hpp:38: top 24 bits scaled by 2^-24
inline float unit_float(std::mt19937_64& g) { return static_cast<float>(g() >> 40) * 0x1p-24f; }

}  // namespace

extern "C" {

fkd_status fkd_build_tree(const float* points, int64_t n, int32_t dim, float* out) {
    if (n < 0 || n > int64_t(0x7fffffff)) {
        fkd::set_host_error("build: size out of range");
        return FKD_DATA_ERROR;
    }
    if (n > 0 && dim < 1) {
        fkd::set_host_error("build: dimension must be >= 1");
        return FKD_DATA_ERROR;
    }
    for (int64_t i = 0; i < n; ++i)  // require_finite(points, "build") (tree.cpp:81)
        for (int d = 0; d < dim; ++d)
            if (!std::isfinite(points[i * dim + d])) {
                fkd::set_host_error("build: non-finite coordinate in point " + std::to_string(i));
                return FKD_DATA_ERROR;
            }
    if (n == 0) return FKD_OK;
    std::vector<int> ord(static_cast<size_t>(n));
    std::iota(ord.begin(), ord.end(), 0);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    int levels = 0;
    while ((1u << levels) < 2 * hw && levels < 8) ++levels;
    Builder b{points, dim, out};
    b.build(ord.data(), n, 0, 0, levels);
    return FKD_OK;
}

uint64_t fkd_result_hash(const int32_t* counts, const fkd_hit* hits, int64_t m, int32_t stride) {
    // src/batch.cpp:30-48: FNV-1a, little-endian bytes of each 32-bit word
    uint64_t h = 0xcbf29ce484222325ull;
    auto mix = [&h](uint32_t v) {
        for (int i = 0; i < 4; ++i) {
            h ^= (v >> (8 * i)) & 0xffu;
            h *= 0x100000001b3ull;
        }
    };
    for (int64_t q = 0; q < m; ++q) {
        const int32_t c = counts[q];
        mix(static_cast<uint32_t>(c));
        for (int32_t j = 0; j < c; ++j) {
            const fkd_hit& hit = hits[q * stride + j];
            uint32_t bits;
            std::memcpy(&bits, &hit.dist2, 4);
            mix(static_cast<uint32_t>(hit.node));
            mix(bits);
        }
    }
    return h;
}

fkd_status fkd_random_points(uint64_t master, uint64_t stream, int64_t count, int32_t dim,
                             float* out) {
    if (count < 0 || dim < 1) {
        fkd::set_host_error("random points: bad shape");
        return FKD_DATA_ERROR;
    }
    std::mt19937_64 g(stream_seed(master, stream));  // random_points (rng.hpp:46-53)
    const int64_t total = count * dim;
    for (int64_t i = 0; i < total; ++i) out[i] = unit_float(g);
    return FKD_OK;
}

// Clustered workload: `blobs` centres drawn as
// random_points(stream 3); each point picks blob = next_u64() % blobs and adds
// float(z) * sigma per axis, z = sqrt(-2 ln(1-u1)) cos(2 pi u2) in double,
// u = (next_u64() >> 11) * 2^-53.  Host-only (libm-dependent).
fkd_status fkd_clustered_points(uint64_t master, uint64_t stream, int64_t count, int32_t dim,
                                int32_t blobs, float sigma, float* out) {
    if (count < 0 || dim < 1 || blobs < 1) {
        fkd::set_host_error("clustered points: bad shape");
        return FKD_DATA_ERROR;
    }
    std::vector<float> centres(size_t(blobs) * dim);
    fkd_random_points(master, 3, blobs, dim, centres.data());
    std::mt19937_64 g(stream_seed(master, stream));
    const double two_pi = 6.283185307179586476925286766559;
    for (int64_t i = 0; i < count; ++i) {
        const uint64_t b = g() % uint64_t(blobs);
        for (int d = 0; d < dim; ++d) {
            const double u1 = double(g() >> 11) * 0x1p-53;
            const double u2 = double(g() >> 11) * 0x1p-53;
            const double z = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(two_pi * u2);
            out[i * dim + d] = centres[size_t(b) * dim + d] + static_cast<float>(z) * sigma;
        }
    }
    return FKD_OK;
}

}  // extern "C"
