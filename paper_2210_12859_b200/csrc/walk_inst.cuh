// walk_inst.cuh — explicit instantiation helpers; one translation unit per
// dimension (walk_d*.cu) so nvcc compiles the kernel matrix in parallel.
#pragma once
#include "walk.cuh"

namespace fkd {

inline unsigned walk_blocks(int64_t m, int threads) {
    return unsigned((m + threads - 1) / threads);
}

template <int D, int S, int KB>
int launch_bucket(const WalkArgs& a, bool stats, bool unordered, cudaStream_t st) {
    const unsigned grid = walk_blocks(a.m, 256);
    if (stats) {
        if (unordered)
            walk_kernel<D, S, KB, true, true><<<grid, 256, 0, st>>>(a);
        else
            walk_kernel<D, S, KB, true, false><<<grid, 256, 0, st>>>(a);
    } else {
        if (unordered)
            walk_kernel<D, S, KB, false, true><<<grid, 256, 0, st>>>(a);
        else
            walk_kernel<D, S, KB, false, false><<<grid, 256, 0, st>>>(a);
    }
    return 1;
}

template <int D, int S>
int launch_fixed(const WalkArgs& a, int KB, bool stats, bool unordered, cudaStream_t st) {
    switch (KB) {
        case 1: return launch_bucket<D, S, 1>(a, stats, unordered, st);
        case 2: return launch_bucket<D, S, 2>(a, stats, unordered, st);
        case 4: return launch_bucket<D, S, 4>(a, stats, unordered, st);
        case 8: return launch_bucket<D, S, 8>(a, stats, unordered, st);
        case 16: return launch_bucket<D, S, 16>(a, stats, unordered, st);
        case 32: return launch_bucket<D, S, 32>(a, stats, unordered, st);
        case 64: return launch_bucket<D, S, 64>(a, stats, unordered, st);
        default: return 0;
    }
}

template <int D>
int launch_heap(const WalkArgs& a, bool stats, bool unordered, cudaStream_t st) {
    const unsigned grid = walk_blocks(a.m, 128);
    if (stats) {
        if (unordered)
            walk_heap_kernel<D, true, true><<<grid, 128, 0, st>>>(a);
        else
            walk_heap_kernel<D, true, false><<<grid, 128, 0, st>>>(a);
    } else {
        if (unordered)
            walk_heap_kernel<D, false, true><<<grid, 128, 0, st>>>(a);
        else
            walk_heap_kernel<D, false, false><<<grid, 128, 0, st>>>(a);
    }
    return 1;
}

// per-dimension entry points (defined in walk_d<D>.cu)
int launch_walk_d1(const WalkArgs&, int S, int KB, bool, bool, cudaStream_t);
int launch_walk_d2(const WalkArgs&, int S, int KB, bool, bool, cudaStream_t);
int launch_walk_d3(const WalkArgs&, int S, int KB, bool, bool, cudaStream_t);
int launch_walk_d4(const WalkArgs&, int S, int KB, bool, bool, cudaStream_t);
int launch_walk_d5(const WalkArgs&, int S, int KB, bool, bool, cudaStream_t);
int launch_walk_d6(const WalkArgs&, int S, int KB, bool, bool, cudaStream_t);
int launch_walk_d7(const WalkArgs&, int S, int KB, bool, bool, cudaStream_t);
int launch_walk_d8(const WalkArgs&, int S, int KB, bool, bool, cudaStream_t);
int launch_walk_heap(const WalkArgs&, int dim, bool, bool, cudaStream_t);

}  // namespace fkd
