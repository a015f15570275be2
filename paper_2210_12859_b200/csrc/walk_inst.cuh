// walk_inst.cuh — explicit instantiation helpers; one translation unit per
// dimension (walk_d*.cu) so nvcc compiles the kernel matrix in parallel.
#pragma once
#include "overflow.cuh"
#include "walk.cuh"

#include <algorithm>
#include <cstdlib>

// CTAs per SM of the overflow (CTA) pass: 1 -> 4 cuts the C3 fcp tail 0.28 -> 0.09 ms
#ifndef FKD_OVF_CTAS
#define FKD_OVF_CTAS 4
#endif
#ifndef FKD_L1_CARVEOUT
#define FKD_L1_CARVEOUT -1
#endif

namespace fkd {

inline unsigned walk_blocks(int64_t m, int threads) {
    return unsigned((m + threads - 1) / threads);
}

// Tail pass over the queries the walk kernel stopped (overflow.cuh); a
// persistent grid reads the device-side overflow count, so no host sync.
template <int D, int S, int KB>
void launch_overflow(const WalkArgs& a, cudaStream_t st) {
    constexpr int T = KB >= 20 ? 256 : 512;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    overflow_kernel<D, S, KB, T><<<sms * FKD_OVF_CTAS, T, 0, st>>>(a);
}

// -DFKD_L1_CARVEOUT=<percent>: preferred shared-memory carveout of the
// (shared-memory-free) walk kernels; the default (-1) leaves the driver's
// choice, which already gives them the largest L1 (0% times the same, 50%
// costs +3-4%: profiles/r01j_carveout_ab.log).
template <class K>
void set_carveout(K kernel) {
    if constexpr (FKD_L1_CARVEOUT >= 0)
        cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, FKD_L1_CARVEOUT);
}

// Threads per walk block: kWalkThreads, or half of it when that keeps more
// warps resident — a register count that strands part of the register file
// in whole blocks (96 registers: 2 blocks of 256 = 16 warps per SM, but 5 of
// 128 = 20).  N = 10M uniform: 4-D kNN20 9.09 -> 8.66 ms, kNN32 16.3 -> 14.9,
// kNN64 25.1 -> 20.3, 3-D kNN32 5.97 -> 5.61; C3, kNN8/16/50 unchanged
// (profiles/r02/r02at_walk_block_ab.log).
template <class K>
int pick_walk_threads(K kernel) {
    int full = 0, half = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&full, kernel, kWalkThreads, 0) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&half, kernel, kWalkThreads / 2, 0) != cudaSuccess) {
        cudaGetLastError();
        return kWalkThreads;
    }
    return half * (kWalkThreads / 2) > full * kWalkThreads ? kWalkThreads / 2 : kWalkThreads;
}

template <class K>
void launch_walk_grid(K kernel, const WalkArgs& a, int threads, cudaStream_t st) {
    set_carveout(kernel);
    kernel<<<walk_blocks(a.m, threads), threads, 0, st>>>(a);
}

template <int D, int S, int KB, bool STATS, bool UNORDERED>
void launch_one(const WalkArgs& a, cudaStream_t st) {
    static const int threads = pick_walk_threads(walk_kernel<D, S, KB, STATS, UNORDERED>);
    launch_walk_grid(walk_kernel<D, S, KB, STATS, UNORDERED>, a, threads, st);
}

template <int D, int S, int KB, bool UNORDERED>
void launch_round(const WalkArgs& a, cudaStream_t st) {
    static const int threads = pick_walk_threads(walk_round_kernel<D, S, KB, UNORDERED>);
    launch_walk_grid(walk_round_kernel<D, S, KB, UNORDERED>, a, threads, st);
}

// phase 0: the walk kernel; phase 1: the overflow pass (when budgeted);
// phase 3: one continuation round or the resume pass.
template <int D, int S, int KB>
int launch_bucket(const WalkArgs& a, bool stats, bool unordered, int phase, cudaStream_t st) {
    if (phase == 1) {
        if (stats || a.budget <= 0) return 0;
        launch_overflow<D, S, KB>(a, st);
        return 1;
    }
    if (phase == 3) {
        if (unordered)
            launch_round<D, S, KB, true>(a, st);
        else
            launch_round<D, S, KB, false>(a, st);
        return 1;
    }
    if (stats) {
        if (unordered)
            launch_one<D, S, KB, true, true>(a, st);
        else
            launch_one<D, S, KB, true, false>(a, st);
    } else {
        if (unordered)
            launch_one<D, S, KB, false, true>(a, st);
        else
            launch_one<D, S, KB, false, false>(a, st);
    }
    return 1;
}

template <int D, int S>
int launch_fixed(const WalkArgs& a, int KB, bool stats, bool unordered, int phase, cudaStream_t st) {
    switch (KB) {
        case 1: return launch_bucket<D, S, 1>(a, stats, unordered, phase, st);
        case 2: return launch_bucket<D, S, 2>(a, stats, unordered, phase, st);
        case 4: return launch_bucket<D, S, 4>(a, stats, unordered, phase, st);
        case 8: return launch_bucket<D, S, 8>(a, stats, unordered, phase, st);
        case 16: return launch_bucket<D, S, 16>(a, stats, unordered, phase, st);
        case 20: return launch_bucket<D, S, 20>(a, stats, unordered, phase, st);
        case 32: return launch_bucket<D, S, 32>(a, stats, unordered, phase, st);
        case 50: return launch_bucket<D, S, 50>(a, stats, unordered, phase, st);
        case 64: return launch_bucket<D, S, 64>(a, stats, unordered, phase, st);
        default: return 0;
    }
}

// 9..16-D: the production walk only (ordered, no counters: STATS and
// unordered batches take the heap kernel there), buckets 1 / 8 / 16 / 32 / 64
// (walk_bucket_of(k, dim) rounds k up to one)
template <int D, int S, int KB>
int launch_bucket_hd(const WalkArgs& a, bool stats, bool unordered, int phase, cudaStream_t st) {
    if (stats || unordered) return 0;
    if (phase == 1) {
        if (a.budget <= 0) return 0;
        launch_overflow<D, S, KB>(a, st);
        return 1;
    }
    if (phase == 3)
        launch_round<D, S, KB, false>(a, st);
    else
        launch_one<D, S, KB, false, false>(a, st);
    return 1;
}

template <int D, int S>
int launch_fixed_hd(const WalkArgs& a, int KB, bool stats, bool unordered, int phase, cudaStream_t st) {
    switch (KB) {
        case 1: return launch_bucket_hd<D, S, 1>(a, stats, unordered, phase, st);
        case 8: return launch_bucket_hd<D, S, 8>(a, stats, unordered, phase, st);
        case 16: return launch_bucket_hd<D, S, 16>(a, stats, unordered, phase, st);
        case 32: return launch_bucket_hd<D, S, 32>(a, stats, unordered, phase, st);
        case 64: return launch_bucket_hd<D, S, 64>(a, stats, unordered, phase, st);
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
int launch_walk_d1(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d2(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d3(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d4(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d5(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d6(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d7(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d9(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d10(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d11(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d12(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d13(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d14(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d15(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d16(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_d8(const WalkArgs&, int S, int KB, bool, bool, int phase, cudaStream_t);
int launch_walk_heap(const WalkArgs&, int dim, bool, bool, cudaStream_t);

}  // namespace fkd
