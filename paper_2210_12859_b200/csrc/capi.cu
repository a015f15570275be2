// capi.cu — the C ABI (include/fkd_b200.h): device tree store, batch
// dispatch, validation and the chunked host pipeline.
//
// Replaces flatkd::run_batch (src/batch.cpp:71-134) and
// KdTree::from_level_order (src/tree.cpp:71-78) at the drop-in boundary.
// No CPU fallback exists: every query is answered by the sm_100a kernels in
// walk.cuh; without a usable device the calls fail with FKD_NO_DEVICE.
#include <algorithm>
#include <immintrin.h>
#include <chrono>
#include <atomic>
#include <cmath>
#include <memory>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <string>
#include <new>
#include <thread>
#include <vector>

#include "fkd_b200.h"
#include "build.cuh"
#include "knobs.hpp"
#include "order.cuh"
#include "trace.cuh"
#include "walk.cuh"
#include "walk_inst.cuh"

namespace fkd {
namespace {

thread_local std::string g_err;

fkd_status fail(fkd_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

#define FKD_CUDA(expr)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(FKD_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

constexpr int64_t kSortChunk = int64_t(1) << 30;  // u32 ids, int item counts in CUB
// Block timeline buffer (fkd_debug_block_trace; FKD_BLOCK_TRACE builds only)
struct BlockTraceConfig {
    BlockTraceRec* buf = nullptr;
    unsigned long long* next = nullptr;
    long long cap = 0;
};
BlockTraceConfig g_btrace;

constexpr int kSmallWords = 64;   // per-workspace device counters (Workspace::small)
constexpr int kCountFlag = 12;    // host pipeline: a walked count differed from the host-written one
constexpr int kBatchTotals = 16;  // first per-batch totals word
constexpr int kMaxGroup = (kSmallWords - kBatchTotals) / 3;  // batches per host pipeline

constexpr int kMaxRegDim = 16;  // dims with compile-time walk kernels (larger: the heap kernel)
int walk_bucket_of(int k);
int walk_bucket_of(int k, int dim, bool stats = false, bool unordered = false);
// The rounds run for register lists of <= 4 slots (fcp, k <= 4) and, in
// batches of >= 2^22 queries, 8 slots (a 1M-query kNN8 batch is 4-8% slower
// with them: the round boundaries cost more than the small batch's warps lose).
// From 7-D up walks are thousands of trips long (8-D kNN16: ~6k with box
// pruning): kNN lists take no rounds and a first budget of 8192 trips, fcp
// 1024 (8-D, M = 1M: kNN16 123 -> 101 ms, kNN8 85 -> 73, fcp 33.6 -> 28.2;
// 5-D / 6-D indifferent; profiles/r02/r02ad_budget_hd.log).
constexpr int kLongWalkDim = 7;
inline bool rounds_on(int k, int64_t m, const Knobs& kn, int dim) {
    const int kb = walk_bucket_of(k);
    if (dim >= kLongWalkDim && k > 1) return false;
    return kb <= 4 || (kb == 8 && m >= kn.rounds_min_m);
}
// From 12-D nearly every walk outgrows any first budget, and parking them
// all only to finish them in the resume / CTA passes costs more than one
// walk to the end (M = 1M, N = 1M: 12-D kNN8 1026 -> 846 ms, 16-D 21.1 ->
// 5.8 s; 10-D keeps the budget, 37 vs 49 ms; profiles/r02/r02bd_hd_budget_ab.log)
constexpr int kNoBudgetDim = 12;
// Batches of a few hundred queries walk without a budget below the long-walk
// dims (the rounds, resume and CTA passes would be five more launches and
// counter resets on a call whose time is launches plus its longest walk) and
// without the Morton sort (FKD_MORTON_MIN_M): C3 tree, pinned call, M = 1 /
// 10 / 100: fcp 82 / 108 / 117 -> 62 / 84 / 95 us, kNN8 82 / 146 / 160 -> 69 /
// 134 / 150 us (tools/latency.py, profiles/r02/r02bf_small_batch_*.log).
// Parking them all into the CTA pass instead is slower for kNN (160 us at M = 1).
#ifndef FKD_SMALL_BATCH
#define FKD_SMALL_BATCH 512
#endif
// first walk's loop trips before a query parks (FKD_BUDGET < 0: per kind; 0: no budget)
inline int first_budget(int k, int64_t m, const Knobs& kn, int dim) {
    if (dim >= kNoBudgetDim || (m < FKD_SMALL_BATCH && dim < kLongWalkDim)) return 0;
    if (dim >= kLongWalkDim) return k == 1 ? 1024 : 8192;
    if (k == 1) return 112;
    if (!rounds_on(k, m, kn, dim)) return 3072;
    return walk_bucket_of(k) <= 4 ? 256 : 384;
}
// resume pass trips (FKD_RESUME_TRIPS = 0): 4 x the per-kind budget without rounds
// kNN: 8-D kNN16 (C4) 12288 -> 49152 cuts the CTA pass 269 -> 61 ms and the batch 353 -> 318 ms;
// 4-D kNN16/50/64 and 5-D kNN16 finish inside 12288 (unchanged); tools/tail8d_ab2.sh
inline int resume_trips_default(int k) { return k == 1 ? 4096 : 49152; }

// Continuation-round schedule (knobs.hpp): measured (tools/rounds_ab.sh,
// tools/rounds_knn_ab.sh, profiles/r01e_rounds_*): fcp walk -14% (3-D C3) to
// -30% (4-D), kNN4 4-D -18%, kNN8 walk + tail -3% (C3) / -7% (4-D); for lists
// of >= 16 slots parking costs more than the denser warps save (2-D kNN16 +2%,
// 4-D kNN20 +48%), so those keep one long budgeted walk.  fcp batches below
// 2^22 queries stop after two rounds: their few parked walks finish sooner in
// the CTA pass than in a latency-bound 448-trip round (clustered 1.25M / 2.5M:
// -22% / -13%), while at 10M the third round keeps the resume pass off (C3 fcp
// 2.49 vs 3.03 ms without it; profiles/r01i_fcp_*ab.log).
const std::vector<int>& round_schedule(const Knobs& kn, int k, int64_t m, int dim) {
    static const std::vector<int> none;
    if (k == 1) return (kn.rounds_fcp_env || m >= kn.rounds_min_m) ? kn.rounds_fcp : kn.rounds_fcp_small;
    if (kn.rounds_knn_all) return kn.rounds_knn_env;
    if (!rounds_on(k, m, kn, dim)) return none;
    return walk_bucket_of(k) <= 4 ? kn.rounds_knn4 : kn.rounds_knn8;
}

// The store starts node_shift() empty slots into its allocation.  With one
// slot, siblings 2c+1 / 2c+2 share an aligned pair of slots (for 16-byte
// nodes: one 32-byte sector) instead of straddling two, so the far child's
// sector usually arrived with the close child's.  Measured
// (tools/node_shift_ab.sh, profiles/r01j_node_shift_ab.log): C3 kNN8 walk
// -1.6%, fcp -1.5%, uniform kNN8 -0.8%, 4-D kNN16 -1%; -DFKD_NODE_SHIFT=0
// restores the unshifted store.
#ifndef FKD_NODE_SHIFT
#define FKD_NODE_SHIFT 1
#endif
constexpr int64_t node_shift() { return FKD_NODE_SHIFT; }

// Store layout: padded vectors (1, 4, 4, 4, 8, 8, 8, 8 floats); building with
// -DFKD_PACKED_LAYOUT=1 keeps 2-D and 3-D nodes at 8 and 12 bytes (SURVEY §7
// step 3: chosen by measurement).
#ifndef FKD_PACKED_LAYOUT
#define FKD_PACKED_LAYOUT 0
#endif
int store_stride(int dim) {
    constexpr bool packed = FKD_PACKED_LAYOUT != 0;
    switch (dim) {
        case 1: return 1;
        case 2: return packed ? 2 : 4;  // 16-byte nodes with the split plane: 2-D kNN16 -1%, fcp -3%
        case 3: return packed ? 3 : 4;
        case 4: return 4;
        case 5: case 6: case 7: case 8: return 8;
        case 9: case 10: case 11: return 12;  // three 16-byte vectors, the split plane in the last float
        case 12: case 13: case 14: case 15: case 16: return 16;
        default: return dim;
    }
}

struct Workspace {
    int device = 0;
    cudaStream_t stream = nullptr;  // own stream (host path)
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // host path: this slot's last H2D / walk / D2H completion (timing disabled)
    cudaEvent_t pe[4] = {nullptr, nullptr, nullptr, nullptr};  // [3]: walk -> tail stream hand-off
    cudaStream_t cin = nullptr, cout = nullptr;  // copy streams (first slot of a call)
    cudaStream_t tail = nullptr;                 // high-priority stream for the tail passes
    uint32_t* keys = nullptr;       // [2 * cap] keys in/out
    uint32_t* ids = nullptr;        // [2 * cap] ids in/out
    int64_t key_cap = 0;
    void* sort_tmp = nullptr;
    size_t sort_tmp_bytes = 0;
    // [kSmallWords]: 0 bad, 1-3 steps/visited/processed, 5-6 ovf count/next,
    // 8 resume count, 10 round count, 12 count flag; from kBatchTotals: 3 totals per batch
    // of a multi-batch host pipeline
    unsigned long long* small = nullptr;
    uint32_t* ovf = nullptr;                // overflow query ids
    int64_t ovf_cap = 0;
    uint32_t* wave_ids = nullptr;           // [2 * cap] parked-id lists (rounds, resume pass)
    int64_t wave_cap = 0;
    int2* wave_state = nullptr;             // [cap]
    int64_t wave_state_cap = 0;
    unsigned long long* h_small = nullptr;  // pinned mirror
    // host-path staging
    float* q = nullptr;
    int64_t q_cap = 0;
    int32_t* counts = nullptr;
    int64_t c_cap = 0;
    fkd_hit* hits = nullptr;
    int64_t h_cap = 0;

    ~Workspace() {
        cudaSetDevice(device);
        cudaFree(keys);
        cudaFree(ids);
        cudaFree(sort_tmp);
        cudaFree(ovf);
        cudaFree(wave_ids);
        cudaFree(wave_state);
        cudaFree(small);
        cudaFreeHost(h_small);
        cudaFree(q);
        cudaFree(counts);
        cudaFree(hits);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : pe)
            if (e) cudaEventDestroy(e);
        if (cin) cudaStreamDestroy(cin);
        if (tail) cudaStreamDestroy(tail);
        if (cout) cudaStreamDestroy(cout);
        if (stream) cudaStreamDestroy(stream);
    }
};

template <class T>
cudaError_t grow(T*& p, int64_t& cap, int64_t need) {
    if (need <= cap) return cudaSuccess;
    cudaFree(p);
    p = nullptr;
    cap = 0;
    const int64_t want = std::max<int64_t>(need, 1024);
    cudaError_t e = cudaMalloc(&p, size_t(want) * sizeof(T));
    if (e == cudaSuccess) cap = want;
    return e;
}

struct Replica {
    int device = 0;
    float* alloc = nullptr;  // node_shift() + n slots of stride floats
    float* nodes = nullptr;  // alloc + node_shift() * stride: node i's slot
    std::mutex mu;
    std::vector<Workspace*> pool;

    ~Replica() {
        for (Workspace* w : pool) delete w;
        cudaSetDevice(device);
        cudaFree(alloc);
    }
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// ---- pageable caller buffers -------------------------------------------
// The reference's callers hold queries and results in std::vector (pageable
// memory).  cudaMemcpyAsync from/to pageable memory is staged by the driver
// one copy at a time and blocks the host (21 GB/s D2H measured, and the
// chunk pipeline serialises behind it: C3 kNN8 64 ms instead of 16 ms).
// fkd_run_batch instead stages pageable buffers through pooled pinned
// buffers of its own, moved by a host copy pool (up to 16 threads, streaming
// stores: while the copy engine writes into pinned memory, 16 threads copy
// pinned -> warm pageable memory at ~63 GB/s, above the PCIe rate), so the
// DMA engines stream nearly as with pinned caller buffers
// (tools/micro/host_copy.cpp, copy_contention.cpp).
class CopyPool {
  public:
    static CopyPool& get() {
        static CopyPool* p = new CopyPool();  // never destroyed: workers may outlive static teardown
        return *p;
    }
    int parts() const { return int(workers_.size()) + 1; }
    // Runs f(0..parts-1) in parallel (part 0 on the caller) and waits.
    template <class F>
    void run(int parts, F&& f) {
        struct Group {
            std::mutex mu;
            std::condition_variable cv;
            int left = 0;
        } g;
        g.left = parts - 1;
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (int i = 1; i < parts; ++i)
                tasks_.push_back([&g, &f, i] {
                    f(i);
                    std::lock_guard<std::mutex> l2(g.mu);
                    if (--g.left == 0) g.cv.notify_one();
                });
        }
        cv_.notify_all();
        f(0);
        std::unique_lock<std::mutex> lk(g.mu);
        g.cv.wait(lk, [&] { return g.left == 0; });
    }

  private:
    CopyPool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const int want = read_knobs().copy_threads;
        // every hardware thread up to 16: with streaming stores the copy
        // scales to 16 threads while the copy engine writes (C3 pageable
        // call 29.5 -> 24.5-26.3 ms against 8 threads and memcpy,
        // profiles/r02/r02ao_copy_pool_ab.log)
        const int n = (want > 0 ? want : int(std::min(16u, hw))) - 1;  // + the calling thread
        for (int i = 0; i < n; ++i)
            workers_.emplace_back([this] {
                for (;;) {
                    std::function<void()> t;
                    {
                        std::unique_lock<std::mutex> lk(mu_);
                        cv_.wait(lk, [&] { return !tasks_.empty(); });
                        t = std::move(tasks_.front());
                        tasks_.pop_front();
                    }
                    t();
                }
            });
        for (auto& w : workers_) w.detach();
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> tasks_;
    std::vector<std::thread> workers_;
};

// memcpy with non-temporal (streaming) stores: the destination lines are
// written whole without being read first (no read-for-ownership), which
// glibc's memcpy does only above a size threshold the pool's per-thread
// pieces stay under.  Falls back to memcpy without AVX2.
__attribute__((target("avx2"))) void stream_copy_avx2(char* d, const char* s, size_t n) {
    const size_t head = std::min(n, size_t((64 - (reinterpret_cast<uintptr_t>(d) & 63)) & 63));
    std::memcpy(d, s, head);
    d += head;
    s += head;
    n -= head;
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 64));
        const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), e);
    }
    std::memcpy(d + i, s + i, n - i);
    _mm_sfence();
}

// std::fill with streaming stores (whole lines, no read-for-ownership).
__attribute__((target("avx2"))) void stream_fill_avx2(int32_t* d, int64_t n, int32_t v) {
    int64_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = v;
    const __m256i x = _mm256_set1_epi32(v);
    for (; i + 8 <= n; i += 8) _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), x);
    for (; i < n; ++i) d[i] = v;
    _mm_sfence();
}

void copy_piece(char* d, const char* s, size_t n, bool stream) {
    static const bool avx2 = __builtin_cpu_supports("avx2");
    if (stream && avx2 && n >= (size_t(1) << 20))
        stream_copy_avx2(d, s, n);
    else
        std::memcpy(d, s, n);
}

void par_copy(void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    CopyPool& pool = CopyPool::get();
    static const bool stream = read_knobs().stream_copy;
    const int parts = bytes < (size_t(4) << 20) ? 1 : pool.parts();
    if (parts == 1) {
        copy_piece(static_cast<char*>(dst), static_cast<const char*>(src), bytes, stream);
        return;
    }
    const size_t per = ((bytes + parts - 1) / parts + 4095) & ~size_t(4095);
    pool.run(parts, [&](int i) {
        const size_t lo = std::min(bytes, size_t(i) * per), hi = std::min(bytes, lo + per);
        if (hi > lo) copy_piece(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo, stream);
    });
}

void par_fill(int32_t* dst, int64_t count, int32_t v) {
    if (count <= 0) return;
    CopyPool& pool = CopyPool::get();
    const int parts = count < (int64_t(1) << 20) ? 1 : pool.parts();
    const int64_t per = ((count + parts - 1) / parts + 1023) & ~int64_t(1023);
    static const bool stream = read_knobs().stream_copy && __builtin_cpu_supports("avx2");
    auto part = [&](int i) {
        const int64_t lo = std::min(count, int64_t(i) * per), hi = std::min(count, lo + per);
        if (stream && hi - lo >= (int64_t(1) << 18))
            stream_fill_avx2(dst + lo, hi - lo, v);
        else
            std::fill(dst + lo, dst + hi, v);
    };
    if (parts == 1) part(0); else pool.run(parts, part);
}

// First non-finite float of p[0, count) or -1 (require_finite, point.hpp:59-63:
// a float is non-finite iff its exponent bits are all ones).  The block OR is
// branch-free so the compiler vectorises it; the exact index is searched
// only inside a block that has one.
int64_t first_nonfinite(const float* p, int64_t count) {
    const uint32_t* u = reinterpret_cast<const uint32_t*>(p);
    constexpr int64_t kBlock = 4096;
    for (int64_t b = 0; b < count; b += kBlock) {
        const int64_t e = std::min(count, b + kBlock);
        uint32_t any = 0;
        for (int64_t i = b; i < e; ++i) any |= uint32_t((u[i] & 0x7f800000u) == 0x7f800000u);
        if (any)
            for (int64_t i = b; i < e; ++i)
                if ((u[i] & 0x7f800000u) == 0x7f800000u) return i;
    }
    return -1;
}

// par_copy + first_nonfinite of the copied floats (dst is cache-hot per
// 256 KB piece).  Returns the first non-finite float index or -1.
int64_t par_copy_check(float* dst, const float* src, int64_t count) {
    if (count <= 0) return -1;
    CopyPool& pool = CopyPool::get();
    const size_t bytes = size_t(count) * sizeof(float);
    const int parts = bytes < (size_t(4) << 20) ? 1 : pool.parts();
    const int64_t per = ((count + parts - 1) / parts + 1023) & ~int64_t(1023);
    std::vector<int64_t> first(size_t(parts), -1);
    auto part = [&](int i) {
        const int64_t lo = std::min(count, int64_t(i) * per), hi = std::min(count, lo + per);
        constexpr int64_t kPiece = 65536;  // floats
        for (int64_t b = lo; b < hi; b += kPiece) {
            const int64_t n = std::min(kPiece, hi - b);
            std::memcpy(dst + b, src + b, size_t(n) * sizeof(float));
            if (first[size_t(i)] < 0) {
                const int64_t f = first_nonfinite(dst + b, n);
                if (f >= 0) first[size_t(i)] = b + f;
            }
        }
    };
    if (parts == 1) part(0); else pool.run(parts, part);
    for (int64_t f : first)
        if (f >= 0) return f;
    return -1;
}

// first_nonfinite over the copy pool (read-only).
int64_t par_check(const float* src, int64_t count) {
    if (count <= 0) return -1;
    CopyPool& pool = CopyPool::get();
    const int parts = count < (int64_t(1) << 20) ? 1 : pool.parts();
    const int64_t per = ((count + parts - 1) / parts + 1023) & ~int64_t(1023);
    std::vector<int64_t> first(size_t(parts), -1);
    auto part = [&](int i) {
        const int64_t lo = std::min(count, int64_t(i) * per), hi = std::min(count, lo + per);
        const int64_t f = first_nonfinite(src + lo, hi - lo);
        if (f >= 0) first[size_t(i)] = lo + f;
    };
    if (parts == 1) part(0); else pool.run(parts, part);
    for (int64_t f : first)
        if (f >= 0) return f;
    return -1;
}

bool is_pageable(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

// Pooled pinned host staging (portable across devices), grown on demand.
struct HostStage {
    char* p = nullptr;
    size_t cap = 0;
};
std::mutex g_stage_mu;
std::vector<HostStage> g_stage_pool;

cudaError_t acquire_stage(size_t bytes, HostStage* out) {
    {
        // best fit: the smallest pooled buffer that holds `bytes`, else the
        // largest (re-allocated below), so a call's query and result rings
        // each find their own buffer again on the next call
        std::lock_guard<std::mutex> lk(g_stage_mu);
        auto best = g_stage_pool.end();
        for (auto it = g_stage_pool.begin(); it != g_stage_pool.end(); ++it) {
            if (best == g_stage_pool.end()) {
                best = it;
                continue;
            }
            const bool fits = it->cap >= bytes, best_fits = best->cap >= bytes;
            if ((fits && (!best_fits || it->cap < best->cap)) || (!fits && !best_fits && it->cap > best->cap))
                best = it;
        }
        if (best != g_stage_pool.end()) {
            *out = *best;
            g_stage_pool.erase(best);
        }
    }
    if (out->cap >= bytes) return cudaSuccess;
    cudaFreeHost(out->p);
    *out = HostStage{};
    void* p = nullptr;
    cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable);
    if (e == cudaSuccess) *out = HostStage{static_cast<char*>(p), bytes};
    return e;
}

// The pool keeps at most kStagePoolMax buffers of at most kStageKeepMax
// bytes each; anything else goes back to the OS at release, so a huge batch
// never leaves gigabytes pinned (staging is a bounded per-chunk ring, so a
// call needs at most slots x chunk bytes).
constexpr size_t kStageKeepMax = size_t(2) << 30;
constexpr size_t kStagePoolMax = 8;

void release_stage(HostStage s) {
    if (!s.p) return;
    if (s.cap > kStageKeepMax) {
        cudaFreeHost(s.p);
        return;
    }
    HostStage drop{};
    {
        std::lock_guard<std::mutex> lk(g_stage_mu);
        g_stage_pool.push_back(s);
        if (g_stage_pool.size() > kStagePoolMax) {
            auto smallest = std::min_element(g_stage_pool.begin(), g_stage_pool.end(),
                                             [](const HostStage& a, const HostStage& b) { return a.cap < b.cap; });
            drop = *smallest;
            g_stage_pool.erase(smallest);
        }
    }
    if (drop.p) cudaFreeHost(drop.p);
}

}  // namespace

const char* set_host_error(const std::string& msg) {
    g_err = msg;
    return g_err.c_str();
}

}  // namespace fkd

struct fkd_tree {
    int64_t n = 0;
    int32_t dim = 0;
    int32_t stride = 0;
    fkd::MortonFrame frame{};
    std::vector<fkd::Replica*> reps;
};

namespace fkd {
namespace {

fkd_status acquire_ws(Replica& r, Workspace** out) {
    {
        std::lock_guard<std::mutex> lk(r.mu);
        if (!r.pool.empty()) {
            *out = r.pool.back();
            r.pool.pop_back();
            return FKD_OK;
        }
    }
    auto* w = new Workspace();
    w->device = r.device;
    DeviceGuard g(r.device);
    cudaError_t e = cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking);
    for (auto& ev : w->ev)
        if (e == cudaSuccess) e = cudaEventCreate(&ev);
    for (auto& ev : w->pe)
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&w->cin, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&w->cout, cudaStreamNonBlocking);
    if (e == cudaSuccess) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        e = cudaStreamCreateWithPriority(&w->tail, cudaStreamNonBlocking, hi);
    }
    if (e == cudaSuccess) e = cudaMalloc(&w->small, kSmallWords * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMallocHost(&w->h_small, kSmallWords * sizeof(unsigned long long));
    if (e != cudaSuccess) {
        delete w;
        return fail(FKD_CUDA_ERROR, std::string("workspace: ") + cudaGetErrorString(e));
    }
    *out = w;
    return FKD_OK;
}

void release_ws(Replica& r, Workspace* w) {
    std::lock_guard<std::mutex> lk(r.mu);
    r.pool.push_back(w);
}

// Largest k on a register list (larger k: the heap kernel).
#ifndef FKD_REG_MAXK
#define FKD_REG_MAXK 64
#endif
// Register-list walks exist for dims 1..kMaxRegDim; dims 9..16 carry the
// buckets 1 / 8 / 16 / 32 / 64 only (k rounds up; the unused leading slots
// hold the dummy key), which keeps their eight kernel sets small.
int walk_bucket_of(int k, int dim, bool stats, bool unordered) {
    if (k > FKD_REG_MAXK || dim > kMaxRegDim) return 0;
    if (dim > 8 && (stats || unordered)) return 0;  // 9..16-D register walks: production (ordered) only
    if (dim > 8) return k <= 1 ? 1 : (k <= 8 ? 8 : (k <= 16 ? 16 : (k <= 32 ? 32 : 64)));
    return walk_bucket_of(k);
}
int walk_bucket_of(int k) {
    if (k > FKD_REG_MAXK) return 0;
    if (k <= 1) return 1;
    if (k <= 2) return 2;
    if (k <= 4) return 4;
    if (k <= 8) return 8;
    if (k <= 16) return 16;
    if (k <= 20) return 20;
    if (k <= 32) return 32;
    if (k <= 50) return 50;
    if (k <= 64) return 64;
    return 0;
}

// Validation of batch.cpp:72-80, in the reference's order.
fkd_status validate(const fkd_tree* t, int64_t m, int32_t dim, const fkd_batch_options* o,
                    float* cap2) {
    if (!t) return fail(FKD_INVALID_ARGUMENT, "null tree");
    if (!o) return fail(FKD_INVALID_ARGUMENT, "null options");
    if (o->kind != FKD_FCP && o->kind != FKD_KNN)
        return fail(FKD_INVALID_ARGUMENT, "unknown query kind");
    if (o->kind == FKD_KNN && o->k < 1) return fail(FKD_INVALID_ARGUMENT, "knn: k must be >= 1");
    if (std::isnan(o->max_radius) || o->max_radius < 0.0f)
        return fail(FKD_DATA_ERROR, "max radius must be >= 0 or inf");
    if (o->engine != FKD_ENGINE_STACK_FREE && o->engine != FKD_ENGINE_RECURSIVE)
        return fail(FKD_INVALID_ARGUMENT, "unknown engine");
    if (m < 0) return fail(FKD_INVALID_ARGUMENT, "negative query count");
    if (t->n > 0 && m > 0 && dim != t->dim)
        return fail(FKD_DATA_ERROR, "query dimension " + std::to_string(dim) +
                                        " does not match tree dimension " + std::to_string(t->dim));
    if (dim < 1 && m > 0) return fail(FKD_DATA_ERROR, "query dimension must be >= 1");
    *cap2 = o->max_radius * o->max_radius;  // squared_radius_cap (point.hpp:78-82)
    return FKD_OK;
}

#ifndef FKD_MORTON_MIN_M
#define FKD_MORTON_MIN_M 512
#endif
bool use_morton(const fkd_tree* t, const fkd_batch_options* o, int64_t m) {
    if (o->flags & FKD_FLAG_NO_MORTON) return false;
    if (!(o->flags & FKD_FLAG_MORTON)) return false;
    // from 9-D the key covers the first 8 axes; below FKD_MORTON_MIN_M queries
    // the sort's launches cost more than the order saves
    return t->n > 0 && m >= FKD_MORTON_MIN_M && t->dim <= kMaxRegDim;
}

// A Morton order computed by another batch of the same submission over the
// same query array (fkd_run_batches_device): its walk order, the flag its key
// pass checked the queries into, and the event after which both are ready.
struct SharedOrder {
    const uint32_t* order = nullptr;
    unsigned long long* bad = nullptr;
    cudaEvent_t ready = nullptr;
};

// Enqueues one batch (device pointers) on `st`; no synchronisation.  Writes
// the first bad query id and the stat totals into w->small (with a shared
// order: into the sorting batch's flag).  `ev_sorted`, if given, is recorded
// once the walk order exists.
fkd_status enqueue(const fkd_tree* t, Replica& r, Workspace* w, const float* d_q, int64_t m,
                   const fkd_batch_options* o, float cap2, int32_t* d_counts, fkd_hit* d_hits,
                   fkd_query_stats* d_per_query, bool stats, cudaStream_t st, int* launches,
                   int* walk_launches, const Knobs& tu, cudaEvent_t ev_mid, cudaEvent_t ev_tail = nullptr,
                   int64_t id_offset = 0, cudaStream_t tail_st = nullptr, int budget_div = 1,
                   const SharedOrder* share = nullptr, cudaEvent_t ev_sorted = nullptr,
                   unsigned long long* totals = nullptr) {
    const int k = o->kind == FKD_KNN ? o->k : 1;
    if (t->n == 0) {  // every query returns empty; queries are not read (batch.cpp:75)
        *launches += fill_empty(d_counts, d_hits, m, k, st);
        FKD_CUDA(cudaGetLastError());
        return FKD_OK;
    }
    if (share && share->order) {  // ordered (and checked) by the sorting batch
        FKD_CUDA(cudaStreamWaitEvent(st, share->ready, 0));
        if (ev_mid) FKD_CUDA(cudaEventRecord(ev_mid, st));
    }
    const bool sort = use_morton(t, o, m) && !(share && share->order);
    // sub-batches of <= 2^30 positions: u32 ids in the sort and int32 query ids in the walk
    const int64_t chunk = std::min<int64_t>(m, kSortChunk);
    if (sort) {
        if (2 * chunk > w->key_cap) {
            cudaFree(w->keys);
            cudaFree(w->ids);
            w->keys = w->ids = nullptr;
            w->key_cap = 0;
            FKD_CUDA(cudaMalloc(&w->keys, size_t(2 * chunk) * sizeof(uint32_t)));
            FKD_CUDA(cudaMalloc(&w->ids, size_t(2 * chunk) * sizeof(uint32_t)));
            w->key_cap = 2 * chunk;
        }
        const size_t need = morton_temp_bytes(chunk, t->dim);
        if (need > w->sort_tmp_bytes) {
            cudaFree(w->sort_tmp);
            w->sort_tmp = nullptr;
            w->sort_tmp_bytes = 0;
            FKD_CUDA(cudaMalloc(&w->sort_tmp, need));
            w->sort_tmp_bytes = need;
        }
    }
    // require_finite(queries) (batch.cpp:79) over the WHOLE batch before any
    // walk writes a slot: the key pass checks each sub-batch it sorts; a batch
    // of several sub-batches, or one walked without the key pass, is scanned
    // first.  The walk kernels exit at entry once *bad is set.
    if ((!sort || m > chunk || t->dim > 8) && !(share && share->order)) {  // from 9-D the key pass reads 8 axes
        *launches += scan_queries(d_q, m, t->dim, w->small, id_offset, st);
        FKD_CUDA(cudaGetLastError());
    }
    for (int64_t base = 0; base < m; base += chunk) {
        const int64_t cm = std::min(chunk, m - base);
        WalkArgs a{};
        a.nodes = r.nodes;
        a.btrace = g_btrace.buf;  // tag: the list length (fcp 1) and the kernel phase
        a.btrace_next = g_btrace.next;
        a.btrace_cap = g_btrace.cap;
        a.btrace_tag = uint32_t(k) << 8;
        a.n = int32_t(t->n);
        a.dim = t->dim;
        a.stride = t->stride;
        a.queries = d_q + base * t->dim;
        a.m = cm;
        a.cap2 = cap2;
        a.k = k;
        a.recursive_stats = o->engine == FKD_ENGINE_RECURSIVE;
        a.counts = d_counts + base;
        a.hits = d_hits + base * k;
        a.totals = totals ? totals : w->small + 1;
        a.per_query = d_per_query ? d_per_query + base : nullptr;
        a.bad = w->small;
        a.id_base = id_offset + base;
        int budget = tu.budget >= 0 ? tu.budget : first_budget(k, cm, tu, t->dim);
        if (budget_div > 1 && budget > 0) budget = std::max(64, budget / budget_div);
        a.budget = (stats || walk_bucket_of(k, t->dim, stats, (o->flags & FKD_FLAG_UNORDERED) != 0) == 0) ? 0 : budget;
        if (a.budget > 0) {
            FKD_CUDA(grow(w->ovf, w->ovf_cap, cm));
            FKD_CUDA(grow(w->wave_state, w->wave_state_cap, cm));
            FKD_CUDA(grow(w->wave_ids, w->wave_cap, 2 * cm));
            a.ovf_ids = w->ovf;
            a.ovf_count = w->small + 5;
            a.ovf_next = w->small + 6;
            a.wave_state = w->wave_state;
            FKD_CUDA(cudaMemsetAsync(w->small + 5, 0, 2 * sizeof(unsigned long long), st));
            // a GPU-full of over-budget queries is bulk work, not a tail
            int dev = 0, sms = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            a.resume_min = tu.resume_min > 0 ? tu.resume_min : int64_t(sms) * 64;
        }
        if (sort) {
            const int64_t half = w->key_cap / 2;
            const int rc = morton_order(a.queries, cm, t->dim, t->frame, w->keys, w->keys + half,
                                        w->ids, w->ids + half, w->sort_tmp, w->sort_tmp_bytes, w->small,
                                        a.id_base, st);
            if (rc < 0) return fail(FKD_CUDA_ERROR, "morton ordering failed");
            *launches += rc;
            a.order = w->ids + half;
            if (ev_sorted) FKD_CUDA(cudaEventRecord(ev_sorted, st));
        } else if (share && share->order) {
            a.order = share->order;
            a.bad = share->bad;
        }
        if (ev_mid && base == 0) FKD_CUDA(cudaEventRecord(ev_mid, st));
        const bool unordered = (o->flags & FKD_FLAG_UNORDERED) != 0;
        int nl = 0;
        {
            nl = launch_walk(a, t->dim, t->stride, stats, unordered, 0, st);
            if (nl <= 0) return fail(FKD_CUDA_ERROR, "no kernel for this configuration");
            FKD_CUDA(cudaGetLastError());
            if (a.budget > 0 && tail_st) {
                // the tail passes run on a high-priority stream so that, in a
                // pipeline of concurrent chunks, they take SM slots as soon as
                // blocks retire instead of queueing behind the next chunks' walks
                FKD_CUDA(cudaEventRecord(w->pe[3], st));
                FKD_CUDA(cudaStreamWaitEvent(tail_st, w->pe[3], 0));
            }
            const cudaStream_t ts = (a.budget > 0 && tail_st) ? tail_st : st;
            const std::vector<int>& rounds = round_schedule(tu, k, cm, t->dim);
            if (a.budget > 0 && !rounds.empty()) {
                // continuation rounds: the parked walks, compacted into dense
                // warps, continue for `trips` more trips per round; lists
                // ping-pong between ovf_ids and the upper half of wave_ids
                const int64_t half = w->wave_cap / 2;
                uint32_t* lists[2] = {a.ovf_ids, w->wave_ids + half};
                unsigned long long* cnts[2] = {a.ovf_count, w->small + 10};
                int cur = 0;
                for (int trips : rounds) {
                    WalkArgs r = a;
                    r.trips = trips;
                    r.resume_min = 0;  // every round runs, whatever the count
                    r.wave_in = lists[cur];
                    r.wave_n_in = cnts[cur];
                    r.wave_out = lists[cur ^ 1];
                    r.wave_n_out = cnts[cur ^ 1];
                    FKD_CUDA(cudaMemsetAsync(cnts[cur ^ 1], 0, sizeof(unsigned long long), ts));
                    nl += launch_walk(r, t->dim, t->stride, stats, unordered, 3, ts);
                    FKD_CUDA(cudaGetLastError());
                    cur ^= 1;
                }
                a.ovf_ids = lists[cur];
                a.ovf_count = cnts[cur];
            }
            if (a.budget > 0) {
                // resume pass: one more round (walk_round_kernel), run only
                // when at least resume_min walks are still parked (decided on
                // the device: bulk long walks, e.g. 8-D), for at most
                // resume_trips more steps; its survivors (parked again) are the
                // CTA pass's list
                FKD_CUDA(cudaMemsetAsync(w->small + 8, 0, sizeof(unsigned long long), ts));
                a.wave_out = w->wave_ids;
                a.wave_n_out = w->small + 8;
                WalkArgs r = a;
                r.trips = tu.resume_trips > 0 ? tu.resume_trips
                                              : (tu.resume_trips < 0 ? 0x7fffffff : resume_trips_default(k));
                r.wave_in = a.ovf_ids;
                r.wave_n_in = a.ovf_count;
                nl += launch_walk(r, t->dim, t->stride, stats, unordered, 3, ts);
                FKD_CUDA(cudaGetLastError());
            }
        }
        const cudaStream_t ts = (a.budget > 0 && tail_st) ? tail_st : st;
        if (ev_tail && base == 0) FKD_CUDA(cudaEventRecord(ev_tail, ts));
        const int tail = launch_walk(a, t->dim, t->stride, stats, unordered, 1, ts);  // overflow pass
        FKD_CUDA(cudaGetLastError());
        if (ts != st) {
            FKD_CUDA(cudaEventRecord(w->pe[3], ts));
            FKD_CUDA(cudaStreamWaitEvent(st, w->pe[3], 0));
        }
        *launches += nl + tail;
        *walk_launches += nl + tail;
    }
    return FKD_OK;
}

}  // namespace


int launch_walk(const WalkArgs& a, int dim, int stride, bool stats, bool unordered, int phase,
                cudaStream_t st) {
    const int KB = walk_bucket_of(a.k, dim, stats, unordered);
    if (KB == 0) return phase == 0 ? launch_walk_heap(a, dim, stats, unordered, st) : 0;
    switch (dim) {
        case 1: return launch_walk_d1(a, stride, KB, stats, unordered, phase, st);
        case 2: return launch_walk_d2(a, stride, KB, stats, unordered, phase, st);
        case 3: return launch_walk_d3(a, stride, KB, stats, unordered, phase, st);
        case 4: return launch_walk_d4(a, stride, KB, stats, unordered, phase, st);
        case 5: return launch_walk_d5(a, stride, KB, stats, unordered, phase, st);
        case 6: return launch_walk_d6(a, stride, KB, stats, unordered, phase, st);
        case 7: return launch_walk_d7(a, stride, KB, stats, unordered, phase, st);
        case 8: return launch_walk_d8(a, stride, KB, stats, unordered, phase, st);
        case 9: return launch_walk_d9(a, stride, KB, stats, unordered, phase, st);
        case 10: return launch_walk_d10(a, stride, KB, stats, unordered, phase, st);
        case 11: return launch_walk_d11(a, stride, KB, stats, unordered, phase, st);
        case 12: return launch_walk_d12(a, stride, KB, stats, unordered, phase, st);
        case 13: return launch_walk_d13(a, stride, KB, stats, unordered, phase, st);
        case 14: return launch_walk_d14(a, stride, KB, stats, unordered, phase, st);
        case 15: return launch_walk_d15(a, stride, KB, stats, unordered, phase, st);
        case 16: return launch_walk_d16(a, stride, KB, stats, unordered, phase, st);
        default: return 0;
    }
}

}  // namespace fkd

using namespace fkd;

extern "C" {

const char* fkd_last_error(void) { return g_err.c_str(); }

const char* fkd_version(void) { return "fkd_b200 0.1 (sm_100a)"; }

void fkd_default_options(fkd_batch_options* o) {
    o->kind = FKD_FCP;
    o->k = 1;
    o->max_radius = INFINITY;
    o->engine = FKD_ENGINE_STACK_FREE;
    o->threads = 0;
    o->collect_stats = 0;
    o->flags = FKD_FLAG_MORTON;
}

void* fkd_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
    return p;
}

void fkd_host_free(void* p) { cudaFreeHost(p); }

int64_t fkd_tree_size(const fkd_tree* t) { return t ? t->n : 0; }
int32_t fkd_tree_dim(const fkd_tree* t) { return t ? t->dim : 0; }

fkd_status fkd_morton_keys(const fkd_tree* t, const float* d_queries, int64_t m, int32_t dim, uint32_t* d_keys,
                           int32_t* key_bits, void* stream) {
    if (!t) return fail(FKD_INVALID_ARGUMENT, "null tree");
    if (key_bits) *key_bits = t->n > 0 ? t->frame.bits * std::min(t->dim, 8) : 0;
    if (m < 0) return fail(FKD_INVALID_ARGUMENT, "negative query count");
    if (m == 0 || t->n == 0) return FKD_OK;
    if (dim != t->dim)
        return fail(FKD_DATA_ERROR, "query dimension " + std::to_string(dim) + " does not match tree dimension " +
                                        std::to_string(t->dim));
    if (t->reps.empty()) return fail(FKD_NO_DEVICE, "tree has no device replica");
    DeviceGuard g(t->reps[0]->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned long long* bad = nullptr;
    FKD_CUDA(cudaMallocAsync(&bad, sizeof(unsigned long long), st));
    FKD_CUDA(cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), st));
    if (morton_keys(d_queries, m, dim, t->frame, d_keys, bad, st) < 0) return fail(FKD_CUDA_ERROR, "morton keys");
    if (dim > 8) scan_queries(d_queries, m, dim, bad, 0, st);  // the key reads the first 8 axes
    FKD_CUDA(cudaGetLastError());
    unsigned long long h = 0;
    FKD_CUDA(cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, st));
    FKD_CUDA(cudaFreeAsync(bad, st));
    FKD_CUDA(cudaStreamSynchronize(st));
    if (h != kNoBad) return fail(FKD_DATA_ERROR, "queries: non-finite coordinate in point " + std::to_string(h));
    return FKD_OK;
}

fkd_status fkd_debug_block_trace(void* d_records, void* d_counter, int64_t cap) {
    if (d_records && !FKD_BLOCK_TRACE)
        return fail(FKD_INVALID_ARGUMENT, "library built without FKD_BLOCK_TRACE (make EXTRA=-DFKD_BLOCK_TRACE=1)");
    g_btrace.buf = static_cast<BlockTraceRec*>(d_records);
    g_btrace.next = static_cast<unsigned long long*>(d_counter);
    g_btrace.cap = d_records ? cap : 0;
    return FKD_OK;
}

int32_t fkd_tree_replicas(const fkd_tree* t, int32_t* devices, int32_t cap) {
    if (!t) return 0;
    const int32_t n = int32_t(t->reps.size());
    for (int32_t i = 0; devices && i < n && i < cap; ++i) devices[i] = t->reps[i]->device;
    return n;
}

void fkd_tree_destroy(fkd_tree* t) {
    if (!t) return;
    for (Replica* r : t->reps) delete r;
    delete t;
}

static fkd_status set_frame(fkd_tree* t, const float* lo, const float* hi) {
    const int dim = t->dim;
    t->frame.bits = morton_bits_per_dim(std::min(dim, 8));
    const float top = float((1u << t->frame.bits) - 1u);
    for (int d = 0; d < 8; ++d) {
        t->frame.lo[d] = 0.0f;
        t->frame.scale[d] = 0.0f;
    }
    for (int d = 0; d < dim && d < 8; ++d) {
        t->frame.lo[d] = lo[d];
        const double ext = double(hi[d]) - double(lo[d]);
        t->frame.scale[d] = ext > 0.0 ? float(top / ext) : 0.0f;
    }
    return FKD_OK;
}



static fkd_status alloc_store(Replica* r, int64_t n, int stride) {
    const int64_t sh = node_shift();
    FKD_CUDA(cudaMalloc(&r->alloc, size_t(n + sh) * stride * sizeof(float)));
    r->nodes = r->alloc + sh * stride;
    return FKD_OK;
}

static fkd_status make_replica(fkd_tree* t, int dev, const float* src, bool src_on_device,
                               cudaStream_t st) {
    auto* r = new Replica();
    r->device = dev;
    t->reps.push_back(r);
    DeviceGuard g(dev);
    const int64_t n = t->n;
    if (n == 0) return FKD_OK;
    const size_t store_bytes = size_t(n) * t->stride * sizeof(float);
    if (fkd_status e = alloc_store(r, n, t->stride); e != FKD_OK) return e;
    if (t->stride == t->dim) {
        FKD_CUDA(cudaMemcpyAsync(r->nodes, src, store_bytes,
                                 src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    } else {
        const float* dsrc = src;
        float* tmp = nullptr;
        if (!src_on_device) {
            FKD_CUDA(cudaMalloc(&tmp, size_t(n) * t->dim * sizeof(float)));
            FKD_CUDA(cudaMemcpyAsync(tmp, src, size_t(n) * t->dim * sizeof(float),
                                     cudaMemcpyHostToDevice, st));
            dsrc = tmp;
        }
        pack_nodes(dsrc, n, t->dim, t->stride, r->nodes, st);
        FKD_CUDA(cudaGetLastError());
        if (tmp) {
            FKD_CUDA(cudaStreamSynchronize(st));
            cudaFree(tmp);
        }
    }
    FKD_CUDA(cudaStreamSynchronize(st));
    return FKD_OK;
}

// Further replicas are copied device to device from the first one — one
// upload, then a fan-out of the packed store over NVLink / NVSwitch (SURVEY
// §8(e)).  The fan-out is a pipelined chain, the way a ring broadcast moves
// data: the store is cut into kFanChunk pieces and piece c hops
// dev[0] -> dev[1] -> ... -> dev[R], each hop on a stream of its destination
// device, starting as soon as piece c has arrived at the hop's source.  Every
// GPU sends and receives each byte once, so on NVSwitch (full bandwidth to
// every peer) the whole fan-out takes about (store + R x piece) / link rate
// instead of R store copies back to back (1.6 GB at C5, 8 GPUs: ~2.5 ms
// rather than ~12 ms one after another from device 0).  Peer access is
// enabled where the pair supports it; cudaMemcpyPeerAsync stages through the
// host otherwise.
static constexpr size_t kFanChunk = size_t(64) << 20;

static fkd_status fanout_replicas(fkd_tree* t, const std::vector<int>& devs) {
    if (devs.empty()) return FKD_OK;
    std::vector<Replica*> chain{t->reps.front()};
    for (int dev : devs) {
        auto* r = new Replica();
        r->device = dev;
        t->reps.push_back(r);
        chain.push_back(r);
    }
    if (t->n == 0) return FKD_OK;
    const size_t bytes = size_t(t->n + node_shift()) * t->stride * sizeof(float);
    for (size_t i = 1; i < chain.size(); ++i) {
        DeviceGuard g(chain[i]->device);
        if (fkd_status e = alloc_store(chain[i], t->n, t->stride); e != FKD_OK) return e;
        const int src = chain[i - 1]->device, dst = chain[i]->device;
        if (src != dst) {
            int can = 0;
            cudaDeviceCanAccessPeer(&can, dst, src);
            if (can) {
                cudaError_t e = cudaDeviceEnablePeerAccess(src, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (e != cudaSuccess) return fail(FKD_CUDA_ERROR, std::string("peer access: ") + cudaGetErrorString(e));
            }
        }
    }
    const size_t pieces = (bytes + kFanChunk - 1) / kFanChunk;
    const size_t hops = chain.size() - 1;
    std::vector<cudaStream_t> st(hops, nullptr);
    std::vector<cudaEvent_t> arrived(hops * pieces, nullptr);  // piece c at chain[h + 1]
    fkd_status err = FKD_OK;
    auto cuda = [&](cudaError_t e, const char* what) {
        if (e != cudaSuccess && err == FKD_OK) err = fail(FKD_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
        return e == cudaSuccess;
    };
    for (size_t h = 0; h < hops && err == FKD_OK; ++h) {
        DeviceGuard g(chain[h + 1]->device);
        cuda(cudaStreamCreateWithFlags(&st[h], cudaStreamNonBlocking), "fan-out stream");
        for (size_t c = 0; c < pieces && err == FKD_OK; ++c)
            cuda(cudaEventCreateWithFlags(&arrived[h * pieces + c], cudaEventDisableTiming), "fan-out event");
    }
    // enqueue piece-major so every hop's stream sees its pieces in order and
    // the waits name events recorded earlier in host order
    for (size_t c = 0; c < pieces && err == FKD_OK; ++c) {
        const size_t off = c * kFanChunk, len = std::min(kFanChunk, bytes - off);
        for (size_t h = 0; h < hops && err == FKD_OK; ++h) {
            DeviceGuard g(chain[h + 1]->device);
            if (h > 0 && !cuda(cudaStreamWaitEvent(st[h], arrived[(h - 1) * pieces + c], 0), "fan-out wait")) break;
            const char* from = reinterpret_cast<const char*>(chain[h]->alloc) + off;
            char* to = reinterpret_cast<char*>(chain[h + 1]->alloc) + off;
            if (!cuda(cudaMemcpyPeerAsync(to, chain[h + 1]->device, from, chain[h]->device, len, st[h]),
                      "fan-out copy"))
                break;
            cuda(cudaEventRecord(arrived[h * pieces + c], st[h]), "fan-out event");
        }
    }
    for (size_t h = 0; h < hops; ++h) {
        if (!st[h]) continue;
        DeviceGuard g(chain[h + 1]->device);
        cuda(cudaStreamSynchronize(st[h]), "fan-out");
        cudaStreamDestroy(st[h]);
    }
    for (auto& e : arrived)
        if (e) cudaEventDestroy(e);
    return err;
}

fkd_status fkd_tree_create(const float* level_order, int64_t n, int32_t dim,
                           const int32_t* devices, int32_t ndev, fkd_tree** out) {
    if (!out) return fail(FKD_INVALID_ARGUMENT, "null output");
    *out = nullptr;
    // child slots 2c+1 / 2c+2 are int32 (traverse.hpp:228-229): fine below 2^30 nodes
    if (n < 0 || n >= (int64_t(1) << 30)) return fail(FKD_DATA_ERROR, "tree size out of range (must be < 2^30)");
    if (dim < 0 || (n > 0 && dim < 1)) return fail(FKD_DATA_ERROR, "point set: negative dimension");
    if (n > 0 && !level_order) return fail(FKD_INVALID_ARGUMENT, "null tree data");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        return fail(FKD_NO_DEVICE, "no CUDA device visible (the B200 path has no CPU fallback)");
    // KdTree::from_level_order -> require_finite(nodes, "tree nodes") (tree.cpp:72)
    std::vector<float> lo(std::max(dim, 1), INFINITY), hi(std::max(dim, 1), -INFINITY);
    for (int64_t i = 0; i < n; ++i) {
        const float* p = level_order + i * dim;
        for (int d = 0; d < dim; ++d) {
            if (!std::isfinite(p[d]))
                return fail(FKD_DATA_ERROR, "tree nodes: non-finite coordinate in point " + std::to_string(i));
            lo[d] = std::min(lo[d], p[d]);
            hi[d] = std::max(hi[d], p[d]);
        }
    }
    auto* t = new fkd_tree();
    t->n = n;
    t->dim = dim;
    t->stride = store_stride(dim);
    if (n > 0) set_frame(t, lo.data(), hi.data());
    std::vector<int> devs;
    if (devices && ndev > 0) {
        devs.assign(devices, devices + ndev);
    } else {
        int cur = 0;
        cudaGetDevice(&cur);
        devs.push_back(cur);
    }
    for (const int dev : devs)
        if (dev < 0 || dev >= count) {
            fkd_tree_destroy(t);
            return fail(FKD_INVALID_ARGUMENT, "device id out of range");
        }
    fkd_status s = make_replica(t, devs[0], level_order, false, nullptr);
    if (s == FKD_OK) s = fanout_replicas(t, std::vector<int>(devs.begin() + 1, devs.end()));
    if (s != FKD_OK) {
        fkd_tree_destroy(t);
        return s;
    }
    *out = t;
    return FKD_OK;
}

fkd_status fkd_tree_add_replicas(fkd_tree* t, const int32_t* devices, int32_t ndev) {
    if (!t) return fail(FKD_INVALID_ARGUMENT, "null tree");
    if (t->reps.empty()) return fail(FKD_NO_DEVICE, "tree has no device replica");
    if (ndev <= 0) return FKD_OK;
    if (!devices) return fail(FKD_INVALID_ARGUMENT, "null device list");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        return fail(FKD_NO_DEVICE, "no CUDA device visible (the B200 path has no CPU fallback)");
    for (int32_t i = 0; i < ndev; ++i)
        if (devices[i] < 0 || devices[i] >= count) return fail(FKD_INVALID_ARGUMENT, "device id out of range");
    const size_t had = t->reps.size();
    const fkd_status s = fanout_replicas(t, std::vector<int>(devices, devices + ndev));
    if (s != FKD_OK) {  // a failed fan-out leaves the tree as it was (no half-copied replica)
        for (size_t i = had; i < t->reps.size(); ++i) delete t->reps[i];
        t->reps.resize(had);
    }
    return s;
}

fkd_status fkd_tree_create_device(const float* d_level_order, int64_t n, int32_t dim, void* stream,
                                  fkd_tree** out) {
    if (!out) return fail(FKD_INVALID_ARGUMENT, "null output");
    *out = nullptr;
    // child slots 2c+1 / 2c+2 are int32 (traverse.hpp:228-229): fine below 2^30 nodes
    if (n < 0 || n >= (int64_t(1) << 30)) return fail(FKD_DATA_ERROR, "tree size out of range (must be < 2^30)");
    if (dim < 0 || (n > 0 && dim < 1)) return fail(FKD_DATA_ERROR, "point set: negative dimension");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        return fail(FKD_NO_DEVICE, "no CUDA device visible (the B200 path has no CPU fallback)");
    int dev = 0;
    FKD_CUDA(cudaGetDevice(&dev));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto* t = new fkd_tree();
    t->n = n;
    t->dim = dim;
    t->stride = store_stride(dim);
    if (n > 0) {
        unsigned* d_lohi = nullptr;
        unsigned long long* d_bad = nullptr;
        std::vector<unsigned> lohi(16);
        for (int d = 0; d < 8; ++d) {
            lohi[2 * d] = 0xffffffffu;
            lohi[2 * d + 1] = 0u;
        }
        unsigned long long bad = kNoBad;
        cudaError_t e = cudaMalloc(&d_lohi, 16 * sizeof(unsigned));
        if (e == cudaSuccess) e = cudaMalloc(&d_bad, sizeof(unsigned long long));
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_lohi, lohi.data(), 16 * sizeof(unsigned), cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_bad, &bad, sizeof(bad), cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) {
            tree_scan(d_level_order, n, dim, d_lohi, d_bad, st);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(lohi.data(), d_lohi, 16 * sizeof(unsigned), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        cudaFree(d_lohi);
        cudaFree(d_bad);
        if (e != cudaSuccess) {
            delete t;
            return fail(FKD_CUDA_ERROR, std::string("tree scan: ") + cudaGetErrorString(e));
        }
        if (bad != kNoBad) {
            delete t;
            return fail(FKD_DATA_ERROR, "tree nodes: non-finite coordinate in point " + std::to_string(bad));
        }
        float lo[8], hi[8];
        for (int d = 0; d < 8; ++d) {
            lo[d] = ordered_to_float(lohi[2 * d]);
            hi[d] = ordered_to_float(lohi[2 * d + 1]);
        }
        set_frame(t, lo, hi);
    }
    fkd_status s = make_replica(t, dev, d_level_order, true, st);
    if (s != FKD_OK) {
        fkd_tree_destroy(t);
        return s;
    }
    *out = t;
    return FKD_OK;
}

// bad = ~0 (no bad query), totals = 0.  Memsets, not a pageable H2D copy,
// which would synchronise the stream and serialise the host pipeline.
static cudaError_t reset_small(Workspace* w, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(w->small, 0xFF, sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(w->small + 1, 0, 7 * sizeof(unsigned long long), st);
    return e;
}

static fkd_status finish_small(Workspace* w, int64_t base, unsigned long long* bad,
                               unsigned long long tot[3]) {
    const unsigned long long b = w->h_small[0];
    if (b != kNoBad && (*bad == kNoBad || b + base < *bad)) *bad = b + base;
    tot[0] += w->h_small[1];
    tot[1] += w->h_small[2];
    tot[2] += w->h_small[3];
    return FKD_OK;
}

fkd_status fkd_build_tree_device(const float* d_points, int64_t n, int32_t dim, float* d_out,
                                 void* stream) {
    if (n < 0 || n > int64_t(0x7fffffff)) return fail(FKD_DATA_ERROR, "build: size out of range");
    if (n == 0) return FKD_OK;
    if (dim < 1) return fail(FKD_DATA_ERROR, "build: dimension must be >= 1");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // require_finite(points, "build") (tree.cpp:81), on the device
    unsigned* d_lohi = nullptr;
    unsigned long long* d_bad = nullptr;
    unsigned long long bad = kNoBad;
    FKD_CUDA(cudaMalloc(&d_lohi, 16 * sizeof(unsigned)));
    FKD_CUDA(cudaMalloc(&d_bad, sizeof(unsigned long long)));
    FKD_CUDA(cudaMemsetAsync(d_bad, 0xFF, sizeof(unsigned long long), st));
    FKD_CUDA(cudaMemsetAsync(d_lohi, 0, 16 * sizeof(unsigned), st));
    tree_scan(d_points, n, dim, d_lohi, d_bad, st);
    FKD_CUDA(cudaGetLastError());
    FKD_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
    FKD_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_lohi);
    cudaFree(d_bad);
    if (bad != kNoBad) return fail(FKD_DATA_ERROR, "build: non-finite coordinate in point " + std::to_string(bad));
    const BuildStatus bs = build_tree_device(d_points, n, dim, d_out, st);
    if (bs.err != cudaSuccess) return fail(FKD_CUDA_ERROR, std::string("build: ") + bs.what + ": " + cudaGetErrorString(bs.err));
    FKD_CUDA(cudaStreamSynchronize(st));
    return FKD_OK;
}

fkd_status fkd_tree_build(const float* points, int64_t n, int32_t dim, const int32_t* devices,
                          int32_t ndev, float* level_order_out, fkd_tree** out) {
    if (!out) return fail(FKD_INVALID_ARGUMENT, "null output");
    *out = nullptr;
    if (n < 0 || n > int64_t(0x7fffffff)) return fail(FKD_DATA_ERROR, "build: size out of range");
    if (n > 0 && (dim < 1 || !points)) return fail(FKD_DATA_ERROR, "build: bad point set");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        return fail(FKD_NO_DEVICE, "no CUDA device visible (the B200 path has no CPU fallback)");
    int dev0 = 0;
    if (devices && ndev > 0) dev0 = devices[0]; else cudaGetDevice(&dev0);
    if (dev0 < 0 || dev0 >= count) return fail(FKD_INVALID_ARGUMENT, "device id out of range");
    std::vector<float> nodes(size_t(n) * size_t(std::max(dim, 1)));
    {
        DeviceGuard g(dev0);
        float *d_pts = nullptr, *d_out = nullptr;
        const size_t bytes = size_t(n) * size_t(std::max(dim, 1)) * sizeof(float);
        if (n > 0) {
            FKD_CUDA(cudaMalloc(&d_pts, bytes));
            FKD_CUDA(cudaMalloc(&d_out, bytes));
            FKD_CUDA(cudaMemcpy(d_pts, points, bytes, cudaMemcpyHostToDevice));
        }
        fkd_status s = fkd_build_tree_device(d_pts, n, dim, d_out, nullptr);
        if (s == FKD_OK && n > 0) {
            cudaError_t e = cudaMemcpy(nodes.data(), d_out, bytes, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) s = fail(FKD_CUDA_ERROR, std::string("build readback: ") + cudaGetErrorString(e));
        }
        cudaFree(d_pts);
        cudaFree(d_out);
        if (s != FKD_OK) return s;
    }
    if (level_order_out && n > 0) std::copy(nodes.begin(), nodes.end(), level_order_out);
    return fkd_tree_create(nodes.data(), n, dim, devices, ndev, out);
}

fkd_status fkd_run_batch_device(const fkd_tree* t, const float* d_q, int64_t m, int32_t dim,
                                const fkd_batch_options* o, int32_t* d_counts, fkd_hit* d_hits,
                                fkd_query_stats* stats, fkd_query_stats* d_per_query, void* stream,
                                fkd_timings* timings) {
    fkd_device_batch b{};
    b.d_queries = d_q;
    b.m = m;
    b.dim = dim;
    if (o) b.opt = *o;
    b.d_counts = d_counts;
    b.d_hits = d_hits;
    b.stats = stats;
    b.d_per_query = d_per_query;
    b.timings = timings;
    if (!o) return fail(FKD_INVALID_ARGUMENT, "null options");
    const fkd_status s = fkd_run_batches_device(t, &b, 1, stream);
    return s;
}

}  // extern "C"

namespace fkd {
struct BatchItem {
    fkd_device_batch* b = nullptr;
    float cap2 = 0.0f;
    Workspace* w = nullptr;
    cudaStream_t st = nullptr;
    int launches = 0, walk_launches = 0;
    bool run = false;
    double cost = 0.0;
    unsigned long long* bad_src = nullptr;  // the flag of the batch whose order this one shared
};
}  // namespace fkd

extern "C" {

// Several independent batches in one submission (e.g. the fcp and the kNN
// request of a step, or two clients' batches).  Each runs exactly as
// fkd_run_batch_device would, with its own workspace, on its own stream
// forked from the caller's; the most expensive batch (by kind, k and size)
// gets the highest stream priority, so its blocks are dispatched first and
// the cheaper batches' walks fill the SMs its straggler warps, continuation
// rounds and CTA pass leave idle — the one-batch tail phases run at
// 24-82% of the SMs (profiles/r01k_knn8_kernels.jsonl).  Results, statuses
// and counters are each batch's own; the call synchronises the caller's
// stream once, after every batch.
fkd_status fkd_run_batches_device(const fkd_tree* t, fkd_device_batch* batches, int32_t n, void* stream) {
    if (n < 0 || (n > 0 && !batches)) return fail(FKD_INVALID_ARGUMENT, "bad batch list");
    if (!t) return fail(FKD_INVALID_ARGUMENT, "null tree");
    using Item = BatchItem;
    std::vector<Item> items(static_cast<size_t>(n));
    fkd_status first = FKD_OK;
    std::string first_msg;
    auto note = [&](fkd_device_batch* b, fkd_status s) {
        b->status = s;
        if (s != FKD_OK && first == FKD_OK) {
            first = s;
            first_msg = g_err;
        }
    };
    // validation in the reference's order, per batch (batch.cpp:72-80)
    for (int32_t i = 0; i < n; ++i) {
        Item& it = items[size_t(i)];
        it.b = &batches[i];
        fkd_device_batch* b = it.b;
        if (b->stats) *b->stats = fkd_query_stats{0, 0, 0};
        if (b->timings) *b->timings = fkd_timings{0.0f, 0.0f, 0.0f, 0, 0, 0};
        fkd_status s = validate(t, b->m, b->dim, &b->opt, &it.cap2);
        if (s == FKD_OK && b->m > 0 && t->reps.empty()) s = fail(FKD_NO_DEVICE, "tree has no device replica");
        if (s == FKD_OK && b->m > 0 && (reinterpret_cast<uintptr_t>(b->d_hits) & 7u) != 0)
            s = fail(FKD_INVALID_ARGUMENT, "hits buffer must be 8-byte aligned");
        note(b, s);
        it.run = s == FKD_OK && b->m > 0;
        const int k = b->opt.kind == FKD_KNN ? b->opt.k : 1;
        it.cost = double(b->m) * (k == 1 ? 1.0 : 2.0 + std::log2(double(k)));
    }
    std::vector<Item*> order;
    for (Item& it : items)
        if (it.run) order.push_back(&it);
    if (order.empty()) return first == FKD_OK ? FKD_OK : fail(first, first_msg);
    std::stable_sort(order.begin(), order.end(), [](const Item* a, const Item* b) { return a->cost > b->cost; });
    Replica& r = *t->reps[0];
    DeviceGuard g(r.device);
    cudaStream_t caller = static_cast<cudaStream_t>(stream);
    const Knobs kn = read_knobs();
    fkd_status err = FKD_OK;
    for (Item* it : order) {
        if (err == FKD_OK) err = acquire_ws(r, &it->w);
        if (err != FKD_OK) break;
        // one batch: the caller's stream; several: the costliest on the
        // workspace's high-priority stream, the others on normal ones
        it->st = order.size() == 1 ? caller : (it == order.front() ? it->w->tail : it->w->stream);
    }
    auto cuda = [&](cudaError_t e, const char* what) {
        if (e != cudaSuccess && err == FKD_OK) err = fail(FKD_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
        return e == cudaSuccess;
    };
    size_t enq = 0;
    if (err == FKD_OK && order.size() > 1) {  // fork from the caller's stream
        Workspace* w0 = order.front()->w;
        if (cuda(cudaEventRecord(w0->pe[0], caller), "fork"))
            for (Item* it : order) cuda(cudaStreamWaitEvent(it->st, w0->pe[0], 0), "fork");
    }
    // Batches over the same query array share one Morton order: the walk
    // order never changes a result (each query is independent), so sorting
    // identical queries twice is redundant work.  The first (costliest) such
    // batch sorts and checks the queries; the others wait for its order.
    auto sortable = [&](const Item* it) {
        return use_morton(t, &it->b->opt, it->b->m) && it->b->m <= kSortChunk;
    };
    std::vector<SharedOrder> shares(order.size());
    for (size_t i = 0; i < order.size(); ++i) {
        Item* it = order[i];
        if (err != FKD_OK) break;
        fkd_device_batch* b = it->b;
        Workspace* w = it->w;
        cudaStream_t st = it->st;
        const bool want_stats = b->stats != nullptr || b->d_per_query != nullptr;
        const SharedOrder* share = nullptr;
        for (size_t j = 0; j < i && sortable(it); ++j) {
            const fkd_device_batch* o2 = order[j]->b;
            if (shares[j].order && o2->d_queries == b->d_queries && o2->m == b->m && o2->dim == b->dim) {
                share = &shares[j];
                break;
            }
        }
        if (!cuda(reset_small(w, st), "reset")) break;
        if (b->timings) cuda(cudaEventRecord(w->ev[0], st), "event");
        const fkd_status e = enqueue(t, r, w, b->d_queries, b->m, &b->opt, it->cap2, b->d_counts, b->d_hits,
                                     b->d_per_query, want_stats, st, &it->launches, &it->walk_launches, kn,
                                     b->timings ? w->ev[1] : nullptr, b->timings ? w->ev[3] : nullptr, 0,
                                     nullptr, 1, share, (!share && sortable(it)) ? w->pe[2] : nullptr);
        if (e == FKD_OK && !share && sortable(it) && order.size() > 1)
            shares[i] = SharedOrder{w->ids + w->key_cap / 2, w->small, w->pe[2]};
        it->bad_src = share ? share->bad : nullptr;
        if (e != FKD_OK) {
            err = e;
            break;
        }
        if (b->timings) cuda(cudaEventRecord(w->ev[2], st), "event");
        cuda(cudaMemcpyAsync(w->h_small, w->small, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st),
             "readback");
        if (order.size() > 1 && cuda(cudaEventRecord(w->pe[1], st), "join")) cuda(cudaStreamWaitEvent(caller, w->pe[1], 0), "join");
        ++enq;
    }
    // one synchronisation for all: the non-finite check must be a status
    const cudaError_t se = cudaStreamSynchronize(caller);
    for (Item* it : order)  // (after an error, batches forked but not joined)
        if (it->w && it->st != caller) cudaStreamSynchronize(it->st);
    if (se != cudaSuccess && err == FKD_OK) err = fail(FKD_CUDA_ERROR, std::string("batch: ") + cudaGetErrorString(se));
    for (size_t i = 0; i < order.size(); ++i) {
        Item* it = order[i];
        if (!it->w) continue;
        fkd_device_batch* b = it->b;
        Workspace* w = it->w;
        if (err != FKD_OK || i >= enq) {
            note(b, err != FKD_OK ? err : FKD_CUDA_ERROR);
        } else {
            unsigned long long bad = kNoBad, tot[3] = {0, 0, 0};
            finish_small(w, 0, &bad, tot);
            if (it->bad_src)  // checked by the batch whose order it shared (same queries)
                for (Item* o2 : order)
                    if (o2->w && o2->w->small == it->bad_src) bad = std::min(bad, o2->w->h_small[0]);
            if (bad != kNoBad) {
                note(b, fail(FKD_DATA_ERROR, "queries: non-finite coordinate in point " + std::to_string(bad)));
            } else {
                if (b->stats) *b->stats = fkd_query_stats{int64_t(tot[0]), int64_t(tot[1]), int64_t(tot[2])};
                if (b->timings) {
                    cudaEventElapsedTime(&b->timings->order_ms, w->ev[0], w->ev[1]);
                    cudaEventElapsedTime(&b->timings->walk_ms, w->ev[1], w->ev[2]);
                    cudaEventElapsedTime(&b->timings->tail_ms, w->ev[3], w->ev[2]);
                    b->timings->launches = it->launches;
                    b->timings->walk_launches = it->walk_launches;
                    b->timings->overflowed = int64_t(w->h_small[5]);
                }
            }
        }
        release_ws(r, w);
    }
    if (first != FKD_OK) return fail(first, first_msg);
    return FKD_OK;
}

}  // extern "C"

// ---- host-buffer path (fkd_run_batch, fkd_run_batches) ---------------------
//
// The batch is sharded over the tree's devices in contiguous blocks (the
// reference's OpenMP loop over queries, batch.cpp:93-103, lifted to devices);
// each device's shard runs as its own pipeline, enqueued by its own host
// thread.  Per device, the shard is cut into a graduated chunk schedule —
// small first chunks (the first H2D + walk overlap nothing), shard/div middle
// chunks, small last chunks (the last D2H overlaps nothing) — and every chunk
// is one job per batch of the group (the batches of one fkd_run_batches call
// over the same query array: the chunk's queries are uploaded, checked and
// Morton-ordered once and walked by every batch).  Jobs run on `streams`
// slot streams, so the H2D engine, the SMs and the D2H engine stay busy:
//   copy-in stream : H2D chunk c                          -> ev_in[c]
//   slot stream    : wait ev_in[c]; order + walk (job j)  -> ev_walk[j]
//   copy-out stream: wait ev_walk[j]; D2H counts, hits    -> ev_out[j]
// Device staging is "full" when the shard's queries and every batch's results
// fit in a quarter of the free memory (all H2Ds are then issued up front, so
// the copy-in finishes before it shares PCIe with the copy-out); otherwise a
// chunk's queries live in its first job's slot and each job's results in its
// own slot, reused R jobs later once the previous users are done.
//
// Pageable caller buffers (std::vector / NumPy: what a reference caller
// holds) are staged through bounded rings of pinned host slots: a query
// chunk is copied into its ring slot by the host copy pool just before its
// H2D (the copy also runs require_finite, batch.cpp:79), and a drain thread
// enqueues each job's D2H into a result ring slot and copies the slot out
// to the caller once the D2H has landed, R jobs behind.  Results reach the
// caller's buffers only after every query of the batch passed the host check,
// so a rejected batch leaves pageable outputs untouched, as the reference
// throws before its BatchResult exists (batch.cpp:79 before :82-86).
// Without a pinned ring (allocation failure, FKD_PAGEABLE_STAGING=0) the
// pageable pointers go to cudaMemcpyAsync directly.
namespace fkd {
namespace {

struct GroupBatch {  // one batch of a host group (all share the query array)
    const fkd_batch_options* o = nullptr;
    float cap2 = 0.0f;
    int k = 1;
    int32_t* counts = nullptr;
    fkd_hit* hits = nullptr;
    bool want_stats = false;
    fkd_query_stats* stats = nullptr;
};

struct PipeJob {
    int64_t base, count, off;  // the chunk: global query offset, size, offset in the device's shard
    int chunk, b, ws;          // chunk index, batch index, slot (workspace) index
};

struct DevicePipe {
    int di = 0;
    Replica* rep = nullptr;
    std::vector<Workspace*> wss;
    std::vector<PipeJob> jobs;  // chunk-major, batch-minor
    int nchunks = 0;
    bool full = false;
    bool pg_q = false, pg_out = false;
    HostStage qst{}, rst{};
    int64_t max_chunk = 0, qring = 1, rring = 1;
    size_t r_slot_bytes = 0;
    std::vector<cudaEvent_t> ev_in;                    // per chunk
    std::vector<cudaEvent_t> ev_sorted, ev_walk, ev_out;  // per job
    cudaEvent_t ev_start = nullptr;                       // FKD_PIPE_TRACE
    std::vector<cudaEvent_t> ev_wstart, ev_tstart;        // FKD_PIPE_TRACE: walk / tail start per job
    // enqueue thread -> drain thread hand-off
    std::mutex mu;
    std::condition_variable cv;
    size_t enqueued = 0, d2h_enqueued = 0;
    bool enq_done = false;
};

struct PipeShared {
    std::mutex mu;
    std::condition_variable cv;
    fkd_status err = FKD_OK;
    std::string msg;
    std::atomic<bool> stop{false};
    int checks_left = 0;                   // enqueue threads still running their host checks
    unsigned long long host_bad = kNoBad;  // first non-finite query found on the host

    void error(fkd_status s, const std::string& m) {
        std::lock_guard<std::mutex> lk(mu);
        if (err == FKD_OK) {
            err = s;
            msg = m;
        }
        stop = true;
        cv.notify_all();
    }
    void bad(unsigned long long id) {
        std::lock_guard<std::mutex> lk(mu);
        host_bad = std::min(host_bad, id);
    }
    void checks_done() {
        std::lock_guard<std::mutex> lk(mu);
        --checks_left;
        cv.notify_all();
    }
    bool wait_checks() {  // true: every query passed and nothing failed
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return checks_left == 0 || err != FKD_OK; });
        return err == FKD_OK && host_bad == kNoBad;
    }
};

std::vector<int64_t> chunk_schedule(const Knobs& kn, int64_t total, int64_t full_chunk) {
    std::vector<int64_t> sizes;
    auto uniform = [&] {
        for (int64_t b = 0; b < total; b += full_chunk) sizes.push_back(std::min(full_chunk, total - b));
        return sizes;
    };
    if (kn.chunk > 0 || total <= 2 * full_chunk) return uniform();
    // head ramp full/2^h .. full/2, tail ramp full/2 .. full/2^t
    std::vector<int64_t> head, tail;
    for (int j = kn.ramp_head; j >= 1; --j) head.push_back(std::max<int64_t>(1024, full_chunk >> j));
    for (int j = 1; j <= kn.ramp_tail; ++j) tail.push_back(std::max<int64_t>(1024, full_chunk >> j));
    int64_t left = total;
    for (int64_t v : head) left -= v;
    for (int64_t v : tail) left -= v;
    if (left < 0) return uniform();  // too short for the ramps
    sizes = head;
    while (left > 0) {
        sizes.push_back(std::min(full_chunk, left));
        left -= sizes.back();
    }
    sizes.insert(sizes.end(), tail.begin(), tail.end());
    return sizes;
}

// The chunked pipeline over one query array and the batches of its group
// (validated by the caller; m > 0, 1 <= group size <= kMaxGroup).
fkd_status run_host_group(const fkd_tree* t, const float* queries, int64_t m, int32_t dim,
                          std::vector<GroupBatch>& batches, const Knobs& kn) {
    const int B = int(batches.size());
    int kmax = 1;
    double out_bytes_per_query = 0.0;
    for (const GroupBatch& g : batches) {
        kmax = std::max(kmax, g.k);
        out_bytes_per_query += 4.0 + 8.0 * g.k;
    }
    const bool check = t->n > 0;  // require_finite only with a non-empty tree (batch.cpp:75)
    // Unbounded radius: every query gets exactly min(k, n) hits (trees and
    // queries are finite, so every d2 passes d2 <= inf), so those counts are
    // written on the host instead of copied (a third of an fcp batch's D2H
    // bytes); a device pass over the walked counts raises an invariant error
    // should one ever differ.
    std::vector<int32_t> ccount(size_t(B), -1);
    for (int b = 0; b < B; ++b)
        if (kn.host_counts && t->n > 0 && std::isinf(batches[size_t(b)].cap2))
            ccount[size_t(b)] = int32_t(std::min<int64_t>(batches[size_t(b)].k, t->n));
    const int ndev = int(t->reps.size());
    const int64_t per_dev = (m + ndev - 1) / ndev;
    // middle chunk = shard / div: 8 for kNN lists (D2H-bound: C3 kNN8 pinned
    // 15.6 ms vs 16.3 at 4); 4 for one-slot results, whose call is bound by
    // the chunk walks (C3 fcp pageable 9.4 -> 7.4 ms, pinned 4.7 -> 4.6;
    // tools/e2e_ab.py, profiles/r02/r02h_e2e_ab.log)
    const int64_t div = kn.chunk_div > 0 ? kn.chunk_div : (kmax == 1 ? 4 : 8);
    const int64_t full_chunk = kn.chunk > 0 ? kn.chunk
                                            : std::min<int64_t>(int64_t(4) << 20,
                                                                std::max<int64_t>(int64_t(256) << 10,
                                                                                  (per_dev + div - 1) / div));
    bool want_pg_q = kn.pageable_staging && is_pageable(queries);
    bool want_pg_out = false;
    for (const GroupBatch& g : batches)
        want_pg_out |= kn.pageable_staging && (is_pageable(g.counts) || is_pageable(g.hits));

    std::vector<std::unique_ptr<DevicePipe>> pipes;
    PipeShared sh;
    fkd_status err = FKD_OK;
    // ---- plan: shards, chunks, jobs, slots, device staging, host rings, events
    for (int di = 0; di < ndev && err == FKD_OK; ++di) {
        const int64_t lo = std::min<int64_t>(m, di * per_dev), hi = std::min<int64_t>(m, lo + per_dev);
        if (hi <= lo) continue;
        auto P = std::make_unique<DevicePipe>();
        P->di = di;
        P->rep = t->reps[di];
        DeviceGuard g(P->rep->device);
        const std::vector<int64_t> sizes = chunk_schedule(kn, hi - lo, full_chunk);
        P->nchunks = int(sizes.size());
        const size_t njobs = sizes.size() * size_t(B);
        // at least one slot per batch: in full staging batch b keeps its
        // results in slot b's buffers
        const int nws = int(std::max<size_t>(size_t(B), std::min<size_t>(njobs, size_t(kn.streams))));
        for (int j = 0; j < nws && err == FKD_OK; ++j) {
            Workspace* w = nullptr;
            err = acquire_ws(*P->rep, &w);
            if (err == FKD_OK) P->wss.push_back(w);
        }
        if (err != FKD_OK) {
            for (Workspace* w : P->wss) release_ws(*P->rep, w);
            break;
        }
        // the workspace that already holds the largest staging serves as slot 0
        std::stable_sort(P->wss.begin(), P->wss.end(),
                         [](const Workspace* x, const Workspace* y) { return x->h_cap > y->h_cap; });
        int64_t base = lo;
        for (size_t c = 0; c < sizes.size(); ++c) {
            for (int b = 0; b < B; ++b) {
                const size_t j = P->jobs.size();
                P->jobs.push_back(PipeJob{base, sizes[c], base - lo, int(c), b, int(j % P->wss.size())});
            }
            P->max_chunk = std::max(P->max_chunk, sizes[c]);
            base += sizes[c];
        }
        const int64_t shard = hi - lo;
        Workspace* w0 = P->wss[0];
        bool fits = w0->q_cap >= shard * dim;
        for (int b = 0; b < B && fits; ++b)
            fits = P->wss[size_t(b)]->c_cap >= shard && P->wss[size_t(b)]->h_cap >= shard * batches[size_t(b)].k;
        if (!fits && kn.full_staging) {
            size_t free_b = 0, total_b = 0;
            cudaMemGetInfo(&free_b, &total_b);
            fits = double(shard) * (double(dim) * 4 + out_bytes_per_query) <= 0.25 * double(free_b);
        }
        P->full = kn.full_staging && fits;
        for (size_t wi = 0; wi < P->wss.size() && err == FKD_OK; ++wi) {
            Workspace* w = P->wss[wi];
            int64_t q_need = 0, c_need = 0, h_need = 0;
            if (P->full) {
                if (wi == 0) q_need = shard * dim;
                if (int(wi) < B) {
                    c_need = shard;
                    h_need = shard * batches[wi].k;
                }
            } else {
                for (const PipeJob& jb : P->jobs)
                    if (jb.ws == int(wi)) {
                        if (jb.b == 0) q_need = std::max(q_need, jb.count * dim);  // the chunk's query buffer
                        c_need = std::max(c_need, jb.count);
                        h_need = std::max(h_need, jb.count * batches[size_t(jb.b)].k);
                    }
            }
            cudaError_t e = grow(w->q, w->q_cap, q_need);
            if (e == cudaSuccess) e = grow(w->counts, w->c_cap, c_need);
            if (e == cudaSuccess) e = grow(w->hits, w->h_cap, h_need);
            if (e != cudaSuccess) err = fail(FKD_CUDA_ERROR, std::string("staging: ") + cudaGetErrorString(e));
        }
        // pinned host rings for pageable caller buffers (fall back to direct
        // pageable copies when pinned memory is not available)
        P->qring = std::min<int64_t>(kn.host_ring, P->nchunks);
        P->rring = std::min<int64_t>(int64_t(kn.host_ring) * B, int64_t(P->jobs.size()));
        if (err == FKD_OK && want_pg_q) {
            P->pg_q = acquire_stage(size_t(P->qring * P->max_chunk) * dim * sizeof(float), &P->qst) == cudaSuccess;
            if (!P->pg_q) cudaGetLastError();
        }
        if (err == FKD_OK && want_pg_out) {
            P->r_slot_bytes = (size_t(P->max_chunk) * (sizeof(int32_t) + size_t(kmax) * sizeof(fkd_hit)) + 255) &
                              ~size_t(255);
            P->pg_out = acquire_stage(size_t(P->rring) * P->r_slot_bytes, &P->rst) == cudaSuccess;
            if (!P->pg_out) cudaGetLastError();
        }
        P->ev_in.assign(size_t(P->nchunks), nullptr);
        for (auto* v : {&P->ev_sorted, &P->ev_walk, &P->ev_out}) v->assign(P->jobs.size(), nullptr);
        for (auto* v : {&P->ev_in, &P->ev_sorted, &P->ev_walk, &P->ev_out})
            for (auto& e : *v)
                if (err == FKD_OK && cudaEventCreateWithFlags(&e, kn.pipe_trace ? cudaEventDefault : cudaEventDisableTiming) !=
                                         cudaSuccess)
                    err = fail(FKD_CUDA_ERROR, "event create failed");
        if (kn.pipe_trace && err == FKD_OK) {
            cudaEventCreate(&P->ev_start);
            cudaEventRecord(P->ev_start, P->wss[0]->cin);
            P->ev_wstart.assign(P->jobs.size(), nullptr);
            P->ev_tstart.assign(P->jobs.size(), nullptr);
            for (auto& e : P->ev_wstart) cudaEventCreate(&e);
            for (auto& e : P->ev_tstart) cudaEventCreate(&e);
        }
        for (Workspace* w : P->wss) {
            cudaError_t e = reset_small(w, w->stream);
            if (e != cudaSuccess && err == FKD_OK) err = fail(FKD_CUDA_ERROR, std::string("reset: ") + cudaGetErrorString(e));
        }
        if (err == FKD_OK) {  // per-batch totals in slot 0's counter block
            cudaError_t e = cudaMemsetAsync(w0->small + kBatchTotals, 0, size_t(3 * B) * sizeof(unsigned long long),
                                            w0->stream);
            if (e == cudaSuccess) e = cudaMemsetAsync(w0->small + kCountFlag, 0, sizeof(unsigned long long), w0->stream);
            if (e != cudaSuccess) err = fail(FKD_CUDA_ERROR, std::string("reset: ") + cudaGetErrorString(e));
        }
        pipes.push_back(std::move(P));
    }
    // Host check of the queries (require_finite, batch.cpp:79): fused into the
    // staging copy (pageable queries, full device staging); up front when the
    // outputs are staged but the queries are not copied by the host, or the
    // device ring would make the enqueue thread wait on the drain thread.
    // With pinned outputs and pinned queries only the device checks (the key
    // pass / scan flags the batch and its walks exit): pinned outputs are then
    // unspecified on error, as documented in fkd_b200.h.
    bool any_out = false, fused_all = true;
    for (auto& P : pipes) {
        any_out |= P->pg_out;
        fused_all &= P->pg_q && P->full;
    }
    const bool fused = check && any_out && fused_all;
    if (err == FKD_OK && check && any_out && !fused) {
        const int64_t f = par_check(queries, m * dim);
        if (f >= 0) err = fail(FKD_DATA_ERROR, "queries: non-finite coordinate in point " + std::to_string(f / dim));
    }
    sh.checks_left = int(pipes.size());

    // ---- per-device enqueue (and drain) threads
    auto job_results = [&](DevicePipe& P, const PipeJob& jb, int32_t** dc, fkd_hit** dh) {
        if (P.full) {
            Workspace* rb = P.wss[size_t(jb.b)];
            *dc = rb->counts + jb.off;
            *dh = rb->hits + jb.off * batches[size_t(jb.b)].k;
        } else {
            *dc = P.wss[size_t(jb.ws)]->counts;
            *dh = P.wss[size_t(jb.ws)]->hits;
        }
    };
    auto enqueue_pipe = [&](DevicePipe& P) {
        DeviceGuard g(P.rep->device);
        Workspace* io = P.wss[0];
        std::vector<int64_t> last_job_on_ws(P.wss.size(), -1);
        // jobs that still read a slot's query buffer / Morton order
        std::vector<std::vector<size_t>> q_readers(P.wss.size()), order_readers(P.wss.size());
        auto cuda = [&](cudaError_t e, const char* what) {
            if (e != cudaSuccess) sh.error(FKD_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
            return e == cudaSuccess;
        };
        bool stop = false;
        for (int c = 0; c < P.nchunks && !stop && !sh.stop; ++c) {
            const size_t j0 = size_t(c) * size_t(B);
            const PipeJob& first = P.jobs[j0];
            Workspace* qw = P.wss[size_t(first.ws)];  // ring staging: the chunk's query buffer
            float* dq = P.full ? io->q + first.off * dim : qw->q;
            const float* src = queries + first.base * dim;
            if (P.pg_q) {
                const int64_t slot = c % P.qring;
                if (c >= P.qring && !cuda(cudaEventSynchronize(P.ev_in[size_t(c - P.qring)]), "staging")) break;
                float* stq = reinterpret_cast<float*>(P.qst.p) + slot * P.max_chunk * dim;
                const int64_t f = par_copy_check(stq, src, first.count * dim);
                if (check && f >= 0) {  // this and later chunks are not walked
                    sh.bad((unsigned long long)(first.base + f / dim));
                    break;
                }
                src = stq;
            }
            if (!P.full)  // the query buffer's previous readers are done
                for (size_t r : q_readers[size_t(first.ws)])
                    if (!cuda(cudaStreamWaitEvent(io->cin, P.ev_walk[r], 0), "wait")) stop = true;
            if (stop ||
                !cuda(cudaMemcpyAsync(dq, src, size_t(first.count) * dim * sizeof(float), cudaMemcpyHostToDevice,
                                      io->cin), "H2D") ||
                !cuda(cudaEventRecord(P.ev_in[size_t(c)], io->cin), "event"))
                break;
            q_readers[size_t(first.ws)].clear();
            SharedOrder share{};
            for (int b = 0; b < B && !stop; ++b) {
                const size_t j = j0 + size_t(b);
                const PipeJob& jb = P.jobs[j];
                const GroupBatch& gb = batches[size_t(b)];
                Workspace* w = P.wss[size_t(jb.ws)];
                const int64_t prev = last_job_on_ws[size_t(jb.ws)];
                last_job_on_ws[size_t(jb.ws)] = int64_t(j);
                int32_t* dc = nullptr;
                fkd_hit* dh = nullptr;
                job_results(P, jb, &dc, &dh);
                if (!cuda(cudaStreamWaitEvent(w->stream, P.ev_in[size_t(c)], 0), "wait")) break;
                // this slot's Morton order may still be read by another batch's walk
                for (size_t r : order_readers[size_t(jb.ws)])
                    if (!cuda(cudaStreamWaitEvent(w->stream, P.ev_walk[r], 0), "wait")) stop = true;
                order_readers[size_t(jb.ws)].clear();
                if (!P.full && prev >= 0) {  // the slot's results buffer: its previous D2H must be done
                    if (P.pg_out) {
                        std::unique_lock<std::mutex> lk(P.mu);
                        P.cv.wait(lk, [&] { return P.d2h_enqueued > size_t(prev) || sh.stop; });
                        if (sh.stop) stop = true;
                    }
                    if (!stop && !cuda(cudaStreamWaitEvent(w->stream, P.ev_out[size_t(prev)], 0), "wait")) stop = true;
                }
                if (stop) break;
                int launches = 0, wl = 0;
                const bool sharing = b > 0 && share.order != nullptr && use_morton(t, gb.o, jb.count);
                const fkd_status e =
                    enqueue(t, *P.rep, w, dq, jb.count, gb.o, gb.cap2, dc, dh, nullptr, gb.want_stats, w->stream,
                            &launches, &wl, kn, P.ev_start ? P.ev_wstart[j] : nullptr,
                            P.ev_start ? P.ev_tstart[j] : nullptr, jb.base, w->tail, c == 0 ? kn.first_budget_div : 1,
                            sharing ? &share : nullptr, (b == 0 && B > 1) ? P.ev_sorted[j] : nullptr,
                            io->small + kBatchTotals + 3 * b);
                if (e != FKD_OK) {
                    sh.error(e, g_err);
                    stop = true;
                    break;
                }
                if (ccount[size_t(b)] >= 0 && check_counts(dc, jb.count, ccount[size_t(b)], io->small + kCountFlag,
                                                           w->stream) < 0) {
                    sh.error(FKD_CUDA_ERROR, "count check launch failed");
                    stop = true;
                    break;
                }
                if (b == 0 && B > 1 && use_morton(t, gb.o, jb.count) && jb.count <= kSortChunk)
                    share = SharedOrder{w->ids + w->key_cap / 2, w->small, P.ev_sorted[j]};
                if (!cuda(cudaEventRecord(P.ev_walk[j], w->stream), "event")) {
                    stop = true;
                    break;
                }
                q_readers[size_t(first.ws)].push_back(j);
                if (sharing) order_readers[size_t(first.ws)].push_back(j);
                if (!P.pg_out) {
                    if (ccount[size_t(b)] >= 0) par_fill(gb.counts + jb.base, jb.count, ccount[size_t(b)]);
                    if (!cuda(cudaStreamWaitEvent(io->cout, P.ev_walk[j], 0), "wait") ||
                        (ccount[size_t(b)] < 0 &&
                         !cuda(cudaMemcpyAsync(gb.counts + jb.base, dc, size_t(jb.count) * sizeof(int32_t),
                                               cudaMemcpyDeviceToHost, io->cout), "D2H")) ||
                        !cuda(cudaMemcpyAsync(gb.hits + jb.base * gb.k, dh, size_t(jb.count) * gb.k * sizeof(fkd_hit),
                                              cudaMemcpyDeviceToHost, io->cout), "D2H") ||
                        !cuda(cudaEventRecord(P.ev_out[j], io->cout), "event")) {
                        stop = true;
                        break;
                    }
                } else {
                    std::lock_guard<std::mutex> lk(P.mu);
                    P.enqueued = j + 1;
                    P.cv.notify_all();
                }
            }
        }
        {
            std::lock_guard<std::mutex> lk(P.mu);
            P.enq_done = true;
            P.cv.notify_all();
        }
        sh.checks_done();
    };
    auto drain_pipe = [&](DevicePipe& P) {
        DeviceGuard g(P.rep->device);
        Workspace* io = P.wss[0];
        const size_t ring = size_t(P.rring);
        bool gate = false, ok = false;
        using clk = std::chrono::steady_clock;
        const auto t_origin = clk::now();
        auto ms_since = [&](clk::time_point t) { return std::chrono::duration<double, std::milli>(t - t_origin).count(); };
        auto copy_out = [&](size_t j) {
            const PipeJob& jb = P.jobs[j];
            const GroupBatch& gb = batches[size_t(jb.b)];
            const auto t0 = clk::now();
            if (cudaEventSynchronize(P.ev_out[j]) != cudaSuccess) {
                sh.error(FKD_CUDA_ERROR, "D2H failed");
                return;
            }
            const auto t1 = clk::now();
            if (!gate) {  // results reach the caller only once every query passed the check
                ok = fused ? sh.wait_checks() : (sh.err == FKD_OK);
                gate = true;
            }
            if (!ok || sh.stop) return;
            const char* slot = P.rst.p + (j % ring) * P.r_slot_bytes;
            if (ccount[size_t(jb.b)] >= 0)
                par_fill(gb.counts + jb.base, jb.count, ccount[size_t(jb.b)]);
            else
                par_copy(gb.counts + jb.base, slot, size_t(jb.count) * sizeof(int32_t));
            par_copy(gb.hits + jb.base * gb.k, slot + size_t(P.max_chunk) * sizeof(int32_t),
                     size_t(jb.count) * gb.k * sizeof(fkd_hit));
            if (kn.pipe_trace)  // host side of the pageable drain, ms from the drain thread's start
                std::fprintf(stderr, "dev %d job %zu copy-out wait %.3f-%.3f copy %.3f-%.3f (%.1f MB)\n", P.di, j,
                             ms_since(t0), ms_since(t1), ms_since(t1), ms_since(clk::now()),
                             double(jb.count) * (4.0 + 8.0 * gb.k) / 1e6);
        };
        size_t j = 0;
        for (;; ++j) {
            {
                std::unique_lock<std::mutex> lk(P.mu);
                P.cv.wait(lk, [&] { return P.enqueued > j || P.enq_done; });
                if (P.enqueued <= j) break;
            }
            if (j >= ring) copy_out(j - ring);
            const PipeJob& jb = P.jobs[j];
            const GroupBatch& gb = batches[size_t(jb.b)];
            int32_t* dc = nullptr;
            fkd_hit* dh = nullptr;
            job_results(P, jb, &dc, &dh);
            char* slot = P.rst.p + (j % ring) * P.r_slot_bytes;
            const bool good = cudaStreamWaitEvent(io->cout, P.ev_walk[j], 0) == cudaSuccess &&
                              (ccount[size_t(jb.b)] >= 0 ||
                               cudaMemcpyAsync(slot, dc, size_t(jb.count) * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                               io->cout) == cudaSuccess) &&
                              cudaMemcpyAsync(slot + size_t(P.max_chunk) * sizeof(int32_t), dh,
                                              size_t(jb.count) * gb.k * sizeof(fkd_hit), cudaMemcpyDeviceToHost,
                                              io->cout) == cudaSuccess &&
                              cudaEventRecord(P.ev_out[j], io->cout) == cudaSuccess;
            {
                std::lock_guard<std::mutex> lk(P.mu);
                P.d2h_enqueued = j + 1;
                P.cv.notify_all();
            }
            if (!good) {
                sh.error(FKD_CUDA_ERROR, "D2H enqueue failed");
                ++j;
                break;
            }
        }
        for (size_t jj = j > ring ? j - ring : 0; jj < j; ++jj) copy_out(jj);
    };
    if (err == FKD_OK) {
        std::vector<std::thread> threads;
        // one enqueue thread per device (the caller's thread serves the last
        // one) and a drain thread per device with staged outputs
        for (auto& P : pipes)
            if (P->pg_out) threads.emplace_back(drain_pipe, std::ref(*P));
        for (size_t i = 0; i + 1 < pipes.size(); ++i) threads.emplace_back(enqueue_pipe, std::ref(*pipes[i]));
        if (!pipes.empty()) enqueue_pipe(*pipes.back());
        for (auto& th : threads) th.join();
        if (sh.err != FKD_OK) err = fail(sh.err, sh.msg);
    }
    // ---- drain every stream, read the device flags and totals, release
    unsigned long long bad = kNoBad;
    std::vector<unsigned long long> tot(size_t(3 * B), 0ull);
    bool count_differs = false;
    for (auto& P : pipes) {
        DeviceGuard g(P->rep->device);
        // every slot stream first: the batch totals and the count flag in
        // slot 0's words are written by walks on all of them
        for (cudaStream_t cs : {P->wss[0]->cin, P->wss[0]->cout}) {
            cudaError_t e = cudaStreamSynchronize(cs);
            if (e != cudaSuccess && err == FKD_OK) err = fail(FKD_CUDA_ERROR, std::string("stream: ") + cudaGetErrorString(e));
        }
        for (Workspace* w : P->wss) {
            cudaError_t e = cudaStreamSynchronize(w->stream);
            if (e != cudaSuccess && err == FKD_OK) err = fail(FKD_CUDA_ERROR, std::string("stream: ") + cudaGetErrorString(e));
        }
        for (Workspace* w : P->wss) {
            cudaError_t e = cudaMemcpyAsync(w->h_small, w->small, kSmallWords * sizeof(unsigned long long),
                                            cudaMemcpyDeviceToHost, w->stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(w->stream);
            if (e != cudaSuccess && err == FKD_OK) err = fail(FKD_CUDA_ERROR, std::string("readback: ") + cudaGetErrorString(e));
            if (err == FKD_OK && w->h_small[0] != kNoBad) bad = std::min(bad, (unsigned long long)w->h_small[0]);
        }
        if (err == FKD_OK) {
            for (int i = 0; i < 3 * B; ++i) tot[size_t(i)] += P->wss[0]->h_small[kBatchTotals + i];
            count_differs |= P->wss[0]->h_small[kCountFlag] != 0;
        }
        if (P->ev_start && err == FKD_OK) {  // FKD_PIPE_TRACE: per-job timeline, ms from the first H2D
            for (size_t j = 0; j < P->jobs.size(); ++j) {
                float tin = 0, tws = 0, tts = 0, tw = 0, tout = 0;
                cudaEventElapsedTime(&tin, P->ev_start, P->ev_in[size_t(P->jobs[j].chunk)]);
                cudaEventElapsedTime(&tws, P->ev_start, P->ev_wstart[j]);
                cudaEventElapsedTime(&tts, P->ev_start, P->ev_tstart[j]);
                cudaEventElapsedTime(&tw, P->ev_start, P->ev_walk[j]);
                cudaEventElapsedTime(&tout, P->ev_start, P->ev_out[j]);
                std::fprintf(stderr,
                             "dev %d job %zu chunk %d batch %d n=%lld h2d_end %.3f walk_start %.3f tail_start %.3f "
                             "walk_end %.3f d2h_end %.3f\n",
                             P->di, j, P->jobs[j].chunk, P->jobs[j].b, (long long)P->jobs[j].count, tin, tws, tts, tw,
                             tout);
            }
            cudaEventDestroy(P->ev_start);
            for (auto& e : P->ev_wstart) cudaEventDestroy(e);
            for (auto& e : P->ev_tstart) cudaEventDestroy(e);
        }
        for (Workspace* w : P->wss) release_ws(*P->rep, w);
        for (auto* v : {&P->ev_in, &P->ev_sorted, &P->ev_walk, &P->ev_out})
            for (auto& e : *v)
                if (e) cudaEventDestroy(e);
        release_stage(P->qst);  // every stream that used them is drained
        release_stage(P->rst);
    }
    if (err != FKD_OK) return err;
    bad = std::min(bad, sh.host_bad);
    if (bad != kNoBad)
        return fail(FKD_DATA_ERROR, "queries: non-finite coordinate in point " + std::to_string(bad));
    if (count_differs)
        return fail(FKD_INVARIANT_ERROR, "unbounded-radius batch: a query's hit count differs from min(k, n)");
    for (int b = 0; b < B; ++b)
        if (batches[size_t(b)].stats)
            *batches[size_t(b)].stats = fkd_query_stats{int64_t(tot[size_t(3 * b)]), int64_t(tot[size_t(3 * b + 1)]),
                                                        int64_t(tot[size_t(3 * b + 2)])};
    return FKD_OK;
}

}  // namespace
}  // namespace fkd

fkd_status fkd_run_batch(const fkd_tree* t, const float* queries, int64_t m, int32_t dim,
                         const fkd_batch_options* o, int32_t* counts, fkd_hit* hits,
                         fkd_query_stats* stats) {
    float cap2 = 0.0f;
    fkd_status s = validate(t, m, dim, o, &cap2);
    if (s != FKD_OK) return s;
    if (stats) *stats = fkd_query_stats{0, 0, 0};
    if (m == 0) return FKD_OK;
    if (t->reps.empty()) return fail(FKD_NO_DEVICE, "tree has no device replica");
    std::vector<GroupBatch> group(1);
    group[0].o = o;
    group[0].cap2 = cap2;
    group[0].k = o->kind == FKD_KNN ? o->k : 1;
    group[0].counts = counts;
    group[0].hits = hits;
    group[0].want_stats = o->collect_stats != 0;
    group[0].stats = stats;
    return run_host_group(t, queries, m, dim, group, read_knobs());
}

// Several host-buffer batches in one call.  Batches over the same query
// array (same pointer, m, dim) form a group that runs as ONE pipeline: the
// queries cross PCIe, are checked and Morton-ordered once per chunk, and
// every batch of the group walks each chunk, so the copy engines stream the
// group's results back to back (C3 fcp + kNN8: one upload of 120 MB instead
// of two, and the fcp walks fill the D2H-bound kNN8 pipeline).  Groups run
// one after another.  Each batch keeps its own results, counters and status.
fkd_status fkd_run_batches(const fkd_tree* t, fkd_host_batch* batches, int32_t n) {
    if (n < 0 || (n > 0 && !batches)) return fail(FKD_INVALID_ARGUMENT, "bad batch list");
    fkd_status first = FKD_OK;
    std::string first_msg;
    auto note = [&](fkd_host_batch* b, fkd_status s) {
        b->status = s;
        if (s != FKD_OK && first == FKD_OK) {
            first = s;
            first_msg = g_err;
        }
    };
    std::vector<char> done(size_t(n), 0);
    std::vector<float> cap2(size_t(n), 0.0f);
    for (int32_t i = 0; i < n; ++i) {
        fkd_host_batch* b = &batches[i];
        b->status = FKD_OK;
        if (b->stats) *b->stats = fkd_query_stats{0, 0, 0};
        fkd_status s = validate(t, b->m, b->dim, &b->opt, &cap2[size_t(i)]);
        if (s == FKD_OK && b->m > 0 && t->reps.empty()) s = fail(FKD_NO_DEVICE, "tree has no device replica");
        if (s != FKD_OK || b->m == 0) {
            note(b, s);
            done[size_t(i)] = 1;
        }
    }
    const Knobs kn = read_knobs();
    for (int32_t i = 0; i < n; ++i) {
        if (done[size_t(i)]) continue;
        std::vector<int32_t> members;
        for (int32_t j = i; j < n && int(members.size()) < kMaxGroup; ++j)
            if (!done[size_t(j)] && batches[j].queries == batches[i].queries && batches[j].m == batches[i].m &&
                batches[j].dim == batches[i].dim)
                members.push_back(j);
        // the costliest batch first: it sorts the shared chunks and leads each chunk
        std::stable_sort(members.begin(), members.end(), [&](int32_t a, int32_t b) {
            const int ka = batches[a].opt.kind == FKD_KNN ? batches[a].opt.k : 1;
            const int kb = batches[b].opt.kind == FKD_KNN ? batches[b].opt.k : 1;
            return ka > kb;
        });
        std::vector<GroupBatch> group;
        for (int32_t j : members) {
            fkd_host_batch* b = &batches[j];
            GroupBatch g;
            g.o = &b->opt;
            g.cap2 = cap2[size_t(j)];
            g.k = b->opt.kind == FKD_KNN ? b->opt.k : 1;
            g.counts = b->counts;
            g.hits = b->hits;
            g.want_stats = b->opt.collect_stats != 0;
            g.stats = b->stats;
            group.push_back(g);
            done[size_t(j)] = 1;
        }
        const fkd_status s = run_host_group(t, batches[i].queries, batches[i].m, batches[i].dim, group, kn);
        for (int32_t j : members) note(&batches[j], s);
    }
    if (first != FKD_OK) return fail(first, first_msg);
    return FKD_OK;
}

// fkd_submit_batches / fkd_wait: fkd_run_batches on a thread of its own.  The
// pipelines of concurrent jobs take their own workspaces (streams, staging)
// from the replica pools, so nothing is shared but the device and the host
// copy pool.
struct fkd_job {
    std::thread th;
    fkd_status status = FKD_OK;
    std::string err;
};

fkd_status fkd_submit_batches(const fkd_tree* t, fkd_host_batch* batches, int32_t n, fkd_job** job) {
    if (!job) return fail(FKD_INVALID_ARGUMENT, "null job handle");
    *job = nullptr;
    if (n < 0 || (n > 0 && !batches)) return fail(FKD_INVALID_ARGUMENT, "bad batch list");
    fkd_job* j = new (std::nothrow) fkd_job;
    if (!j) return fail(FKD_CUDA_ERROR, "job allocation failed");
    int dev = 0;
    cudaGetDevice(&dev);  // the caller's current device, for the library thread
    try {
        j->th = std::thread([j, t, batches, n, dev] {
            cudaSetDevice(dev);
            j->status = fkd_run_batches(t, batches, n);
            if (j->status != FKD_OK) j->err = fkd::g_err;
        });
    } catch (const std::exception& e) {
        delete j;
        return fail(FKD_CUDA_ERROR, std::string("job thread: ") + e.what());
    }
    *job = j;
    return FKD_OK;
}

fkd_status fkd_wait(fkd_job* j) {
    if (!j) return fail(FKD_INVALID_ARGUMENT, "null job");
    j->th.join();
    const fkd_status s = j->status;
    if (s != FKD_OK) fkd::g_err = j->err;
    delete j;
    return s;
}

extern "C" {

fkd_status fkd_trace_batch(const fkd_tree* t, const float* queries, int32_t m, int32_t dim,
                           int32_t kind, int32_t k, float max_radius, int32_t* counts, fkd_hit* hits,
                           fkd_query_stats* stats, int32_t* events, int64_t cap, int64_t* lens) {
    fkd_batch_options o;
    fkd_default_options(&o);
    o.kind = kind;
    o.k = k;
    o.max_radius = max_radius;
    float cap2 = 0.0f;
    fkd_status s = validate(t, m, dim, &o, &cap2);
    if (s != FKD_OK) return s;
    if (m == 0) return FKD_OK;
    if (cap < 0) return fail(FKD_INVALID_ARGUMENT, "negative trace capacity");
    for (int64_t i = 0; t->n > 0 && i < int64_t(m) * dim; ++i)
        if (!std::isfinite(queries[i]))
            return fail(FKD_DATA_ERROR, "queries: non-finite coordinate in point " + std::to_string(i / dim));
    const int kk = kind == FKD_KNN ? k : 1;
    Replica& r = *t->reps[0];
    DeviceGuard g(r.device);
    float* dq = nullptr;
    int32_t *dc = nullptr, *dev = nullptr;
    fkd_hit* dh = nullptr;
    fkd_query_stats* ds = nullptr;
    int64_t* dl = nullptr;
    auto body = [&]() -> fkd_status {
        FKD_CUDA(cudaMalloc(&dq, size_t(m) * dim * sizeof(float)));
        FKD_CUDA(cudaMalloc(&dc, size_t(m) * sizeof(int32_t)));
        FKD_CUDA(cudaMalloc(&dh, size_t(m) * kk * sizeof(fkd_hit)));
        FKD_CUDA(cudaMalloc(&ds, size_t(m) * sizeof(fkd_query_stats)));
        FKD_CUDA(cudaMalloc(&dev, size_t(std::max<int64_t>(1, m * cap)) * sizeof(int32_t)));
        FKD_CUDA(cudaMalloc(&dl, size_t(m) * sizeof(int64_t)));
        FKD_CUDA(cudaMemcpy(dq, queries, size_t(m) * dim * sizeof(float), cudaMemcpyHostToDevice));
        launch_trace(r.nodes, int32_t(t->n), t->dim, t->stride, dq, m, cap2, kk, dc, dh, ds, dev, cap, dl,
                     nullptr);
        FKD_CUDA(cudaGetLastError());
        FKD_CUDA(cudaMemcpy(counts, dc, size_t(m) * sizeof(int32_t), cudaMemcpyDeviceToHost));
        FKD_CUDA(cudaMemcpy(hits, dh, size_t(m) * kk * sizeof(fkd_hit), cudaMemcpyDeviceToHost));
        if (stats) FKD_CUDA(cudaMemcpy(stats, ds, size_t(m) * sizeof(fkd_query_stats), cudaMemcpyDeviceToHost));
        if (events && cap > 0)
            FKD_CUDA(cudaMemcpy(events, dev, size_t(m) * cap * sizeof(int32_t), cudaMemcpyDeviceToHost));
        if (lens) FKD_CUDA(cudaMemcpy(lens, dl, size_t(m) * sizeof(int64_t), cudaMemcpyDeviceToHost));
        return FKD_OK;
    };
    s = body();
    cudaFree(dq);
    cudaFree(dc);
    cudaFree(dh);
    cudaFree(ds);
    cudaFree(dev);
    cudaFree(dl);
    return s;
}

static fkd_status single(const fkd_tree* t, const float* q, int32_t dim, int kind, int32_t k,
                         float max_radius, fkd_hit* out, int32_t* out_count, fkd_query_stats* stats) {
    // constructor order of FcpCandidates / KnnCandidates (traverse.hpp:88-89,
    // 115-117): the radius is checked before k.
    if (std::isnan(max_radius) || max_radius < 0.0f)
        return fail(FKD_DATA_ERROR, "max radius must be >= 0 or inf");
    if (kind == FKD_KNN && k < 1) return fail(FKD_INVALID_ARGUMENT, "knn: k must be >= 1");
    if (!t) return fail(FKD_INVALID_ARGUMENT, "null tree");
    if (t->n > 0) {  // validate_query (traverse.hpp:186-192)
        if (dim != t->dim)
            return fail(FKD_DATA_ERROR, "query dimension " + std::to_string(dim) +
                                            " does not match tree dimension " + std::to_string(t->dim));
        for (int d = 0; d < dim; ++d)
            if (!std::isfinite(q[d])) return fail(FKD_DATA_ERROR, "query has a non-finite coordinate");
    }
    fkd_batch_options o;
    fkd_default_options(&o);
    o.kind = kind;
    o.k = kind == FKD_KNN ? k : 1;
    o.max_radius = max_radius;
    o.collect_stats = stats != nullptr;
    o.flags = FKD_FLAG_NO_MORTON;
    const int stride = kind == FKD_KNN ? k : 1;
    std::vector<fkd_hit> hits(static_cast<size_t>(stride));
    int32_t count = 0;
    const float dummy = 0.0f;
    fkd_status s = fkd_run_batch(t, t->n > 0 ? q : &dummy, 1, t->n > 0 ? dim : 1, &o, &count,
                                 hits.data(), stats);
    if (s != FKD_OK) return s;
    std::copy(hits.begin(), hits.begin() + count, out);
    *out_count = count;
    return FKD_OK;
}

fkd_status fkd_fcp(const fkd_tree* t, const float* q, int32_t dim, float max_radius, fkd_hit* out,
                   int32_t* out_count, fkd_query_stats* stats) {
    return single(t, q, dim, FKD_FCP, 1, max_radius, out, out_count, stats);
}

fkd_status fkd_knn(const fkd_tree* t, const float* q, int32_t dim, int32_t k, float max_radius,
                   fkd_hit* out, int32_t* out_count, fkd_query_stats* stats) {
    return single(t, q, dim, FKD_KNN, k, max_radius, out, out_count, stats);
}

}  // extern "C"
