// capi.cu — the C ABI (include/fkd_b200.h): device tree store, batch
// dispatch, validation and the chunked host pipeline.
//
// Replaces flatkd::run_batch (src/batch.cpp:71-134) and
// KdTree::from_level_order (src/tree.cpp:71-78) at the drop-in boundary.
// No CPU fallback exists: every query is answered by the sm_100a kernels in
// walk.cuh; without a usable device the calls fail with FKD_NO_DEVICE.
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fkd_b200.h"
#include "build.cuh"
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

struct Tuning {
    int budget = -1;  // -1: per kind (first_budget: fcp 112, kNN <= 4 slots 256, larger lists 3072 loop trips)
    int64_t resume_min = 0;  // 0: SMs x 64 (measured: 8-D and 4-D kNN64 tails; C3's ~2k stay on the CTA pass)
    int resume_trips = 0;    // 0: fcp 4096, kNN 49152 (measured on 8-D); <0: unbounded
    // continuation rounds after the budgeted walk (walk_round_kernel), trips
    // per round.  Measured (tools/rounds_ab.sh, tools/rounds_knn_ab.sh,
    // profiles/r01e_rounds_*): fcp walk -14% (3-D C3) to -30% (4-D), kNN4
    // 4-D -18%, kNN8 walk + tail -3% (C3) / -7% (4-D) / +1% (3-D uniform);
    // for lists of >= 16 slots parking costs more than the denser warps save
    // (2-D kNN16 +2%, 4-D kNN20 +48%), so those keep one long budgeted walk.
    std::vector<int> rounds_fcp{112, 224, 448}, rounds_knn4{256, 512}, rounds_knn8{384, 768, 1536};
    // fcp batches below 2^22 queries stop after two rounds: their few parked walks
    // finish sooner in the CTA pass than in a latency-bound 448-trip round
    // (clustered 1.25M / 2.5M: -22% / -13%; 1M uniform -1%), while at 10M the third
    // round keeps the resume pass off (C3 fcp 2.49 vs 3.03 ms without it)
    // (tools/fcp_small_ab.sh, tools/fcp_rounds_c3_ab.sh, profiles/r01i_fcp_*ab.log)
    std::vector<int> rounds_fcp_small{112, 224};
    bool rounds_fcp_env = false;  // FKD_RROUNDS_FCP given: every batch size
    std::vector<int> rounds_knn_env;
    bool rounds_knn_all = false;  // FKD_RROUNDS_KNN given: every kNN bucket
};

int walk_bucket_of(int k);
// The rounds run for register lists of <= 4 slots (fcp, k <= 4) and, in
// batches of >= 2^22 queries, 8 slots (a 1M-query kNN8 batch is 4-8% slower
// with them: the round boundaries cost more than the small batch's warps lose).
inline bool rounds_on(int k, int64_t m) {
    const int kb = walk_bucket_of(k);
    return kb <= 4 || (kb == 8 && m >= (int64_t(1) << 22));
}
// first walk's loop trips before a query parks (FKD_BUDGET < 0: per kind)
inline int first_budget(int k, int64_t m) {
    if (k == 1) return 112;
    if (!rounds_on(k, m)) return 3072;
    return walk_bucket_of(k) <= 4 ? 256 : 384;
}
// resume pass trips (FKD_RESUME_TRIPS = 0): 4 x the per-kind budget without rounds
// kNN: 8-D kNN16 (C4) 12288 -> 49152 cuts the CTA pass 269 -> 61 ms and the batch 353 -> 318 ms;
// 4-D kNN16/50/64 and 5-D kNN16 finish inside 12288 (unchanged); tools/tail8d_ab2.sh
inline int resume_trips_default(int k) { return k == 1 ? 4096 : 49152; }

std::vector<int> parse_ints(const char* e) {
    std::vector<int> v;
    for (const char* p = e; *p;) {
        const int x = std::atoi(p);
        if (x > 0) v.push_back(x);
        while (*p && *p != ',') ++p;
        if (*p == ',') ++p;
    }
    return v;
}

// Launch tuning, overridable per call for experiments and tests:
// FKD_BUDGET=<first walk's loop trips before a query parks; <0 per kind, 0 off>,
// FKD_RROUNDS_FCP / FKD_RROUNDS_KNN=<t1,t2,..> (continuation rounds; "0": none),
// FKD_RESUME_MIN=<overflow count that selects the resume pass>,
// FKD_RESUME_TRIPS=<steps the resume pass adds before the CTA pass; <0 unbounded>,
Tuning tuning() {
    return [] {
        Tuning x;
        if (const char* e = std::getenv("FKD_BUDGET")) x.budget = std::atoi(e);  // <0: per kind, 0: off
        if (const char* e = std::getenv("FKD_RESUME_MIN")) x.resume_min = std::atoll(e);
        if (const char* e = std::getenv("FKD_RESUME_TRIPS")) x.resume_trips = std::atoi(e);
        if (const char* e = std::getenv("FKD_RROUNDS_FCP")) {
            x.rounds_fcp = parse_ints(e);
            x.rounds_fcp_env = true;
        }
        if (const char* e = std::getenv("FKD_RROUNDS_KNN")) {
            x.rounds_knn_env = parse_ints(e);
            x.rounds_knn_all = true;
        }
        return x;
    }();
}

// Store layout: padded vectors (1, 4, 4, 4, 8, 8, 8, 8 floats) by default;
// FKD_LAYOUT=packed keeps 2-D and 3-D nodes at 8 and 12 bytes (SURVEY §7
// step 3: chosen by measurement).
int store_stride(int dim) {
    static const bool packed = [] {
        const char* e = std::getenv("FKD_LAYOUT");
        return e && std::strcmp(e, "packed") == 0;
    }();
    switch (dim) {
        case 1: return 1;
        case 2: return packed ? 2 : 4;  // 16-byte nodes with the split plane: 2-D kNN16 -1%, fcp -3%
        case 3: return packed ? 3 : 4;
        case 4: return 4;
        case 5: case 6: case 7: case 8: return 8;
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
    unsigned long long* small = nullptr;    // [8]: bad, steps, visited, processed, work, ovf count, ovf next
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
// buffers of its own, moved by a small host copy pool (8 threads copy
// pinned <-> warm pageable memory at ~74 GB/s, above the PCIe rate), so the
// DMA engines stream exactly as with pinned caller buffers
// (tools/micro/host_copy.cpp).
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
        const int n = int(std::min(8u, std::max(1u, hw / 2))) - 1;  // + the calling thread
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

void par_copy(void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    CopyPool& pool = CopyPool::get();
    const int parts = bytes < (size_t(4) << 20) ? 1 : pool.parts();
    if (parts == 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const size_t per = ((bytes + parts - 1) / parts + 4095) & ~size_t(4095);
    pool.run(parts, [&](int i) {
        const size_t lo = std::min(bytes, size_t(i) * per), hi = std::min(bytes, lo + per);
        if (hi > lo) std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
    });
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
        std::lock_guard<std::mutex> lk(g_stage_mu);
        auto best = g_stage_pool.end();
        for (auto it = g_stage_pool.begin(); it != g_stage_pool.end(); ++it)
            if (best == g_stage_pool.end() || it->cap > best->cap) best = it;
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

void release_stage(HostStage s) {
    if (!s.p) return;
    std::lock_guard<std::mutex> lk(g_stage_mu);
    g_stage_pool.push_back(s);
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
    if (e == cudaSuccess) e = cudaMalloc(&w->small, 16 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMallocHost(&w->h_small, 16 * sizeof(unsigned long long));
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

int walk_bucket_of(int k) {
    static const int reg_max = [] {  // experiment: route larger k to the heap kernel
        const char* e = std::getenv("FKD_REG_MAXK");
        return e ? std::atoi(e) : 64;
    }();
    if (k > reg_max) return 0;
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

bool use_morton(const fkd_tree* t, const fkd_batch_options* o, int64_t m) {
    if (o->flags & FKD_FLAG_NO_MORTON) return false;
    if (!(o->flags & FKD_FLAG_MORTON)) return false;
    return t->n > 0 && m > 1 && t->dim <= 8;
}

// Enqueues one batch (device pointers) on `st`; no synchronisation.  Writes
// the first bad query id and the stat totals into w->small.
fkd_status enqueue(const fkd_tree* t, Replica& r, Workspace* w, const float* d_q, int64_t m,
                   const fkd_batch_options* o, float cap2, int32_t* d_counts, fkd_hit* d_hits,
                   fkd_query_stats* d_per_query, bool stats, cudaStream_t st, int* launches,
                   int* walk_launches, cudaEvent_t ev_mid, cudaEvent_t ev_tail = nullptr,
                   int64_t id_offset = 0, cudaStream_t tail_st = nullptr, int budget_div = 1) {
    const int k = o->kind == FKD_KNN ? o->k : 1;
    if (t->n == 0) {  // every query returns empty; queries are not read (batch.cpp:75)
        *launches += fill_empty(d_counts, d_hits, m, k, st);
        FKD_CUDA(cudaGetLastError());
        return FKD_OK;
    }
    const bool sort = use_morton(t, o, m);
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
    if (!sort || m > chunk) {
        *launches += scan_queries(d_q, m, t->dim, w->small, id_offset, st);
        FKD_CUDA(cudaGetLastError());
    }
    for (int64_t base = 0; base < m; base += chunk) {
        const int64_t cm = std::min(chunk, m - base);
        WalkArgs a{};
        a.nodes = r.nodes;
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
        a.totals = w->small + 1;
        a.per_query = d_per_query ? d_per_query + base : nullptr;
        a.bad = w->small;
        a.id_base = id_offset + base;
        const Tuning tu = tuning();
        int budget = tu.budget >= 0 ? tu.budget : first_budget(k, cm);
        if (budget_div > 1 && budget > 0) budget = std::max(64, budget / budget_div);
        a.budget = (stats || walk_bucket_of(k) == 0 || t->dim > 8) ? 0 : budget;
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
            static const std::vector<int> none;
            const std::vector<int>& rounds =
                k == 1 ? ((tu.rounds_fcp_env || cm >= (int64_t(1) << 22)) ? tu.rounds_fcp : tu.rounds_fcp_small)
                       : (tu.rounds_knn_all ? tu.rounds_knn_env
                                            : (!rounds_on(k, cm) ? none
                                                             : (walk_bucket_of(k) <= 4 ? tu.rounds_knn4 : tu.rounds_knn8)));
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

int walk_bucket(int k) { return walk_bucket_of(k); }

int launch_walk(const WalkArgs& a, int dim, int stride, bool stats, bool unordered, int phase,
                cudaStream_t st) {
    const int KB = walk_bucket_of(a.k);
    if (KB == 0 || dim > 8) return phase == 0 ? launch_walk_heap(a, dim, stats, unordered, st) : 0;
    switch (dim) {
        case 1: return launch_walk_d1(a, stride, KB, stats, unordered, phase, st);
        case 2: return launch_walk_d2(a, stride, KB, stats, unordered, phase, st);
        case 3: return launch_walk_d3(a, stride, KB, stats, unordered, phase, st);
        case 4: return launch_walk_d4(a, stride, KB, stats, unordered, phase, st);
        case 5: return launch_walk_d5(a, stride, KB, stats, unordered, phase, st);
        case 6: return launch_walk_d6(a, stride, KB, stats, unordered, phase, st);
        case 7: return launch_walk_d7(a, stride, KB, stats, unordered, phase, st);
        case 8: return launch_walk_d8(a, stride, KB, stats, unordered, phase, st);
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

void fkd_tree_destroy(fkd_tree* t) {
    if (!t) return;
    for (Replica* r : t->reps) delete r;
    delete t;
}

static fkd_status set_frame(fkd_tree* t, const float* lo, const float* hi) {
    const int dim = t->dim;
    t->frame.bits = morton_bits_per_dim(std::min(dim, 8));
    if (const char* e = std::getenv("FKD_MORTON_BITS"))  // experiment: bits per axis
        t->frame.bits = std::max(1, std::min(t->frame.bits, std::atoi(e)));
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

// The store starts node_shift() empty slots into its allocation.  With one
// slot, siblings 2c+1 / 2c+2 share an aligned pair of slots (for 16-byte
// nodes: one 32-byte sector) instead of straddling two, so the far child's
// sector usually arrived with the close child's.  Measured
// (tools/node_shift_ab.sh, profiles/r01j_node_shift_ab.log): C3 kNN8 walk
// -1.6%, fcp -1.5%, uniform kNN8 -0.8%, 4-D kNN16 -1%; FKD_NODE_SHIFT=0
// restores the unshifted store.
static int64_t node_shift() {
    static const int64_t v = [] {
        const char* e = std::getenv("FKD_NODE_SHIFT");
        return e ? int64_t(std::max(0, std::min(8, std::atoi(e)))) : int64_t(1);
    }();
    return v;
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

// Further replicas are copied device to device from the first one (over
// NVLink / NVSwitch between B200s; cudaMemcpyPeer stages through the host
// only when peer access is unavailable) — SURVEY §8(e): one upload, then a
// fan-out of the packed store.
static fkd_status peer_replica(fkd_tree* t, int dev) {
    Replica* src = t->reps.front();
    auto* r = new Replica();
    r->device = dev;
    t->reps.push_back(r);
    if (t->n == 0) return FKD_OK;
    const size_t bytes = size_t(t->n) * t->stride * sizeof(float);
    DeviceGuard g(dev);
    if (fkd_status e = alloc_store(r, t->n, t->stride); e != FKD_OK) return e;
    if (dev == src->device) {
        FKD_CUDA(cudaMemcpy(r->nodes, src->nodes, bytes, cudaMemcpyDeviceToDevice));
    } else {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, dev, src->device);
        if (can) {
            cudaError_t e = cudaDeviceEnablePeerAccess(src->device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        }
        FKD_CUDA(cudaMemcpyPeer(r->nodes, dev, src->nodes, src->device, bytes));
    }
    return FKD_OK;
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
    for (size_t i = 0; i < devs.size(); ++i) {
        const int dev = devs[i];
        if (dev < 0 || dev >= count) {
            fkd_tree_destroy(t);
            return fail(FKD_INVALID_ARGUMENT, "device id out of range");
        }
        fkd_status s = i == 0 ? make_replica(t, dev, level_order, false, nullptr) : peer_replica(t, dev);
        if (s != FKD_OK) {
            fkd_tree_destroy(t);
            return s;
        }
    }
    *out = t;
    return FKD_OK;
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
    float cap2 = 0.0f;
    fkd_status s = validate(t, m, dim, o, &cap2);
    if (s != FKD_OK) return s;
    if (stats) *stats = fkd_query_stats{0, 0, 0};
    if (timings) *timings = fkd_timings{0.0f, 0.0f, 0.0f, 0, 0, 0};
    if (m == 0) return FKD_OK;
    if (t->reps.empty()) return fail(FKD_NO_DEVICE, "tree has no device replica");
    if ((reinterpret_cast<uintptr_t>(d_hits) & 7u) != 0)
        return fail(FKD_INVALID_ARGUMENT, "hits buffer must be 8-byte aligned");
    Replica& r = *t->reps[0];
    DeviceGuard g(r.device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Workspace* w = nullptr;
    if ((s = acquire_ws(r, &w)) != FKD_OK) return s;
    const bool want_stats = stats != nullptr || d_per_query != nullptr;
    int launches = 0, walk_launches = 0;
    auto body = [&]() -> fkd_status {
        FKD_CUDA(reset_small(w, st));
        if (timings) FKD_CUDA(cudaEventRecord(w->ev[0], st));
        fkd_status e = enqueue(t, r, w, d_q, m, o, cap2, d_counts, d_hits, d_per_query, want_stats,
                               st, &launches, &walk_launches, timings ? w->ev[1] : nullptr,
                               timings ? w->ev[3] : nullptr);
        if (e != FKD_OK) return e;
        if (timings) FKD_CUDA(cudaEventRecord(w->ev[2], st));
        FKD_CUDA(cudaMemcpyAsync(w->h_small, w->small, 8 * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, st));
        FKD_CUDA(cudaStreamSynchronize(st));
        unsigned long long bad = kNoBad, tot[3] = {0, 0, 0};
        finish_small(w, 0, &bad, tot);
        if (bad != kNoBad)
            return fail(FKD_DATA_ERROR, "queries: non-finite coordinate in point " + std::to_string(bad));
        if (stats) *stats = fkd_query_stats{int64_t(tot[0]), int64_t(tot[1]), int64_t(tot[2])};
        if (timings) {
            cudaEventElapsedTime(&timings->order_ms, w->ev[0], w->ev[1]);
            cudaEventElapsedTime(&timings->walk_ms, w->ev[1], w->ev[2]);
            cudaEventElapsedTime(&timings->tail_ms, w->ev[3], w->ev[2]);
            timings->launches = launches;
            timings->walk_launches = walk_launches;
            timings->overflowed = int64_t(w->h_small[5]);
        }
        return FKD_OK;
    };
    s = body();
    release_ws(r, w);
    return s;
}

// Host-buffer path: shard over the tree's devices, and per device split the
// shard into chunks that alternate between two workspaces (two streams) so
// the H2D copy of one chunk, the walk of another and the D2H copy of a third
// overlap.  Counts and hits land directly in the caller's buffers.
fkd_status fkd_run_batch(const fkd_tree* t, const float* queries, int64_t m, int32_t dim,
                         const fkd_batch_options* o, int32_t* counts, fkd_hit* hits,
                         fkd_query_stats* stats) {
    float cap2 = 0.0f;
    fkd_status s = validate(t, m, dim, o, &cap2);
    if (s != FKD_OK) return s;
    if (stats) *stats = fkd_query_stats{0, 0, 0};
    if (m == 0) return FKD_OK;
    if (t->reps.empty()) return fail(FKD_NO_DEVICE, "tree has no device replica");
    const int k = o->kind == FKD_KNN ? o->k : 1;
    const bool want_stats = o->collect_stats != 0;
    const int ndev = int(t->reps.size());
    const int64_t per_dev = (m + ndev - 1) / ndev;
    // Chunking: a graduated schedule per device shard — small first chunks
    // (the first H2D + walk cannot overlap anything), full-size middle
    // chunks (shard/8), small last chunks (the last D2H cannot overlap
    // anything) — and four slots (workspaces) per device so the H2D engine,
    // the SMs and the D2H engine stay busy at once.  FKD_CHUNK fixes a
    // uniform size; FKD_CHUNK_DIV / FKD_STREAMS are experiment knobs.
    const char* chunk_env = std::getenv("FKD_CHUNK");
    const int64_t chunk_div = [] {
        const char* e = std::getenv("FKD_CHUNK_DIV");
        return e ? std::max(1, std::atoi(e)) : 8;
    }();
    const int n_streams = [] {  // measured (decoupled copy streams): 4 slots beat 6 by ~5% on C3 kNN8 e2e
        const char* e = std::getenv("FKD_STREAMS");
        return e ? std::max(1, std::atoi(e)) : 4;
    }();
    // ramp depths (FKD_RAMP_HEAD / FKD_RAMP_TAIL: experiment knobs)
    const int ramp_head = [] {
        const char* e = std::getenv("FKD_RAMP_HEAD");
        return e ? std::max(0, std::min(6, std::atoi(e))) : 2;
    }();
    const int ramp_tail = [] {
        const char* e = std::getenv("FKD_RAMP_TAIL");
        return e ? std::max(0, std::min(6, std::atoi(e))) : 2;
    }();
    const int64_t full_chunk = chunk_env
        ? std::max<int64_t>(1024, std::atoll(chunk_env))
        : std::min<int64_t>(int64_t(4) << 20,
                            std::max<int64_t>(int64_t(256) << 10, (per_dev + chunk_div - 1) / chunk_div));
    auto schedule = [&](int64_t total) {
        std::vector<int64_t> sizes;
        if (chunk_env || total <= 2 * full_chunk) {
            for (int64_t b = 0; b < total; b += full_chunk) sizes.push_back(std::min(full_chunk, total - b));
            return sizes;
        }
        // head ramp full/2^h .. full/2, tail ramp full/2 .. full/2^t
        std::vector<int64_t> head, tail;
        for (int j = ramp_head; j >= 1; --j) head.push_back(std::max<int64_t>(1024, full_chunk >> j));
        for (int j = 1; j <= ramp_tail; ++j) tail.push_back(std::max<int64_t>(1024, full_chunk >> j));
        int64_t left = total;
        for (int64_t v : head) left -= v;
        for (int64_t v : tail) left -= v;
        if (left < 0) {  // too short for the ramps: uniform chunks
            for (int64_t b = 0; b < total; b += full_chunk) sizes.push_back(std::min(full_chunk, total - b));
            return sizes;
        }
        sizes = head;
        while (left > 0) {
            sizes.push_back(std::min(full_chunk, left));
            left -= sizes.back();
        }
        sizes.insert(sizes.end(), tail.begin(), tail.end());
        return sizes;
    };

    struct Job {
        int rep;
        Workspace* w;
        int64_t base, count;
        int64_t off;  // offset in the device's shard (full staging)
    };
    std::vector<Job> jobs;
    std::vector<std::vector<Workspace*>> wss(ndev);
    fkd_status err = FKD_OK;
    for (int di = 0; di < ndev && err == FKD_OK; ++di) {
        const int64_t lo = std::min<int64_t>(m, di * per_dev), hi = std::min<int64_t>(m, lo + per_dev);
        if (hi <= lo) continue;
        const std::vector<int64_t> sizes = schedule(hi - lo);
        const int nws = int(std::min<size_t>(sizes.size(), size_t(n_streams)));
        for (int j = 0; j < nws && err == FKD_OK; ++j) {
            Workspace* w = nullptr;
            err = acquire_ws(*t->reps[di], &w);
            if (err == FKD_OK) wss[di].push_back(w);
        }
        // the workspace that already holds the largest staging serves as slot 0
        // (the pool hands workspaces out in no particular order)
        std::stable_sort(wss[di].begin(), wss[di].end(),
                         [](const Workspace* x, const Workspace* y) { return x->h_cap > y->h_cap; });
        int64_t b = lo;
        for (size_t c = 0; c < sizes.size() && err == FKD_OK; ++c) {
            jobs.push_back(Job{di, wss[di][c % wss[di].size()], b, sizes[c], b - lo});
            b += sizes[c];
        }
    }
    // Staging.  Full (default when it fits in a quarter of the free device
    // memory): the first slot holds the whole shard's queries and results,
    // every H2D is issued up front (so the copy-in finishes early instead of
    // sharing the PCIe link with the copy-out: each direction drops from 55 to
    // 44 GB/s when both run) and no chunk waits for a slot's buffers.  Ring
    // (fallback): every slot holds its largest chunk and chunk c reuses slot
    // c mod R's buffers after chunk c-R's walk / D2H.
    std::vector<char> full(ndev, 0);
    if (err == FKD_OK) {
        const int full_env = [] {  // experiment knob: FKD_FULL_STAGING=0 forces the ring
            const char* e = std::getenv("FKD_FULL_STAGING");
            return e ? std::atoi(e) : 1;
        }();
        for (int di = 0; di < ndev && err == FKD_OK; ++di) {
            if (wss[di].empty()) continue;
            DeviceGuard g(t->reps[di]->device);
            int64_t shard = 0;
            for (const Job& j : jobs)
                if (j.rep == di) shard += j.count;
            Workspace* w0 = wss[di][0];
            const int64_t have = std::min({w0->q_cap / std::max(1, dim), w0->c_cap, w0->h_cap / k});
            bool fits = have >= shard;
            if (!fits && full_env != 0) {
                size_t free_b = 0, total_b = 0;
                cudaMemGetInfo(&free_b, &total_b);
                fits = double(shard) * (double(dim) * 4 + 4 + 8.0 * k) <= 0.25 * double(free_b);
            }
            full[di] = full_env != 0 && fits;
            for (Workspace* w : wss[di]) {
                int64_t big = 0;
                for (const Job& j : jobs)
                    if (j.w == w) big = std::max(big, j.count);
                if (full[di]) big = w == w0 ? shard : 0;
                cudaError_t e = grow(w->q, w->q_cap, big * dim);
                if (e == cudaSuccess) e = grow(w->counts, w->c_cap, big);
                if (e == cudaSuccess) e = grow(w->hits, w->h_cap, big * k);
                if (e != cudaSuccess) err = fail(FKD_CUDA_ERROR, std::string("staging: ") + cudaGetErrorString(e));
            }
        }
    }
    // FKD_PIPE_TRACE=1: per-chunk H2D start/end, walk end, D2H end on stderr
    // (development aid; timing events on every stream)
    const bool trace = std::getenv("FKD_PIPE_TRACE") != nullptr && ndev == 1;
    // the first chunk's walk gates the first D2H: a smaller step budget ends
    // its slowest warps sooner (the overflow pass finishes those queries)
    const int first_div = [] {
        const char* e = std::getenv("FKD_FIRST_BUDGET_DIV");
        return e ? std::max(1, std::atoi(e)) : 1;
    }();
    const bool tail_prio = [] {  // experiment knob: FKD_TAIL_PRIO=0 keeps the tails on the slot stream
        const char* e = std::getenv("FKD_TAIL_PRIO");
        return !e || std::atoi(e) != 0;
    }();
    std::vector<cudaEvent_t> tev(trace ? jobs.size() * 4 : 0);
    for (auto& e : tev) cudaEventCreate(&e);
    // Pageable caller buffers go through pinned staging (see CopyPool): the
    // queries of chunk c are copied in by the host just before chunk c is
    // enqueued; results land in the staging and are copied out chunk by
    // chunk as each chunk's D2H completes.  FKD_PAGEABLE_STAGING=0 hands
    // pageable pointers to cudaMemcpyAsync directly (A/B knob).
    const bool stage_env = [] {
        const char* e = std::getenv("FKD_PAGEABLE_STAGING");
        return !e || std::atoi(e) != 0;
    }();
    const bool pg_q = stage_env && is_pageable(queries);
    const bool pg_out = stage_env && (is_pageable(counts) || is_pageable(hits));
    HostStage hst{};
    const float* src_q = queries;
    int32_t* dst_c = counts;
    fkd_hit* dst_h = hits;
    std::vector<cudaEvent_t> done(pg_out ? jobs.size() : 0, nullptr);
    if (err == FKD_OK && (pg_q || pg_out)) {
        const size_t qb = pg_q ? size_t(m) * dim * sizeof(float) : 0;
        const size_t cb = pg_out ? size_t(m) * sizeof(int32_t) : 0;
        const size_t hb = pg_out ? size_t(m) * k * sizeof(fkd_hit) : 0;
        cudaError_t e = acquire_stage(qb + cb + hb, &hst);
        if (e != cudaSuccess) err = fail(FKD_CUDA_ERROR, std::string("host staging: ") + cudaGetErrorString(e));
        if (pg_q) src_q = reinterpret_cast<const float*>(hst.p);
        if (pg_out) {
            dst_c = reinterpret_cast<int32_t*>(hst.p + qb);
            dst_h = reinterpret_cast<fkd_hit*>(hst.p + qb + cb);
        }
        for (size_t ji = 0; ji < done.size() && err == FKD_OK; ++ji) {
            DeviceGuard g(t->reps[jobs[ji].rep]->device);
            e = cudaEventCreateWithFlags(&done[ji], cudaEventDisableTiming);
            if (e != cudaSuccess) err = fail(FKD_CUDA_ERROR, std::string("event: ") + cudaGetErrorString(e));
        }
    }
    // Enqueue, per chunk c on slot s = c mod R (a slot = one workspace: its
    // staging buffers and its compute stream):
    //   copy-in stream : wait walk(c-R) [slot's q is free] ; H2D ; record in(s)
    //   slot stream    : wait in(s), wait out(c-R) [slot's results are free] ;
    //                    order + walk ; record walk(s)
    //   copy-out stream: wait walk(s) ; D2H counts + hits ; record out(s)
    // (the two bracketed waits exist only with ring staging).  One H2D and one D2H stream per device keep both copy engines streaming
    // in chunk order without queueing an H2D behind an unrelated D2H (which
    // a per-slot H2D -> walk -> D2H stream would), and the walks of
    // neighbouring chunks overlap each other's tails on the slot streams.
    // Every wait names an event recorded earlier in host order.  Bad ids
    // (offset by the chunk base) and stat totals accumulate on the device per
    // slot and are read once at the end; nothing blocks the host until the
    // final synchronisation (with pinned caller buffers).
    for (int di = 0; di < ndev && err == FKD_OK; ++di) {
        DeviceGuard g(t->reps[di]->device);
        for (Workspace* w : wss[di]) {
            cudaError_t e = reset_small(w, w->stream);
            if (e != cudaSuccess) err = fail(FKD_CUDA_ERROR, std::string("reset: ") + cudaGetErrorString(e));
        }
    }
    for (size_t ji = 0; ji < jobs.size() && err == FKD_OK; ++ji) {
        const Job& j = jobs[ji];
        Replica& r = *t->reps[j.rep];
        DeviceGuard g(r.device);
        Workspace* w = j.w;
        Workspace* io = wss[j.rep][0];
        const bool ring = !full[j.rep];
        const bool reused = ring && std::count_if(jobs.begin(), jobs.begin() + ji,
                                                  [&](const Job& x) { return x.w == w; }) > 0;
        float* dq = ring ? w->q : io->q + j.off * dim;
        int32_t* dc = ring ? w->counts : io->counts + j.off;
        fkd_hit* dh = ring ? w->hits : io->hits + j.off * k;
        int launches = 0, wl = 0;
        auto tr = [&](int which, cudaStream_t sst) {
            if (trace) cudaEventRecord(tev[ji * 4 + which], sst);
        };
        auto step = [&]() -> fkd_status {
            if (reused) FKD_CUDA(cudaStreamWaitEvent(io->cin, w->pe[1], 0));
            tr(0, io->cin);
            if (pg_q)
                par_copy(const_cast<float*>(src_q) + j.base * dim, queries + j.base * dim,
                         size_t(j.count) * dim * sizeof(float));
            FKD_CUDA(cudaMemcpyAsync(dq, src_q + j.base * dim, size_t(j.count) * dim * sizeof(float),
                                     cudaMemcpyHostToDevice, io->cin));
            FKD_CUDA(cudaEventRecord(w->pe[0], io->cin));
            tr(1, io->cin);
            FKD_CUDA(cudaStreamWaitEvent(w->stream, w->pe[0], 0));
            if (reused) FKD_CUDA(cudaStreamWaitEvent(w->stream, w->pe[2], 0));
            fkd_status e = enqueue(t, r, w, dq, j.count, o, cap2, dc, dh, nullptr,
                                   want_stats, w->stream, &launches, &wl, nullptr, nullptr, j.base,
                                   tail_prio ? w->tail : nullptr, ji == 0 ? first_div : 1);
            if (e != FKD_OK) return e;
            FKD_CUDA(cudaEventRecord(w->pe[1], w->stream));
            tr(2, w->stream);
            FKD_CUDA(cudaStreamWaitEvent(io->cout, w->pe[1], 0));
            FKD_CUDA(cudaMemcpyAsync(dst_c + j.base, dc, size_t(j.count) * sizeof(int32_t),
                                     cudaMemcpyDeviceToHost, io->cout));
            FKD_CUDA(cudaMemcpyAsync(dst_h + j.base * k, dh, size_t(j.count) * k * sizeof(fkd_hit),
                                     cudaMemcpyDeviceToHost, io->cout));
            FKD_CUDA(cudaEventRecord(w->pe[2], io->cout));
            if (pg_out) FKD_CUDA(cudaEventRecord(done[ji], io->cout));
            tr(3, io->cout);
            return FKD_OK;
        };
        err = step();
    }
    for (int di = 0; di < ndev && err == FKD_OK; ++di) {
        DeviceGuard g(t->reps[di]->device);
        for (Workspace* w : wss[di]) {
            cudaError_t e = cudaMemcpyAsync(w->h_small, w->small, 8 * sizeof(unsigned long long),
                                            cudaMemcpyDeviceToHost, w->stream);
            if (e != cudaSuccess) err = fail(FKD_CUDA_ERROR, std::string("readback: ") + cudaGetErrorString(e));
        }
    }
    // pageable results: copy each chunk out as soon as its D2H has landed
    // (overlaps the later chunks' DMA); on error, skip to the drain below
    for (size_t ji = 0; ji < done.size() && err == FKD_OK; ++ji) {
        const Job& j = jobs[ji];
        cudaError_t e = cudaEventSynchronize(done[ji]);
        if (e != cudaSuccess) {
            err = fail(FKD_CUDA_ERROR, std::string("chunk: ") + cudaGetErrorString(e));
            break;
        }
        par_copy(counts + j.base, dst_c + j.base, size_t(j.count) * sizeof(int32_t));
        par_copy(hits + j.base * k, dst_h + j.base * k, size_t(j.count) * k * sizeof(fkd_hit));
    }
    if (trace && err == FKD_OK) {
        for (auto& e : tev) cudaEventSynchronize(e);
        for (size_t ji = 0; ji < jobs.size(); ++ji) {
            float a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            cudaEventElapsedTime(&a0, tev[0], tev[ji * 4 + 0]);
            cudaEventElapsedTime(&a1, tev[0], tev[ji * 4 + 1]);
            cudaEventElapsedTime(&a2, tev[0], tev[ji * 4 + 2]);
            cudaEventElapsedTime(&a3, tev[0], tev[ji * 4 + 3]);
            std::fprintf(stderr, "chunk %zu n=%lld h2d %.3f-%.3f walk_end %.3f d2h_end %.3f\n", ji,
                         (long long)jobs[ji].count, a0, a1, a2, a3);
        }
    }
    for (auto& e : tev) cudaEventDestroy(e);
    // drain every stream even after an error, then return workspaces
    unsigned long long bad = kNoBad, tot[3] = {0, 0, 0};
    for (int di = 0; di < ndev; ++di) {
        DeviceGuard g(t->reps[di]->device);
        if (!wss[di].empty()) {
            for (cudaStream_t cs : {wss[di][0]->cin, wss[di][0]->cout}) {
                cudaError_t e = cudaStreamSynchronize(cs);
                if (e != cudaSuccess && err == FKD_OK)
                    err = fail(FKD_CUDA_ERROR, std::string("stream: ") + cudaGetErrorString(e));
            }
        }
        for (Workspace* w : wss[di]) {
            cudaError_t e = cudaStreamSynchronize(w->stream);
            if (e != cudaSuccess && err == FKD_OK)
                err = fail(FKD_CUDA_ERROR, std::string("stream: ") + cudaGetErrorString(e));
            if (err == FKD_OK) finish_small(w, 0, &bad, tot);
            release_ws(*t->reps[di], w);
        }
    }
    for (auto& e : done)
        if (e) cudaEventDestroy(e);
    release_stage(hst);  // every stream that used it is drained
    if (err != FKD_OK) return err;
    if (bad != kNoBad)
        return fail(FKD_DATA_ERROR, "queries: non-finite coordinate in point " + std::to_string(bad));
    if (stats) *stats = fkd_query_stats{int64_t(tot[0]), int64_t(tot[1]), int64_t(tot[2])};
    return FKD_OK;
}

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
