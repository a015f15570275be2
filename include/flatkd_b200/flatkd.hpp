// flatkd_b200/flatkd.hpp — the reference's C++ query API over the B200 C ABI.
//
// Header-only shim mirroring flatkd (proj/include/flatkd/{point,tree,
// traverse,batch}.hpp): same names, argument meanings, result layout and
// exception types, in namespace flatkd::b200.  A caller switches by changing
// the include and the namespace:
//
//   flatkd::BatchResult r = flatkd::run_batch(tree, queries, opts);          // CPU
//   flatkd::b200::BatchResult r = flatkd::b200::run_batch(tree, queries, opts);  // B200
//
// Every query runs in the sm_100a kernels behind include/fkd_b200.h; there
// is no host fallback.  When the reference headers are also included,
// flatkd_b200/reference_adapter.hpp accepts the reference's own KdTree /
// PointSet / BatchOptions and fills a flatkd::BatchResult directly.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <ostream>
#include <limits>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "fkd_b200.h"

namespace flatkd::b200 {

// error.hpp:9-18
class DataError : public std::runtime_error {
public:
    explicit DataError(const std::string& what) : std::runtime_error(what) {}
};

class InvariantError : public std::runtime_error {
public:
    explicit InvariantError(const std::string& what) : std::runtime_error(what) {}
};

class DeviceError : public std::runtime_error {
public:
    explicit DeviceError(const std::string& what) : std::runtime_error(what) {}
};

inline void check(fkd_status s) {
    if (s == FKD_OK) return;
    const std::string msg = fkd_last_error();
    switch (s) {
        case FKD_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case FKD_DATA_ERROR: throw DataError(msg);
        case FKD_INVARIANT_ERROR: throw InvariantError(msg);
        default: throw DeviceError(msg);
    }
}

inline constexpr float kInfRadius = std::numeric_limits<float>::infinity();

// traverse.hpp:70-83 — layout-identical to fkd_hit
struct Hit {
    std::int32_t node = -1;
    float dist2 = kInfRadius;

    float distance() const { return std::sqrt(dist2); }
    bool operator==(const Hit&) const = default;
};
static_assert(sizeof(Hit) == sizeof(fkd_hit) && alignof(Hit) == alignof(fkd_hit));

inline bool hit_order(const Hit& a, const Hit& b) {
    if (a.dist2 != b.dist2) return a.dist2 < b.dist2;
    return a.node < b.node;
}

// traverse.hpp:46-54 — layout-identical to fkd_query_stats
struct QueryStats {
    long long steps = 0;
    long long nodes_visited = 0;
    long long nodes_processed = 0;
    static constexpr int state_node_ids = 2;
};
static_assert(sizeof(QueryStats) == sizeof(fkd_query_stats));

// traverse.hpp:56-68
struct TraceEvent {
    enum class Kind : std::uint8_t { processed, bounced };
    Kind kind = Kind::processed;
    std::int32_t node = -1;
    bool operator==(const TraceEvent&) const = default;
};
using Trace = std::vector<TraceEvent>;

inline std::string trace_to_text(const Trace& trace) {  // traverse.cpp:7-16
    std::string out;
    for (const TraceEvent& e : trace) {
        out += e.kind == TraceEvent::Kind::processed ? 'P' : 'B';
        out += ' ';
        out += std::to_string(e.node);
        out += '\n';
    }
    return out;
}

enum class Engine { stack_free, recursive };  // batch.hpp:10
enum class QueryKind { fcp, knn };            // batch.hpp:11

// point.hpp:14-50 (the parts the query path uses)
class PointSet {
public:
    PointSet() = default;
    explicit PointSet(int dim) : dim_(dim) {
        if (dim < 0) throw DataError("point set: negative dimension");
    }
    PointSet(int dim, std::vector<float> data) : dim_(dim), data_(std::move(data)) {
        if (dim < 0) throw DataError("point set: negative dimension");
        if (dim == 0 && !data_.empty()) throw DataError("point set: data with zero dimension");
        if (dim > 0 && data_.size() % static_cast<std::size_t>(dim) != 0)
            throw DataError("point set: data size is not a multiple of the dimension");
    }
    int dim() const { return dim_; }
    int size() const { return dim_ == 0 ? 0 : static_cast<int>(data_.size() / static_cast<std::size_t>(dim_)); }
    bool empty() const { return data_.empty(); }
    std::span<const float> operator[](int i) const {
        return {data_.data() + static_cast<std::size_t>(i) * dim_, static_cast<std::size_t>(dim_)};
    }
    const std::vector<float>& raw() const { return data_; }
    std::vector<float>& raw() { return data_; }

private:
    int dim_ = 0;
    std::vector<float> data_;
};

// batch.hpp:16-23 (+ B200 switches)
struct BatchOptions {
    QueryKind kind = QueryKind::fcp;
    int k = 1;
    float max_radius = kInfRadius;
    Engine engine = Engine::stack_free;
    int threads = 0;  // accepted for signature parity; ignored on the GPU
    bool collect_stats = false;
    bool morton = true;      // walk in Morton order; results stay in input order
    bool unordered = false;  // left-first child order

    fkd_batch_options to_c() const {
        fkd_batch_options o;
        fkd_default_options(&o);
        o.kind = kind == QueryKind::knn ? FKD_KNN : FKD_FCP;
        o.k = k;
        o.max_radius = max_radius;
        o.engine = engine == Engine::recursive ? FKD_ENGINE_RECURSIVE : FKD_ENGINE_STACK_FREE;
        o.threads = threads;
        o.collect_stats = collect_stats ? 1 : 0;
        o.flags = (morton ? FKD_FLAG_MORTON : FKD_FLAG_NO_MORTON) | (unordered ? FKD_FLAG_UNORDERED : 0u);
        return o;
    }
};

// batch.hpp:27-41
struct BatchResult {
    int stride = 1;
    std::vector<std::int32_t> counts;
    std::vector<Hit> hits;
    QueryStats stats;

    std::span<const Hit> hits_for(int query) const {
        return {hits.data() + static_cast<std::size_t>(query) * stride,
                static_cast<std::size_t>(counts[static_cast<std::size_t>(query)])};
    }
    std::uint64_t result_hash() const {
        return fkd_result_hash(counts.data(), reinterpret_cast<const fkd_hit*>(hits.data()),
                               static_cast<int64_t>(counts.size()), stride);
    }
};

// tree.hpp:41-65: a device-resident level-order tree (round-robin split).
class KdTree {
public:
    KdTree() = default;

    static KdTree from_level_order(const PointSet& nodes, std::span<const int> devices = {}) {
        return from_level_order(nodes.raw().data(), nodes.size(), nodes.dim(), devices);
    }

    static KdTree from_level_order(const float* level_order, long long n, int dim,
                                   std::span<const int> devices = {}) {
        fkd_tree* h = nullptr;
        std::vector<int32_t> devs(devices.begin(), devices.end());
        check(fkd_tree_create(level_order, n, dim, devs.empty() ? nullptr : devs.data(),
                              static_cast<int32_t>(devs.size()), &h));
        return adopt(h);
    }

    // Takes ownership of a handle from fkd_tree_create / fkd_tree_create_device.
    static KdTree adopt(fkd_tree* h) {
        KdTree t;
        t.h_ = std::shared_ptr<fkd_tree>(h, fkd_tree_destroy);
        return t;
    }

    int size() const { return h_ ? static_cast<int>(fkd_tree_size(h_.get())) : 0; }
    int dim() const { return h_ ? fkd_tree_dim(h_.get()) : 0; }
    bool empty() const { return size() == 0; }
    const fkd_tree* handle() const { return h_.get(); }

private:
    std::shared_ptr<fkd_tree> h_;
};

// tree.cpp:80-89: host build of the unique left-balanced tree, then upload.
inline PointSet build_level_order(const PointSet& points) {
    std::vector<float> out(points.raw().size());
    check(fkd_build_tree(points.raw().data(), points.size(), points.dim(), out.data()));
    return PointSet(points.dim(), std::move(out));
}

inline KdTree build_tree(const PointSet& points, std::span<const int> devices = {}) {
    return KdTree::from_level_order(build_level_order(points), devices);
}

// batch.cpp:71-134
inline BatchResult run_batch(const KdTree& tree, const float* queries, long long m, int dim,
                             const BatchOptions& options) {
    if (options.kind == QueryKind::knn && options.k < 1)
        throw std::invalid_argument("knn: k must be >= 1");
    BatchResult res;
    res.stride = options.kind == QueryKind::knn ? options.k : 1;
    res.counts.resize(static_cast<std::size_t>(m));
    res.hits.resize(static_cast<std::size_t>(m) * res.stride);
    const fkd_batch_options o = options.to_c();
    fkd_query_stats st{0, 0, 0};
    check(fkd_run_batch(tree.handle(), queries, m, dim, &o, res.counts.data(),
                        reinterpret_cast<fkd_hit*>(res.hits.data()), &st));
    if (options.collect_stats) res.stats = QueryStats{st.steps, st.nodes_visited, st.nodes_processed};
    return res;
}

inline BatchResult run_batch(const KdTree& tree, const PointSet& queries, const BatchOptions& options) {
    return run_batch(tree, queries.raw().data(), queries.size(), queries.dim(), options);
}

// Several run_batch calls in one (fkd_run_batches): requests over the same
// query array share its upload, finiteness check and Morton order, and their
// walks overlap on the device.  Every result equals the run_batch one; the
// first failing request's error is thrown after all have run.
struct BatchRequest {
    const float* queries = nullptr;
    long long m = 0;
    int dim = 0;
    BatchOptions options;
};

inline std::vector<BatchResult> run_batches(const KdTree& tree, std::span<const BatchRequest> requests) {
    std::vector<BatchResult> res(requests.size());
    std::vector<fkd_host_batch> items(requests.size());
    std::vector<fkd_query_stats> st(requests.size(), fkd_query_stats{0, 0, 0});
    for (std::size_t i = 0; i < requests.size(); ++i) {
        const BatchRequest& r = requests[i];
        if (r.options.kind == QueryKind::knn && r.options.k < 1)
            throw std::invalid_argument("knn: k must be >= 1");
        res[i].stride = r.options.kind == QueryKind::knn ? r.options.k : 1;
        res[i].counts.resize(static_cast<std::size_t>(r.m));
        res[i].hits.resize(static_cast<std::size_t>(r.m) * res[i].stride);
        items[i] = fkd_host_batch{r.queries, r.m, r.dim, r.options.to_c(), res[i].counts.data(),
                                  reinterpret_cast<fkd_hit*>(res[i].hits.data()), &st[i], FKD_OK};
    }
    check(fkd_run_batches(tree.handle(), items.data(), static_cast<int32_t>(items.size())));
    for (std::size_t i = 0; i < requests.size(); ++i)
        if (requests[i].options.collect_stats)
            res[i].stats = QueryStats{st[i].steps, st[i].nodes_visited, st[i].nodes_processed};
    return res;
}

// run_batches without blocking (fkd_submit_batches): the job owns its result
// vectors; wait() joins it and returns them (or throws).  A serving loop
// submits batch i+1 before waiting for batch i, so the device overlaps them.
// The query arrays the requests point to must outlive wait().
class Job {
public:
    Job() = default;
    Job(const Job&) = delete;
    Job& operator=(const Job&) = delete;
    Job(Job&& o) noexcept { *this = std::move(o); }
    Job& operator=(Job&& o) noexcept {
        if (this != &o) {
            finish();
            h_ = o.h_;
            o.h_ = nullptr;
            res_ = std::move(o.res_);
            items_ = std::move(o.items_);
            st_ = std::move(o.st_);
            want_stats_ = std::move(o.want_stats_);
        }
        return *this;
    }
    ~Job() { finish(); }

    std::vector<BatchResult> wait() {
        if (!h_) throw std::invalid_argument("job already waited for");
        fkd_job* h = h_;
        h_ = nullptr;
        check(fkd_wait(h));
        for (std::size_t i = 0; i < res_.size(); ++i)
            if (want_stats_[i]) res_[i].stats = QueryStats{st_[i].steps, st_[i].nodes_visited, st_[i].nodes_processed};
        return std::move(res_);
    }

private:
    friend Job submit_batches(const KdTree& tree, std::span<const struct BatchRequest> requests);
    void finish() {
        if (h_) fkd_wait(h_);  // never leave the library thread writing freed vectors
        h_ = nullptr;
    }
    fkd_job* h_ = nullptr;
    std::vector<BatchResult> res_;
    std::vector<fkd_host_batch> items_;
    std::vector<fkd_query_stats> st_;
    std::vector<char> want_stats_;
};

inline Job submit_batches(const KdTree& tree, std::span<const BatchRequest> requests) {
    Job job;
    job.res_.resize(requests.size());
    job.items_.resize(requests.size());
    job.st_.assign(requests.size(), fkd_query_stats{0, 0, 0});
    job.want_stats_.resize(requests.size());
    for (std::size_t i = 0; i < requests.size(); ++i) {
        const BatchRequest& r = requests[i];
        if (r.options.kind == QueryKind::knn && r.options.k < 1)
            throw std::invalid_argument("knn: k must be >= 1");
        BatchResult& res = job.res_[i];
        res.stride = r.options.kind == QueryKind::knn ? r.options.k : 1;
        res.counts.resize(static_cast<std::size_t>(r.m));
        res.hits.resize(static_cast<std::size_t>(r.m) * res.stride);
        job.want_stats_[i] = r.options.collect_stats;
        job.items_[i] = fkd_host_batch{r.queries, r.m, r.dim, r.options.to_c(), res.counts.data(),
                                       reinterpret_cast<fkd_hit*>(res.hits.data()), &job.st_[i], FKD_OK};
    }
    check(fkd_submit_batches(tree.handle(), job.items_.data(), static_cast<int32_t>(job.items_.size()), &job.h_));
    return job;
}

// The same queries under several option sets (fcp + kNN of one point set).
inline std::vector<BatchResult> run_batches(const KdTree& tree, const PointSet& queries,
                                            std::span<const BatchOptions> options) {
    std::vector<BatchRequest> reqs;
    for (const BatchOptions& o : options) reqs.push_back({queries.raw().data(), queries.size(), queries.dim(), o});
    return run_batches(tree, std::span<const BatchRequest>(reqs));
}

namespace detail {

// A traced single query: the GPU walks it with the literal state machine
// (fkd_trace_batch) and returns the reference's event list.
inline std::vector<Hit> traced(const KdTree& tree, std::span<const float> query, int kind, int k,
                               float max_radius, QueryStats* stats, Trace* trace) {
    const int stride = kind == FKD_KNN ? k : 1;
    std::vector<Hit> out(static_cast<std::size_t>(stride > 0 ? stride : 1));
    int32_t count = 0;
    fkd_query_stats st{0, 0, 0};
    int64_t cap = 1 << 16, len = 0;
    std::vector<int32_t> ev;
    for (;;) {  // grow the buffer until the whole trace fits
        ev.assign(static_cast<std::size_t>(cap), 0);
        check(fkd_trace_batch(tree.handle(), query.data(), 1, static_cast<int32_t>(query.size()), kind, k,
                              max_radius, &count, reinterpret_cast<fkd_hit*>(out.data()), &st, ev.data(), cap,
                              &len));
        if (len <= cap) break;
        cap = len;
    }
    if (stats) *stats = QueryStats{st.steps, st.nodes_visited, st.nodes_processed};
    trace->clear();
    for (int64_t i = 0; i < len; ++i) {
        const int32_t e = ev[static_cast<std::size_t>(i)];
        trace->push_back(e >= 0 ? TraceEvent{TraceEvent::Kind::processed, e}
                                : TraceEvent{TraceEvent::Kind::bounced, ~e});
    }
    out.resize(static_cast<std::size_t>(count));
    return out;
}

}  // namespace detail

// traverse.cpp:25-39 over runtime-dimension spans (same argument list,
// including the optional stats and trace outputs, traverse.hpp:297-306)
inline std::optional<Hit> fcp(const KdTree& tree, std::span<const float> query,
                              float max_radius = kInfRadius, QueryStats* stats = nullptr,
                              Trace* trace = nullptr) {
    if (trace) {
        auto h = detail::traced(tree, query, FKD_FCP, 1, max_radius, stats, trace);
        return h.empty() ? std::nullopt : std::optional<Hit>(h[0]);
    }
    Hit h;
    int32_t count = 0;
    fkd_query_stats st{0, 0, 0};
    check(fkd_fcp(tree.handle(), query.data(), static_cast<int32_t>(query.size()), max_radius,
                  reinterpret_cast<fkd_hit*>(&h), &count, stats ? &st : nullptr));
    if (stats) *stats = QueryStats{st.steps, st.nodes_visited, st.nodes_processed};
    return count ? std::optional<Hit>(h) : std::nullopt;
}

inline std::vector<Hit> knn(const KdTree& tree, std::span<const float> query, int k,
                            float max_radius = kInfRadius, QueryStats* stats = nullptr,
                            Trace* trace = nullptr) {
    if (trace && k >= 1) return detail::traced(tree, query, FKD_KNN, k, max_radius, stats, trace);
    std::vector<Hit> out(static_cast<std::size_t>(k > 0 ? k : 1));
    int32_t count = 0;
    fkd_query_stats st{0, 0, 0};
    check(fkd_knn(tree.handle(), query.data(), static_cast<int32_t>(query.size()), k, max_radius,
                  reinterpret_cast<fkd_hit*>(out.data()), &count, stats ? &st : nullptr));
    if (stats) *stats = QueryStats{st.steps, st.nodes_visited, st.nodes_processed};
    out.resize(static_cast<std::size_t>(count));
    return out;
}

// batch.cpp:136-158 (io::format_float is "%.9g", io.cpp:163-167)
inline void write_query_results(std::ostream& out, const BatchResult& result) {
    auto fmt = [](float v) {
        char buf[48];
        std::snprintf(buf, sizeof(buf), "%.9g", static_cast<double>(v));
        return std::string(buf);
    };
    std::string line;
    for (std::size_t q = 0; q < result.counts.size(); ++q) {
        line.clear();
        const auto hits = result.hits_for(static_cast<int>(q));
        if (result.stride == 1) {
            line = hits.empty() ? std::string("-1,inf") : std::to_string(hits[0].node) + ',' + fmt(hits[0].distance());
        } else {
            line = std::to_string(hits.size());
            for (const Hit& h : hits) {
                line += ',';
                line += std::to_string(h.node);
                line += ',';
                line += fmt(h.distance());
            }
        }
        line += '\n';
        out << line;
    }
}

// ---- templated float point types (north_star: "fcp and kNN entry points
// over templated float point types").  Any PointT whose coordinates are D
// contiguous floats (float2/float3/float4, std::array<float, D>, a POD
// struct of D floats) dispatches straight to the D-specialised kernels.
template <class PointT>
constexpr int point_dim_v = static_cast<int>(sizeof(PointT) / sizeof(float));

template <class PointT>
inline std::optional<Hit> fcp(const KdTree& tree, const PointT& q, float max_radius = kInfRadius) {
    static_assert(sizeof(PointT) % sizeof(float) == 0, "PointT must be a packed float vector");
    return fcp(tree, std::span<const float>(reinterpret_cast<const float*>(&q), point_dim_v<PointT>),
               max_radius);
}

template <class PointT>
inline std::vector<Hit> knn(const KdTree& tree, const PointT& q, int k, float max_radius = kInfRadius) {
    static_assert(sizeof(PointT) % sizeof(float) == 0, "PointT must be a packed float vector");
    return knn(tree, std::span<const float>(reinterpret_cast<const float*>(&q), point_dim_v<PointT>), k,
               max_radius);
}

// Batches of typed points: contiguous PointT[m].
template <class PointT>
inline BatchResult run_batch(const KdTree& tree, std::span<const PointT> queries, const BatchOptions& options) {
    static_assert(sizeof(PointT) % sizeof(float) == 0, "PointT must be a packed float vector");
    return run_batch(tree, reinterpret_cast<const float*>(queries.data()),
                     static_cast<long long>(queries.size()), point_dim_v<PointT>, options);
}

template <class PointT>
inline KdTree tree_from_level_order(std::span<const PointT> nodes, std::span<const int> devices = {}) {
    return KdTree::from_level_order(reinterpret_cast<const float*>(nodes.data()),
                                    static_cast<long long>(nodes.size()), point_dim_v<PointT>, devices);
}

}  // namespace flatkd::b200
