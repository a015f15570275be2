// flatkd_b200/reference_adapter.hpp — accept the reference's own types.
//
// For code that already holds flatkd::KdTree / flatkd::PointSet /
// flatkd::BatchOptions (the reference headers, proj/include/flatkd/*.hpp,
// must be included first): upload the tree once with to_device(), then call
// flatkd::b200::run_batch(device_tree, queries, options) — it returns the
// reference's flatkd::BatchResult, filled in place (flatkd::Hit and fkd_hit
// share one layout), and throws the reference's exception types.
#pragma once

#include "flatkd/batch.hpp"
#include "flatkd_b200/flatkd.hpp"

namespace flatkd::b200 {

static_assert(sizeof(flatkd::Hit) == sizeof(fkd_hit) && alignof(flatkd::Hit) == alignof(fkd_hit));
static_assert(sizeof(flatkd::QueryStats) == sizeof(fkd_query_stats));

inline void check_ref(fkd_status s) {
    if (s == FKD_OK) return;
    const std::string msg = fkd_last_error();
    switch (s) {
        case FKD_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case FKD_DATA_ERROR: throw flatkd::DataError(msg);
        case FKD_INVARIANT_ERROR: throw flatkd::InvariantError(msg);
        default: throw DeviceError(msg);
    }
}

// KdTree::from_level_order (tree.cpp:71-78) onto the GPU.  Only the
// round-robin split policy exists on the device (tree.hpp:27-29).
inline KdTree to_device(const flatkd::KdTree& tree, std::span<const int> devices = {}) {
    if (!tree.split_policy().round_robin())
        throw flatkd::DataError("B200 path: only the round-robin split policy is supported");
    fkd_tree* h = nullptr;
    std::vector<int32_t> devs(devices.begin(), devices.end());
    check_ref(fkd_tree_create(tree.nodes().raw().data(), tree.size(), tree.dim(),
                              devs.empty() ? nullptr : devs.data(), static_cast<int32_t>(devs.size()), &h));
    return KdTree::adopt(h);
}

inline fkd_batch_options to_c(const flatkd::BatchOptions& options, bool morton = true) {
    fkd_batch_options o;
    fkd_default_options(&o);
    o.kind = options.kind == flatkd::QueryKind::knn ? FKD_KNN : FKD_FCP;
    o.k = options.k;
    o.max_radius = options.max_radius;
    o.engine = options.engine == flatkd::Engine::recursive ? FKD_ENGINE_RECURSIVE : FKD_ENGINE_STACK_FREE;
    o.threads = options.threads;
    o.collect_stats = options.collect_stats ? 1 : 0;
    o.flags = morton ? FKD_FLAG_MORTON : FKD_FLAG_NO_MORTON;
    return o;
}

// flatkd::run_batch (batch.cpp:71-134) with the reference's types.
inline flatkd::BatchResult run_batch(const KdTree& tree, const flatkd::PointSet& queries,
                                     const flatkd::BatchOptions& options) {
    if (options.kind == flatkd::QueryKind::knn && options.k < 1)
        throw std::invalid_argument("knn: k must be >= 1");
    flatkd::BatchResult res;
    res.stride = options.kind == flatkd::QueryKind::knn ? options.k : 1;
    const int m = queries.size();
    res.counts.assign(static_cast<std::size_t>(m), 0);
    res.hits.assign(static_cast<std::size_t>(m) * res.stride, flatkd::Hit{});
    const fkd_batch_options o = to_c(options);
    fkd_query_stats st{0, 0, 0};
    check_ref(fkd_run_batch(tree.handle(), queries.raw().data(), m, queries.dim(), &o, res.counts.data(),
                            reinterpret_cast<fkd_hit*>(res.hits.data()), &st));
    if (options.collect_stats) {
        res.stats.steps = st.steps;
        res.stats.nodes_visited = st.nodes_visited;
        res.stats.nodes_processed = st.nodes_processed;
    }
    return res;
}

// Several flatkd::run_batch calls over one query set in one submission
// (fkd_run_batches: one upload / finiteness check / Morton order, overlapped
// walks); each result is the one flatkd::run_batch returns.
inline std::vector<flatkd::BatchResult> run_batches(const KdTree& tree, const flatkd::PointSet& queries,
                                                    std::span<const flatkd::BatchOptions> options) {
    std::vector<flatkd::BatchResult> res(options.size());
    std::vector<fkd_host_batch> items(options.size());
    std::vector<fkd_query_stats> st(options.size(), fkd_query_stats{0, 0, 0});
    const int m = queries.size();
    for (std::size_t i = 0; i < options.size(); ++i) {
        const flatkd::BatchOptions& o = options[i];
        if (o.kind == flatkd::QueryKind::knn && o.k < 1) throw std::invalid_argument("knn: k must be >= 1");
        res[i].stride = o.kind == flatkd::QueryKind::knn ? o.k : 1;
        res[i].counts.assign(static_cast<std::size_t>(m), 0);
        res[i].hits.assign(static_cast<std::size_t>(m) * res[i].stride, flatkd::Hit{});
        items[i] = fkd_host_batch{queries.raw().data(), m, queries.dim(), to_c(o), res[i].counts.data(),
                                  reinterpret_cast<fkd_hit*>(res[i].hits.data()), &st[i], FKD_OK};
    }
    check_ref(fkd_run_batches(tree.handle(), items.data(), static_cast<int32_t>(items.size())));
    for (std::size_t i = 0; i < options.size(); ++i)
        if (options[i].collect_stats) {
            res[i].stats.steps = st[i].steps;
            res[i].stats.nodes_visited = st[i].nodes_visited;
            res[i].stats.nodes_processed = st[i].nodes_processed;
        }
    return res;
}

}  // namespace flatkd::b200
