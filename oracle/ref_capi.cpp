// ref_capi.cpp — a C face for the UNMODIFIED reference library, so that
// tests/ and bench.py (reference arm / cpu_baseline leg) can drive it.
//
// TEST INFRASTRUCTURE ONLY.  Compiled together with the reference sources
// straight from /root/reference/proj (see oracle/Makefile) into
// oracle/_ref/libflatkd_ref.so; nothing in the product links this.
// Every entry point forwards to the reference's own public API:
//   flatkd::build_tree              src/tree.cpp:80-89
//   flatkd::run_batch               src/batch.cpp:71-134
//   BatchResult::result_hash        src/batch.cpp:30-48
//   flatkd::fcp / flatkd::knn       src/traverse.cpp:25-39
//   flatkd::random_points           include/flatkd/rng.hpp:46-53
//   testing::random_point_set/query src/testing/instancegen.cpp:12-48
//   testing::run_*_suite            src/testing/selfcheck.cpp:94-266
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "flatkd/batch.hpp"
#include "flatkd/bench.hpp"
#include "flatkd/error.hpp"
#include "flatkd/io.hpp"
#include "flatkd/rng.hpp"
#include "flatkd/testing/instancegen.hpp"
#include "flatkd/testing/oracle.hpp"
#include "flatkd/testing/selfcheck.hpp"
#include "flatkd/traverse.hpp"
#include "flatkd/tree.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const flatkd::DataError& e) {
        g_err = e.what();
        return 2;
    } catch (const flatkd::InvariantError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

flatkd::PointSet make_points(const float* data, long long n, int dim) {
    return flatkd::PointSet(dim, std::vector<float>(data, data + n * dim));
}

struct RefHit {
    int32_t node;
    float dist2;
};
static_assert(sizeof(RefHit) == sizeof(flatkd::Hit));

}  // namespace

extern "C" {

const char* fkr_last_error() { return g_err.c_str(); }

int fkr_layout(int* out) {
    out[0] = (int)sizeof(flatkd::Hit);
    out[1] = (int)offsetof(flatkd::Hit, node);
    out[2] = (int)offsetof(flatkd::Hit, dist2);
    out[3] = (int)sizeof(flatkd::QueryStats);
    out[4] = (int)sizeof(flatkd::TraversalState);
    return 0;
}

int fkr_hardware_threads() { return flatkd::hardware_threads(); }

int fkr_random_points(uint64_t seed, long long count, int dim, float* out) {
    return guarded([&] {
        auto p = flatkd::random_points(seed, count, dim);
        std::memcpy(out, p.raw().data(), p.raw().size() * sizeof(float));
    });
}

// The clustered C3 workload (no reference counterpart): the
// same generator as the product's fkd_clustered_points, written here on the
// reference's own RNG primitives (flatkd::random_points for the centres,
// UniformFloatSource::next_u64 for blobs and Box-Muller draws, rng.hpp:33-53)
// so the reference arm of bench.py needs nothing from the product library.
int fkr_clustered_points(uint64_t master, uint64_t stream, long long count, int dim, int blobs,
                         float sigma, float* out) {
    return guarded([&] {
        if (count < 0 || dim < 1 || blobs < 1) throw flatkd::DataError("clustered points: bad shape");
        const flatkd::PointSet centres =
            flatkd::random_points(flatkd::derive_stream_seed(master, 3), blobs, dim);
        flatkd::UniformFloatSource src(flatkd::derive_stream_seed(master, stream));
        const double two_pi = 6.283185307179586476925286766559;
        for (long long i = 0; i < count; ++i) {
            const std::uint64_t b = src.next_u64() % std::uint64_t(blobs);
            for (int d = 0; d < dim; ++d) {
                const double u1 = double(src.next_u64() >> 11) * 0x1p-53;
                const double u2 = double(src.next_u64() >> 11) * 0x1p-53;
                const double z = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(two_pi * u2);
                out[i * dim + d] = centres.raw()[std::size_t(b) * dim + d] + static_cast<float>(z) * sigma;
            }
        }
    });
}

// flatkd::run_bench_matrix (bench.cpp:64-90) + write_bench_csv (bench.cpp:119-133):
// the reference's own Table-1 rows, CSV text into `out` (returns its length).
long long fkr_bench_matrix_csv(long long n_queries, int k_dim, int kind, int reps, int threads,
                               const long long* n_list, int n_count, const int* k_list, int k_count,
                               const float* r_list, int r_count, char* out, long long cap) {
    long long len = -1;
    guarded([&] {
        flatkd::BenchConfig base;
        base.n_queries = n_queries;
        base.k_dim = k_dim;
        base.kind = kind == 1 ? flatkd::QueryKind::knn : flatkd::QueryKind::fcp;
        base.reps = reps;
        base.threads = threads;
        auto rows = flatkd::run_bench_matrix(base, std::span<const long long>(n_list, n_count),
                                             std::span<const int>(k_list, k_count),
                                             std::span<const float>(r_list, r_count));
        std::ostringstream os;
        flatkd::write_bench_csv(os, rows);
        const std::string s = os.str();
        len = (long long)s.size();
        if (out && cap > 0) {
            const long long n = len < cap - 1 ? len : cap - 1;
            std::memcpy(out, s.data(), std::size_t(n));
            out[n] = 0;
        }
    });
    return len;
}

uint64_t fkr_derive_stream_seed(uint64_t master, uint64_t stream) {
    return flatkd::derive_stream_seed(master, stream);
}

int fkr_build_tree(const float* points, long long n, int dim, float* out) {
    return guarded([&] {
        auto t = flatkd::build_tree(make_points(points, n, dim));
        std::memcpy(out, t.nodes().raw().data(), t.nodes().raw().size() * sizeof(float));
    });
}

int fkr_verify_tree(const float* nodes, long long n, int dim) {
    int bad = 0;
    int rc = guarded([&] {
        auto t = flatkd::KdTree::from_level_order(make_points(nodes, n, dim));
        bad = flatkd::verify_tree(t).has_value() ? 1 : 0;
    });
    return rc ? -rc : bad;
}

int fkr_left_subtree_size(int n) { return flatkd::left_subtree_size(n); }

// run_batch on a level-order tree; kind 0 fcp / 1 knn; engine 0 stack_free / 1 recursive.
int fkr_run_batch(const float* nodes, long long n, int tree_dim, const float* queries, long long m,
                  int query_dim, int kind, int k, float max_radius, int engine, int threads,
                  int collect_stats, int32_t* counts, void* hits, int64_t* stats3,
                  double* seconds) {
    return guarded([&] {
        auto tree = flatkd::KdTree::from_level_order(make_points(nodes, n, tree_dim));
        auto qs = make_points(queries, m, query_dim);
        flatkd::BatchOptions o;
        o.kind = kind == 1 ? flatkd::QueryKind::knn : flatkd::QueryKind::fcp;
        o.k = k;
        o.max_radius = max_radius;
        o.engine = engine == 1 ? flatkd::Engine::recursive : flatkd::Engine::stack_free;
        o.threads = threads;
        o.collect_stats = collect_stats != 0;
        // time only run_batch, as src/bench.cpp:36-39 does
        const auto t0 = std::chrono::steady_clock::now();
        flatkd::BatchResult r = flatkd::run_batch(tree, qs, o);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        std::memcpy(counts, r.counts.data(), r.counts.size() * sizeof(int32_t));
        std::memcpy(hits, r.hits.data(), r.hits.size() * sizeof(flatkd::Hit));
        if (stats3) {
            stats3[0] = r.stats.steps;
            stats3[1] = r.stats.nodes_visited;
            stats3[2] = r.stats.nodes_processed;
        }
    });
}

uint64_t fkr_result_hash(const int32_t* counts, const void* hits, long long m, int stride) {
    flatkd::BatchResult r;
    r.stride = stride;
    r.counts.assign(counts, counts + m);
    const auto* h = static_cast<const flatkd::Hit*>(hits);
    r.hits.assign(h, h + m * stride);
    return r.result_hash();
}

std::size_t fkr_write_results(const int32_t* counts, const void* hits, long long m, int stride,
                              char* out, std::size_t cap) {
    flatkd::BatchResult r;
    r.stride = stride;
    r.counts.assign(counts, counts + m);
    const auto* h = static_cast<const flatkd::Hit*>(hits);
    r.hits.assign(h, h + m * stride);
    std::ostringstream os;
    flatkd::write_query_results(os, r);
    const std::string s = os.str();
    if (out && cap) {
        const std::size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
        std::memcpy(out, s.data(), n);
        out[n] = 0;
    }
    return s.size();
}

// Single query through flatkd::fcp / flatkd::knn, with stats and trace
// (trace events: node for processed, ~node for bounced).
int fkr_query(const float* nodes, long long n, int dim, const float* q, int kind, int k,
              float max_radius, void* out_hits, int* out_count, int64_t* stats3, int32_t* trace,
              long long trace_cap, long long* trace_len) {
    return guarded([&] {
        auto tree = flatkd::KdTree::from_level_order(make_points(nodes, n, dim));
        std::span<const float> qs(q, static_cast<std::size_t>(dim));
        flatkd::QueryStats st;
        flatkd::Trace tr;
        std::vector<flatkd::Hit> hits;
        if (kind == 1) {
            hits = flatkd::knn(tree, qs, k, max_radius, &st, &tr);
        } else {
            auto b = flatkd::fcp(tree, qs, max_radius, &st, &tr);
            if (b) hits.push_back(*b);
        }
        *out_count = (int)hits.size();
        std::memcpy(out_hits, hits.data(), hits.size() * sizeof(flatkd::Hit));
        if (stats3) {
            stats3[0] = st.steps;
            stats3[1] = st.nodes_visited;
            stats3[2] = st.nodes_processed;
        }
        if (trace_len) *trace_len = (long long)tr.size();
        for (std::size_t i = 0; i < tr.size() && (long long)i < trace_cap; ++i)
            trace[i] = tr[i].kind == flatkd::TraceEvent::Kind::processed ? tr[i].node : ~tr[i].node;
    });
}

// testing::BruteForceIndex over a flat point list.
int fkr_brute(const float* points, long long n, int dim, const float* q, int kind, int k,
              float max_radius, void* out_hits, int* out_count) {
    return guarded([&] {
        flatkd::testing::BruteForceIndex idx(make_points(points, n, dim));
        std::span<const float> qs(q, static_cast<std::size_t>(dim));
        std::vector<flatkd::Hit> hits;
        if (kind == 1) {
            hits = idx.knn(qs, k, max_radius);
        } else {
            auto b = idx.fcp(qs, max_radius);
            if (b) hits.push_back(*b);
        }
        *out_count = (int)hits.size();
        std::memcpy(out_hits, hits.data(), hits.size() * sizeof(flatkd::Hit));
    });
}

// instancegen driven by a caller-owned InstanceRng.
void* fkr_instance_rng_new(uint64_t seed) { return new flatkd::testing::InstanceRng(seed); }
void fkr_instance_rng_free(void* r) { delete static_cast<flatkd::testing::InstanceRng*>(r); }
uint64_t fkr_instance_rng_u64(void* r) {
    return static_cast<flatkd::testing::InstanceRng*>(r)->next_u64();
}

int fkr_random_point_set(void* r, int n, int dim, int grid, double dup, float* out) {
    return guarded([&] {
        flatkd::testing::PointGenOptions o;
        o.grid = grid;
        o.dup_fraction = dup;
        auto p = flatkd::testing::random_point_set(*static_cast<flatkd::testing::InstanceRng*>(r), n,
                                                   dim, o);
        std::memcpy(out, p.raw().data(), p.raw().size() * sizeof(float));
    });
}

int fkr_random_query(void* r, int dim, const float* points, int n, float* out) {
    return guarded([&] {
        auto pts = make_points(points, n, dim);
        auto q = flatkd::testing::random_query(*static_cast<flatkd::testing::InstanceRng*>(r), dim, pts);
        std::memcpy(out, q.data(), q.size() * sizeof(float));
    });
}

// io::write_points / write_tree (binary) and io::read_points / read_tree.
int fkr_write_file(const char* path, int tree, const float* data, long long n, int dim) {
    return guarded([&] {
        auto pts = make_points(data, n, dim);
        if (tree)
            flatkd::io::write_tree(path, flatkd::KdTree::from_level_order(pts), flatkd::io::Format::binary);
        else
            flatkd::io::write_points(path, pts, flatkd::io::Format::binary);
    });
}

int fkr_read_file(const char* path, int tree, float* out, long long cap_floats, long long* n, int* dim) {
    return guarded([&] {
        flatkd::PointSet p = tree ? flatkd::io::read_tree(path).nodes() : flatkd::io::read_points(path);
        *n = p.size();
        *dim = p.dim();
        if ((long long)p.raw().size() <= cap_floats) std::memcpy(out, p.raw().data(), p.raw().size() * 4);
    });
}

// The reference property suites; returns failures, fills checks/instances.
long long fkr_trace_suite(uint64_t seed, int instances, int max_n, int qpt, long long* out_instances) {
    flatkd::testing::SuiteConfig c{seed, instances, max_n, qpt};
    auto r = flatkd::testing::run_trace_equivalence_suite(c);
    if (out_instances) *out_instances = r.instances;
    g_err = r.first_failure;
    return r.failures();
}

long long fkr_oracle_suite(uint64_t seed, int instances, int max_n, int qpt, long long* out_checks) {
    flatkd::testing::SuiteConfig c{seed, instances, max_n, qpt};
    auto r = flatkd::testing::run_oracle_equivalence_suite(c);
    if (out_checks) *out_checks = r.checks;
    g_err = r.first_failure;
    return r.failures();
}

long long fkr_structure_suite(int max_shape_n, int sweep_n, long long* out_checks) {
    auto r = flatkd::testing::run_structure_suite(max_shape_n, sweep_n);
    if (out_checks) *out_checks = r.checks;
    g_err = r.first_failure;
    return r.failures;
}

}  // extern "C"
