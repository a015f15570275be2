// shim_parity.cpp — the C++ drop-in, exercised the way a reference user would:
// the same inputs through flatkd::run_batch (the unmodified reference, CPU)
// and flatkd::b200::run_batch (this library, GPU); results must be identical
// byte for byte.  Needs a GPU; run by tests/test_gpu_parity.py.
#include <cstdio>
#include <sstream>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "flatkd/batch.hpp"
#include "flatkd/rng.hpp"
#include "flatkd/testing/instancegen.hpp"
#include "flatkd_b200/reference_adapter.hpp"

namespace {

int failures = 0;

void expect(bool ok, const char* what) {
    if (!ok) {
        ++failures;
        std::printf("FAIL: %s\n", what);
    }
}

bool same(const flatkd::BatchResult& a, const flatkd::BatchResult& b) {
    if (a.stride != b.stride || a.counts != b.counts || a.hits.size() != b.hits.size()) return false;
    return std::memcmp(a.hits.data(), b.hits.data(), a.hits.size() * sizeof(flatkd::Hit)) == 0;
}

struct float3_t {
    float x, y, z;
};

}  // namespace

int main() {
    // uniform batch, all query configurations of the reference's suites
    const auto data = flatkd::random_points(flatkd::derive_stream_seed(7, 1), 50000, 3);
    const auto queries = flatkd::random_points(flatkd::derive_stream_seed(7, 2), 20000, 3);
    const flatkd::KdTree cpu_tree = flatkd::build_tree(data);
    const flatkd::b200::KdTree gpu_tree = flatkd::b200::to_device(cpu_tree);
    for (int kind = 0; kind < 2; ++kind) {
        for (int k : {1, 4, 8, 20, 50}) {
            if (kind == 0 && k != 1) continue;
            for (float r : {flatkd::kInfRadius, 0.25f, 0.01f, 0.0f}) {
                flatkd::BatchOptions o;
                o.kind = kind ? flatkd::QueryKind::knn : flatkd::QueryKind::fcp;
                o.k = k;
                o.max_radius = r;
                o.collect_stats = true;
                const auto ref = flatkd::run_batch(cpu_tree, queries, o);
                const auto gpu = flatkd::b200::run_batch(gpu_tree, queries, o);
                expect(same(ref, gpu), "batch results differ");
                expect(ref.result_hash() == gpu.result_hash(), "result hash differs");
                expect(ref.stats.steps == gpu.stats.steps && ref.stats.nodes_visited == gpu.stats.nodes_visited &&
                           ref.stats.nodes_processed == gpu.stats.nodes_processed,
                       "stats differ");
                o.engine = flatkd::Engine::recursive;
                const auto ref_r = flatkd::run_batch(cpu_tree, queries, o);
                const auto gpu_r = flatkd::b200::run_batch(gpu_tree, queries, o);
                expect(same(ref_r, gpu_r), "recursive-engine results differ");
                expect(ref_r.stats.steps == gpu_r.stats.steps && ref_r.stats.nodes_visited == gpu_r.stats.nodes_visited,
                       "recursive-engine stats differ");
            }
        }
    }

    // several option sets over one query set in one submission (run_batches)
    {
        std::vector<flatkd::BatchOptions> opts(4);
        opts[1].kind = opts[2].kind = opts[3].kind = flatkd::QueryKind::knn;
        opts[1].k = 8;
        opts[2].k = 20;
        opts[2].max_radius = 0.05f;
        opts[3].k = 4;
        opts[3].engine = flatkd::Engine::recursive;
        for (auto& o : opts) o.collect_stats = true;
        const auto gpu = flatkd::b200::run_batches(gpu_tree, queries, std::span<const flatkd::BatchOptions>(opts));
        expect(gpu.size() == opts.size(), "run_batches result count");
        for (std::size_t i = 0; i < opts.size() && i < gpu.size(); ++i) {
            const auto ref = flatkd::run_batch(cpu_tree, queries, opts[i]);
            expect(same(ref, gpu[i]), "run_batches results differ");
            expect(ref.stats.steps == gpu[i].stats.steps && ref.stats.nodes_processed == gpu[i].stats.nodes_processed,
                   "run_batches stats differ");
        }
        // the standalone shim's request form, two query arrays
        flatkd::b200::BatchOptions bo;
        bo.kind = flatkd::b200::QueryKind::knn;
        bo.k = 5;
        const std::vector<flatkd::b200::BatchRequest> reqs{
            {queries.raw().data(), queries.size(), 3, bo},
            {data.raw().data(), 3000, 3, flatkd::b200::BatchOptions{}}};
        const auto two = flatkd::b200::run_batches(gpu_tree, std::span<const flatkd::b200::BatchRequest>(reqs));
        for (int i = 0; i < 2; ++i) {
            const auto one = flatkd::b200::run_batch(gpu_tree, reqs[i].queries, reqs[i].m, 3, reqs[i].options);
            expect(one.counts == two[i].counts && one.hits == two[i].hits, "run_batches requests differ");
        }
        // asynchronous submission: two jobs in flight, collected in order
        auto j1 = flatkd::b200::submit_batches(gpu_tree, std::span<const flatkd::b200::BatchRequest>(reqs));
        auto j2 = flatkd::b200::submit_batches(gpu_tree, std::span<const flatkd::b200::BatchRequest>(reqs));
        const auto a1 = j1.wait();
        const auto a2 = j2.wait();
        for (int i = 0; i < 2; ++i)
            expect(a1[i].counts == two[i].counts && a1[i].hits == two[i].hits && a2[i].hits == two[i].hits,
                   "submit_batches results differ");
    }

    // typed single-query entry points (float3-like struct) vs flatkd::fcp/knn
    for (int i = 0; i < 200; ++i) {
        const auto q = queries[i];
        const float3_t p{q[0], q[1], q[2]};
        const auto ref = flatkd::fcp(cpu_tree, q);
        const auto gpu = flatkd::b200::fcp(gpu_tree, p);
        expect(ref.has_value() == gpu.has_value() && ref->node == gpu->node && ref->dist2 == gpu->dist2,
               "typed fcp differs");
        const auto rk = flatkd::knn(cpu_tree, q, 8, 0.05f);
        const auto gk = flatkd::b200::knn(gpu_tree, p, 8, 0.05f);
        bool eq = rk.size() == gk.size();
        for (std::size_t j = 0; eq && j < rk.size(); ++j) eq = rk[j].node == gk[j].node && rk[j].dist2 == gk[j].dist2;
        expect(eq, "typed knn differs");
    }

    // tie-heavy instances (grid snapping, duplicates, on-plane queries)
    flatkd::testing::InstanceRng rng(11);
    for (int t = 0; t < 40; ++t) {
        const int n = rng.next_int(0, 3000);
        const int dim = rng.next_int(1, 4);
        flatkd::testing::PointGenOptions g;
        g.grid = rng.chance(0.5) ? 8 : 0;
        g.dup_fraction = rng.chance(0.5) ? 0.2 : 0.0;
        const auto pts = flatkd::testing::random_point_set(rng, n, dim, g);
        const auto tree = flatkd::build_tree(pts);
        const auto dt = flatkd::b200::to_device(tree);
        flatkd::PointSet qs(dim);
        for (int j = 0; j < 300; ++j) qs.append(flatkd::testing::random_query(rng, dim, pts));
        for (int k : {1, 3, 8, 16}) {
            flatkd::BatchOptions o;
            o.kind = k == 1 ? flatkd::QueryKind::fcp : flatkd::QueryKind::knn;
            o.k = k;
            o.max_radius = (t % 3 == 0) ? 0.25f : flatkd::kInfRadius;
            o.collect_stats = true;
            const auto ref = flatkd::run_batch(tree, qs, o);
            const auto gpu = flatkd::b200::run_batch(dt, qs, o);
            expect(same(ref, gpu), "tie-heavy results differ");
            expect(ref.stats.nodes_processed == gpu.stats.nodes_processed, "tie-heavy stats differ");
        }
    }

    // the standalone shim: its own types, traces and text output vs the reference
    {
        flatkd::b200::PointSet pts(3, data.raw());
        const auto st_tree = flatkd::b200::build_tree(pts);
        for (int i = 0; i < 50; ++i) {
            const auto q = queries[i];
            flatkd::QueryStats rs;
            flatkd::Trace rt;
            const auto rk = flatkd::knn(cpu_tree, q, 4, 0.1f, &rs, &rt);
            flatkd::b200::QueryStats gs;
            flatkd::b200::Trace gt;
            const auto gk = flatkd::b200::knn(st_tree, q, 4, 0.1f, &gs, &gt);
            bool eq = rk.size() == gk.size() && rt.size() == gt.size() && rs.steps == gs.steps &&
                      rs.nodes_processed == gs.nodes_processed;
            for (std::size_t j = 0; eq && j < rt.size(); ++j)
                eq = rt[j].node == gt[j].node && int(rt[j].kind) == int(gt[j].kind);
            expect(eq, "traced knn differs");
            flatkd::Trace ft;
            flatkd::b200::Trace fg;
            flatkd::fcp(cpu_tree, q, flatkd::kInfRadius, nullptr, &ft);
            flatkd::b200::fcp(st_tree, q, flatkd::b200::kInfRadius, nullptr, &fg);
            expect(flatkd::trace_to_text(ft) == flatkd::b200::trace_to_text(fg), "fcp trace text differs");
        }
        flatkd::BatchOptions o;
        o.kind = flatkd::QueryKind::knn;
        o.k = 3;
        o.max_radius = 0.05f;
        const auto ref = flatkd::run_batch(cpu_tree, queries, o);
        flatkd::b200::BatchOptions bo;
        bo.kind = flatkd::b200::QueryKind::knn;
        bo.k = 3;
        bo.max_radius = 0.05f;
        const auto gpu = flatkd::b200::run_batch(st_tree, flatkd::b200::PointSet(3, queries.raw()), bo);
        std::ostringstream a, b;
        flatkd::write_query_results(a, ref);
        flatkd::b200::write_query_results(b, gpu);
        expect(a.str() == b.str(), "write_query_results text differs");
    }

    // error mapping: the reference's exception types
    try {
        flatkd::BatchOptions o;
        o.kind = flatkd::QueryKind::knn;
        o.k = 0;
        flatkd::b200::run_batch(gpu_tree, queries, o);
        expect(false, "k=0 accepted");
    } catch (const std::invalid_argument&) {
    }
    try {
        flatkd::PointSet bad(3, {0.1f, 0.2f, 0.3f, 0.0f, std::numeric_limits<float>::quiet_NaN(), 0.0f});
        flatkd::b200::run_batch(gpu_tree, bad, flatkd::BatchOptions{});
        expect(false, "NaN query accepted");
    } catch (const flatkd::DataError& e) {
        expect(std::string(e.what()) == "queries: non-finite coordinate in point 1", "NaN message differs");
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
