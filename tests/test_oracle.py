"""The oracle is pinned before it is trusted (CPU only).

* against the committed golden fixtures produced by the UNMODIFIED reference
  (tests/golden/make_golden.py): Fig. 1, traces, batch hashes + stats over
  dims 1-8 and all query configurations, tie-heavy instancegen instances,
  the C1/C2 survey hashes;
* against the reference library itself (oracle/_ref) where it is present.
"""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
INF = float("inf")


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "golden.json")) as f:
        return json.load(f)


def _hits(h):
    return [[int(x["node"]), float(x["dist2"])] for x in h]


def test_figure1(oracle, golden):
    fig = golden["figure1"]
    pts = np.array(fig["points"], np.float32)
    tree = oracle.build_tree(pts)
    assert tree.tolist() == fig["level_order"]
    for case in fig["queries"]:
        hits, st, tr = oracle.query(tree, case["q"], case["kind"], case["k"], case["max_radius"], trace_cap=64)
        assert _hits(hits) == case["hits"], case
        assert [int(st["steps"]), int(st["nodes_visited"]), int(st["nodes_processed"])] == case["stats"]
        assert tr.tolist() == case["trace"]


def test_rng_streams(oracle, golden):
    got = oracle.random_points(oracle.derive_stream_seed(1, 1), 4, 3).reshape(-1).tolist()
    assert got == golden["random_points_seed1_stream1_first12"]
    for s, v in golden["derive_stream_seed"].items():
        assert oracle.derive_stream_seed(1, int(s)) == int(v)


def test_batches_all_configs(oracle, golden):
    trees = {}
    for case in golden["batches"]:
        dim, seed = case["dim"], case["seed"]
        if dim not in trees:
            pts = oracle.random_points(oracle.derive_stream_seed(seed, 1), case["n"], dim)
            qs = oracle.random_points(oracle.derive_stream_seed(seed, 2), case["m"], dim) * np.float32(1.5) - np.float32(0.25)
            trees[dim] = (oracle.build_tree(pts), qs)
        nodes, qs = trees[dim]
        c, h, st, _ = oracle.run_batch(nodes, qs, case["kind"], case["k"], case["max_radius"])
        stride = case["k"] if case["kind"] == "knn" else 1
        assert f"{oracle.result_hash(c, h, stride):016x}" == case["hash"], case
        assert [int(st["steps"]), int(st["nodes_visited"]), int(st["nodes_processed"])] == case["stats"]
        _, _, st_r, _ = oracle.run_batch(nodes, qs, case["kind"], case["k"], case["max_radius"], recursive=True)
        assert [int(st_r["steps"]), int(st_r["nodes_visited"]), int(st_r["nodes_processed"])] == case["stats_recursive"]


def test_tie_heavy_instances(oracle, golden):
    for inst in golden["instances"]:
        pts = np.array(inst["points"], np.float32).reshape(inst["n"], inst["dim"])
        nodes = oracle.build_tree(pts)
        assert nodes.tolist() == inst["level_order"]
        assert oracle.verify_tree(nodes)
        qs = np.array(inst["queries"], np.float32)
        for res in inst["results"]:
            c, h, st, _ = oracle.run_batch(nodes, qs, res["kind"], res["k"], res["max_radius"])
            assert c.tolist() == res["counts"]
            assert _hits(h) == res["hits"]
            assert [int(st["steps"]), int(st["nodes_visited"]), int(st["nodes_processed"])] == res["stats"]
            # brute force agrees with the tree walk (testing/oracle.cpp:15-43)
            bc, bh = oracle.brute_batch(nodes, qs, res["kind"], res["k"], res["max_radius"])
            assert np.array_equal(bc, c) and bh.tobytes() == h.tobytes()


def test_instance_rng_reproduces_reference_generator(oracle, golden):
    rng = oracle.instance_rng(2024)
    for t, inst in enumerate(golden["instances"][:10]):
        n = 1 + (rng.next_u64() % 700)
        dim = 1 + (rng.next_u64() % 4)
        assert (n, dim) == (inst["n"], inst["dim"])
        pts = rng.random_point_set(int(n), int(dim), inst["grid"], inst["dup"])
        assert np.array_equal(pts, np.array(inst["points"], np.float32).reshape(n, dim))
        qs = np.stack([rng.random_query(int(dim), pts) for _ in range(40)])
        assert np.array_equal(qs, np.array(inst["queries"], np.float32))


@pytest.mark.slow
def test_c1_c2_hashes(oracle, golden):
    data = oracle.random_points(oracle.derive_stream_seed(1, 1), 1_000_000, 3)
    qs = oracle.random_points(oracle.derive_stream_seed(1, 2), 1_000_000, 3)
    nodes = oracle.build_tree(data)
    for name, kind, k, r in (("c1_fcp", "fcp", 1, INF), ("c2_knn8_r001", "knn", 8, 0.01)):
        c, h, st, _ = oracle.run_batch(nodes, qs, kind, k, r)
        assert f"{oracle.result_hash(c, h, k if kind == 'knn' else 1):016x}" == golden["c1_c2"][name]["hash"]
        assert [int(st["steps"]), int(st["nodes_visited"]), int(st["nodes_processed"])] == golden["c1_c2"][name]["stats"]


def test_reference_suites_recorded_green(golden):
    for name, (fails, checks) in golden["suites"].items():
        assert fails == 0 and checks > 0, name


# ---- against the reference library itself, where it was built ----

def test_oracle_vs_reference_instancegen(oracle, reference):
    orng = oracle.instance_rng(99)
    rrng = reference.instance_rng(99)
    for _ in range(60):
        a, b = orng.next_u64(), rrng.next_u64()
        assert a == b
        n, dim = 1 + a % 900, 1 + (a >> 20) % 5
        grid, dup = (8, 0.2) if a & 1 else (0, 0.0)
        p1 = orng.random_point_set(int(n), int(dim), grid, dup)
        p2 = rrng.random_point_set(int(n), int(dim), grid, dup)
        assert np.array_equal(p1, p2)
        nodes = reference.build_tree(p2)
        assert np.array_equal(oracle.build_tree(p1), nodes)
        qs1 = np.stack([orng.random_query(int(dim), p1) for _ in range(30)])
        qs2 = np.stack([rrng.random_query(int(dim), p2) for _ in range(30)])
        assert np.array_equal(qs1, qs2)
        for kind, k, r in (("fcp", 1, INF), ("knn", 5, 0.25), ("knn", 16, INF), ("knn", 50, 0.01)):
            for engine in (0, 1):
                c1, h1, s1, _ = oracle.run_batch(nodes, qs1, kind, k, r, recursive=bool(engine))
                c2, h2, s2, _ = reference.run_batch(nodes, qs2, kind, k, r, engine=engine, collect_stats=True)
                assert np.array_equal(c1, c2) and h1.tobytes() == h2.tobytes()
                assert [int(s1["steps"]), int(s1["nodes_visited"]), int(s1["nodes_processed"])] == s2.tolist()
        for q in qs1[:5]:
            for kind, k in (("fcp", 1), ("knn", 4)):
                h1, st1, t1 = oracle.query(nodes, q, kind, k, trace_cap=100000)
                h2, st2, t2 = reference.query(nodes, q, kind, k, trace_cap=100000)
                assert h1.tobytes() == h2.tobytes() and np.array_equal(t1, t2)


def test_oracle_errors_match_reference(oracle, reference):
    from oracle import OracleError

    nodes = oracle.build_tree(oracle.random_points(1, 50, 3))
    bad = np.zeros((4, 3), np.float32)
    bad[2, 1] = np.nan
    for impl in (oracle, reference):
        with pytest.raises(OracleError) as e:
            impl.run_batch(nodes, bad)
        assert e.value.code == 2 and e.value.msg == "queries: non-finite coordinate in point 2"
        with pytest.raises(OracleError) as e:
            impl.run_batch(nodes, bad, "knn", 0)
        assert e.value.code == 1
        with pytest.raises(OracleError) as e:
            impl.run_batch(nodes, np.zeros((2, 2), np.float32))
        assert e.value.msg == "query dimension 2 does not match tree dimension 3"
    # empty tree: no dimension or finiteness checks (batch.cpp:75)
    empty = np.zeros((0, 3), np.float32)
    c, h, _, _ = oracle.run_batch(empty, bad[:, :2].copy(), "knn", 2)
    assert c.tolist() == [0] * 4 and (h["node"] == -1).all()
