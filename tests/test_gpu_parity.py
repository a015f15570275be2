"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bit-exact bar: counts exact, hit nodes and dist2 bits
identical, per-query nodes_processed/visited/steps identical to the
reference's stack-free walk (traverse.hpp:198-248), result_hash equal.
"""
import os
import subprocess

import numpy as np
import pytest

import paper_2210_12859_b200 as fk

pytestmark = pytest.mark.gpu

INF = float("inf")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _kind(k):
    return fk.QueryKind.knn if k > 0 else fk.QueryKind.fcp


def _run_both(oracle, nodes, qs, k, r, morton=True, engine=0):
    """k == 0 -> fcp.  Returns (gpu BatchResult, oracle tuple)."""
    tree = fk.KdTree.from_level_order(nodes)
    opt = fk.BatchOptions(kind=_kind(k), k=max(k, 1), max_radius=r, collect_stats=True,
                          morton=morton, engine=fk.Engine(engine))
    res = fk.run_batch(tree, qs, opt)
    ref = oracle.run_batch(nodes, qs, "knn" if k > 0 else "fcp", max(k, 1), r,
                           recursive=bool(engine), per_query=True)
    return res, ref


def _assert_same(res, ref, what=""):
    c, h, st, _ = ref
    assert np.array_equal(res.counts, c), f"counts differ {what}"
    if res.hits.tobytes() != h.tobytes():
        bad = np.nonzero(res.hits.view(np.uint64) != h.view(np.uint64))[0][:5]
        raise AssertionError(f"hits differ {what} at {bad}: gpu={res.hits[bad]} ref={h[bad]}")
    assert (res.stats.steps, res.stats.nodes_visited, res.stats.nodes_processed) == \
        (int(st["steps"]), int(st["nodes_visited"]), int(st["nodes_processed"])), f"stats {what}"


def test_figure1_goldens():
    # SPEC.md:141-171, selfcheck.cpp:268-274 (Fig. 1 of the paper)
    pts = np.array([[2, 3], [5, 4], [9, 6], [4, 7], [8, 1], [7, 2]], np.float32)
    nodes = fk.build_level_order(pts)
    assert nodes.tolist() == [[7, 2], [5, 4], [9, 6], [2, 3], [4, 7], [8, 1]]
    tree = fk.KdTree.from_level_order(nodes)
    hit, st = fk.fcp(tree, [9, 2], stats=True)
    assert hit == (5, 2.0)
    assert (st.steps, st.nodes_visited, st.nodes_processed) == (9, 7, 3)
    assert fk.fcp(tree, [2, 3]) == (3, 0.0)
    assert fk.knn(tree, [9, 2], 2) == [(5, 2.0), (0, 4.0)]
    assert fk.fcp(tree, [9, 2], max_radius=1.0) is None
    res = fk.run_batch(tree, np.array([[9, 2], [2, 3]], np.float32),
                       fk.BatchOptions(kind=fk.QueryKind.knn, k=3))
    assert fk.write_query_results(res) == "3,5,1.41421354,0,2,2,4\n3,3,0,1,3.1622777,4,4.47213602\n"


@pytest.mark.parametrize("dim", [1, 2, 3, 4, 5, 8, 9])
def test_uniform_all_configs(oracle, dim):
    n, m = 5000, 3000
    nodes = oracle.build_tree(oracle.random_points(100 + dim, n, dim))
    qs = oracle.random_points(200 + dim, m, dim) * np.float32(1.2) - np.float32(0.1)
    for k in (0, 1, 2, 3, 4, 8, 16, 20, 33, 50, 64, 65, 100):
        for r in (INF, 0.25, 0.01, 0.0):
            res, ref = _run_both(oracle, nodes, qs, k, r)
            _assert_same(res, ref, f"dim={dim} k={k} r={r}")


def test_tie_heavy_instances(oracle):
    """instancegen-style trees (grid snap, duplicates) and queries (exact hits,
    on-plane) — the cases that pin hit_order (SURVEY §8(c) tie coverage)."""
    rng = oracle.instance_rng(4242)
    for t in range(120):
        n = rng.next_int(0, 2500)
        dim = rng.next_int(1, 6)
        grid = (8 if rng.chance(0.5) else 16) if rng.chance(0.6) else 0
        dup = 0.2 if rng.chance(0.5) else 0.0
        pts = rng.random_point_set(n, dim, grid, dup)
        nodes = oracle.build_tree(pts) if n else pts
        qs = np.stack([rng.random_query(dim, pts) for _ in range(200)])
        for k in (0, 1, 4, 8, 20, 50):
            r = (INF, 0.25, 0.01, 0.0)[rng.next_int(0, 3)]
            res, ref = _run_both(oracle, nodes.reshape(n, dim), qs, k, r, morton=bool(t % 2))
            _assert_same(res, ref, f"tree#{t} n={n} dim={dim} k={k} r={r}")


def test_recursive_engine_stats(oracle):
    nodes = oracle.build_tree(oracle.random_points(5, 3000, 3))
    qs = oracle.random_points(6, 2000, 3)
    for k in (0, 8):
        res, ref = _run_both(oracle, nodes, qs, k, 0.1, engine=1)
        _assert_same(res, ref, f"recursive k={k}")


def test_per_query_stats_device(oracle):
    import torch

    nodes = oracle.build_tree(oracle.random_points(9, 20000, 3))
    qs = oracle.random_points(10, 5000, 3)
    tree = fk.KdTree.from_level_order(nodes)
    dq = torch.from_numpy(qs).cuda()
    counts = torch.empty(5000, dtype=torch.int32, device="cuda")
    hits = torch.empty(5000 * 8, dtype=torch.int64, device="cuda")
    pq = torch.empty(5000 * 3, dtype=torch.int64, device="cuda")
    st, tm = fk.run_batch_device(tree, dq, counts, hits, fk.BatchOptions(kind=fk.QueryKind.knn, k=8,
                                 collect_stats=True), per_query=pq, timings=True)
    c, h, tot, per = oracle.run_batch(nodes, qs, "knn", 8, INF, per_query=True)
    assert np.array_equal(counts.cpu().numpy(), c)
    assert hits.cpu().numpy().tobytes() == h.tobytes()
    got = pq.cpu().numpy().reshape(-1, 3)
    assert np.array_equal(got[:, 2], per["nodes_processed"])
    assert np.array_equal(got[:, 1], per["nodes_visited"])
    assert np.array_equal(got[:, 0], per["steps"])
    assert tm["walk_launches"] >= 1


def test_unordered_matches_brute_force(oracle):
    for dim in (2, 4, 8):
        nodes = oracle.build_tree(oracle.random_points(30 + dim, 4000, dim))
        qs = oracle.random_points(40 + dim, 1000, dim)
        tree = fk.KdTree.from_level_order(nodes)
        for k, r in ((16, INF), (16, 0.2), (1, INF)):
            opt = fk.BatchOptions(kind=fk.QueryKind.knn, k=k, max_radius=r, unordered=True)
            res = fk.run_batch(tree, qs, opt)
            c, h = oracle.brute_batch(nodes, qs, "knn", k, r)
            assert np.array_equal(res.counts, c)
            assert res.hits.tobytes() == h.tobytes()


@pytest.mark.parametrize("k,r,golden", [
    (0, INF, 0x79446ad66bb295e9),   # C1 fcp 3D N=1M M=1M
    (8, INF, 0x220c5639002591a1),   # kNN8 maxR=inf
    (8, 0.01, 0xd50e9239b721b47a),  # kNN8 maxR=0.01
])
def test_c1_c2_golden_hashes(k, r, golden):
    data = fk.random_points(1, 1, 1_000_000, 3)
    qs = fk.random_points(1, 2, 1_000_000, 3)
    tree = fk.build_tree(data)
    res = fk.run_batch(tree, qs, fk.BatchOptions(kind=_kind(k), k=max(k, 1), max_radius=r,
                                                 collect_stats=True))
    assert res.result_hash() == golden
    if k == 0:
        assert (res.stats.steps, res.stats.nodes_visited, res.stats.nodes_processed) == \
            (108117642, 96233846, 42675025)


def test_edge_cases(oracle):
    tree = fk.KdTree.from_level_order(np.zeros((0, 3), np.float32))
    res = fk.run_batch(tree, np.full((4, 3), np.nan, np.float32), fk.BatchOptions(kind=fk.QueryKind.knn, k=3))
    assert res.counts.tolist() == [0] * 4 and (res.hits["node"] == -1).all() and np.isinf(res.hits["dist2"]).all()
    nodes = oracle.build_tree(oracle.random_points(3, 100, 3))
    tree = fk.KdTree.from_level_order(nodes)
    assert fk.run_batch(tree, np.zeros((0, 3), np.float32)).counts.size == 0
    qs = oracle.random_points(4, 10, 3)
    qs[7, 1] = np.inf
    qs[9, 0] = np.nan
    with pytest.raises(fk.DataError, match="queries: non-finite coordinate in point 7"):
        fk.run_batch(tree, qs)
    with pytest.raises(fk.DataError, match="query dimension 2 does not match tree dimension 3"):
        fk.run_batch(tree, np.zeros((5, 2), np.float32))
    with pytest.raises(fk.InvalidArgument):
        fk.run_batch(tree, qs, fk.BatchOptions(kind=fk.QueryKind.knn, k=0))
    with pytest.raises(fk.DataError, match="max radius"):
        fk.run_batch(tree, qs, fk.BatchOptions(max_radius=float("nan")))
    with pytest.raises(fk.DataError, match="tree nodes: non-finite coordinate in point 1"):
        fk.KdTree.from_level_order(np.array([[0, 0], [np.inf, 1]], np.float32))
    # single-query validation order: radius before k (traverse.hpp:115-117)
    with pytest.raises(fk.DataError):
        fk.knn(tree, [0, 0, 0], 0, max_radius=-1.0)


def test_device_tree_and_path_match_host(oracle):
    import torch

    pts = oracle.random_points(77, 30000, 3)
    nodes = oracle.build_tree(pts)
    t_host = fk.KdTree.from_level_order(nodes)
    t_dev = fk.KdTree.from_device(torch.from_numpy(nodes).cuda())
    qs = oracle.random_points(78, 10000, 3)
    a = fk.run_batch(t_host, qs, fk.BatchOptions(kind=fk.QueryKind.knn, k=4, max_radius=0.05))
    b = fk.run_batch(t_dev, qs, fk.BatchOptions(kind=fk.QueryKind.knn, k=4, max_radius=0.05))
    assert a.hits.tobytes() == b.hits.tobytes() and np.array_equal(a.counts, b.counts)


def test_cpp_shim_against_reference():
    exe = os.path.join(ROOT, "tests", "cpp", "shim_parity")
    if not os.path.exists(exe):
        pytest.skip("shim_parity not built (needs the reference headers at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK" in out.stdout


@pytest.mark.parametrize("budget,resume_min,resume_trips,rounds", [
    ("1", "0", "0", "0"), ("3", "0", "0", "0"), ("50", "0", "0", "0"),   # CTA pass only (few overflow)
    ("2", "1", "-1", "0"), ("40", "1", "-1", "0"),                       # unbounded resume pass
    ("2", "1", "3", "0"), ("5", "1", "40", "0"), ("40", "1", "0", "0"),  # budgeted resume, survivors -> CTA pass
    ("1", "0", "0", "1,1,2,3"), ("4", "0", "0", "4,8"),                  # continuation rounds -> CTA pass
    ("2", "1", "6", "1,2,4"), ("8", "1", "-1", "8"),                     # rounds -> resume pass -> CTA pass
    ("-1", "0", "0", "-"),                                               # the defaults
])
def test_overflow_pass_is_exact(oracle, budget, resume_min, resume_trips, rounds, monkeypatch):
    """Queries stopped by the walk budget continue in compacted continuation
    rounds (walk_round_kernel, FKD_RROUNDS_*), then are finished by the
    CTA-per-query overflow pass (overflow.cuh) or, when many remain
    (FKD_RESUME_MIN=1 forces it), resumed from their parked (curr, prev) by the
    plain-grid resume pass for FKD_RESUME_TRIPS more steps, whose survivors are
    parked again and handed to the CTA pass; results must stay bit-exact in
    every combination."""
    monkeypatch.setenv("FKD_BUDGET", budget)
    monkeypatch.setenv("FKD_RESUME_TRIPS", resume_trips)
    if rounds != "-":
        monkeypatch.setenv("FKD_RROUNDS_FCP", rounds)
        monkeypatch.setenv("FKD_RROUNDS_KNN", rounds)
    if resume_min != "0":
        monkeypatch.setenv("FKD_RESUME_MIN", resume_min)
    else:
        monkeypatch.setenv("FKD_RESUME_MIN", str(1 << 40))
    rng = oracle.instance_rng(777)
    for t in range(24):
        n = rng.next_int(1, 6000)
        dim = rng.next_int(1, 8)
        grid = 8 if t % 3 == 0 else 0
        pts = rng.random_point_set(n, dim, grid, 0.2 if t % 2 else 0.0)
        nodes = oracle.build_tree(pts)
        qs = np.stack([rng.random_query(dim, pts) for _ in range(300)])
        tree = fk.KdTree.from_level_order(nodes)
        for k, r in ((0, INF), (1, 0.25), (4, INF), (8, 0.01), (16, INF), (20, 0.25), (50, INF), (64, 0.0)):
            res = fk.run_batch(tree, qs, fk.BatchOptions(kind=_kind(k), k=max(k, 1), max_radius=r))
            ref = oracle.run_batch(nodes, qs, "knn" if k else "fcp", max(k, 1), r)
            bad = np.nonzero(res.counts != ref[0])[0]
            kk = max(k, 1)
            if len(bad) == 0:
                hb = np.nonzero((res.hits.view(np.uint64) != ref[1].view(np.uint64)).reshape(-1, kk).any(1))[0]
                bad = hb
            assert len(bad) == 0, (t, n, dim, k, r, len(bad), bad[:3].tolist(), res.counts[bad[:1]].tolist(),
                                   ref[0][bad[:1]].tolist(), res.hits.reshape(-1, kk)[bad[:1]].tolist(),
                                   ref[1].reshape(-1, kk)[bad[:1]].tolist())


def test_overflow_clustered_tail(oracle, monkeypatch):
    monkeypatch.setenv("FKD_BUDGET", "256")
    pts = fk.clustered_points(3, 1, 200_000, 3)
    qs = fk.clustered_points(3, 2, 20_000, 3)
    nodes = fk.build_level_order(pts)
    tree = fk.KdTree.from_level_order(nodes)
    for k in (0, 8):
        res = fk.run_batch(tree, qs, fk.BatchOptions(kind=_kind(k), k=max(k, 1)))
        c, h, _, _ = oracle.run_batch(nodes, qs, "knn" if k else "fcp", max(k, 1), INF)
        assert np.array_equal(res.counts, c) and res.hits.tobytes() == h.tobytes()


def test_gpu_builder_byte_identical(oracle):
    """csrc/build.cu vs the reference builder restated (tree.cpp:55-89)."""
    import torch

    rng = oracle.instance_rng(31337)
    cases = [(0, 3), (1, 1), (2, 2), (7, 3), (100, 4), (1000, 3), (4097, 2), (30000, 3), (20000, 8), (5000, 11)]
    for n, dim in cases:
        pts = oracle.random_points(n + dim, n, dim)
        tree = fk.build_tree(pts)
        assert np.array_equal(tree.nodes(), oracle.build_tree(pts)), (n, dim)
    for t in range(40):  # ties: grid snapping, duplicates, signed zeros
        n = rng.next_int(1, 5000)
        dim = rng.next_int(1, 5)
        pts = rng.random_point_set(n, dim, (8, 16, 2)[t % 3], 0.3 if t % 2 else 0.0)
        if t % 4 == 0:
            pts = pts - np.float32(0.5)
            pts[rng.next_int(0, n - 1)] = -0.0
        want = oracle.build_tree(pts)
        got = fk.build_level_order_device(torch.from_numpy(pts).cuda()).cpu().numpy()
        assert got.tobytes() == want.tobytes(), (t, n, dim)
    with pytest.raises(fk.DataError, match="build: non-finite coordinate in point 3"):
        bad = oracle.random_points(1, 10, 3)
        bad[3, 1] = np.inf
        fk.build_tree(bad)


def test_gpu_builder_c1_scale():
    data = fk.random_points(1, 1, 1_000_000, 3)
    assert np.array_equal(fk.build_tree(data).nodes(), fk.build_level_order(data))


def test_device_trace_matches_reference_trace(oracle):
    """fkd_trace_batch (trace.cu) records the reference's Trace event list
    (traverse.hpp:56-68, 206-222) and QueryStats, per query."""
    rng = oracle.instance_rng(55)
    for t in range(30):
        n = rng.next_int(0, 800)
        dim = rng.next_int(1, 5)
        pts = rng.random_point_set(n, dim, 8 if t % 2 else 0, 0.2)
        nodes = oracle.build_tree(pts) if n else pts.reshape(0, dim)
        qs = np.stack([rng.random_query(dim, pts) for _ in range(20)])
        tree = fk.KdTree.from_level_order(nodes)
        for kind, k, r in ((fk.QueryKind.fcp, 1, INF), (fk.QueryKind.knn, 5, 0.25), (fk.QueryKind.knn, 70, INF)):
            counts, hits, stats, events = fk.trace(tree, qs, kind, k, r, cap=20000)
            stride = k if kind == fk.QueryKind.knn else 1
            for i, q in enumerate(qs):
                h, st, tr = oracle.query(nodes, q, "knn" if kind == fk.QueryKind.knn else "fcp", k, r,
                                         trace_cap=20000)
                assert counts[i] == len(h)
                assert hits[i * stride: i * stride + len(h)].tobytes() == h.tobytes()
                assert tuple(stats[i]) == (int(st["steps"]), int(st["nodes_visited"]), int(st["nodes_processed"]))
                assert np.array_equal(events[i], tr), (t, i)


def test_binary_files_round_trip_with_reference(oracle, reference, tmp_path):
    import torch

    pts = oracle.random_points(3, 5000, 3)
    nodes = oracle.build_tree(pts)
    p1, p2, p3 = str(tmp_path / "a.fkdt"), str(tmp_path / "b.fkdx"), str(tmp_path / "c.fkdt")
    reference.write_file(p1, pts)                       # reference writer -> our device reader
    reference.write_file(p2, nodes, tree=True)
    assert np.array_equal(fk.read_points_file_device(p1).cpu().numpy(), pts)
    tree = fk.load_tree(p2)
    assert tree.size() == 5000 and tree.dim() == 3
    qs = oracle.random_points(4, 1000, 3)
    res = fk.run_batch(tree, qs, fk.BatchOptions(kind=fk.QueryKind.knn, k=4))
    c, h, _, _ = oracle.run_batch(nodes, qs, "knn", 4)
    assert res.hits.tobytes() == h.tobytes()
    fk.write_points_file(p3, pts)                       # our writer: byte-identical to the reference's
    assert open(p3, "rb").read() == open(p1, "rb").read()
    with pytest.raises(fk.DataError, match="file has magic FKDX, expected FKDT"):
        fk.read_points_file_device(p2)
    bad = pts.copy()
    bad[17, 2] = np.nan
    fk.write_points_file(p3, bad)
    with pytest.raises(fk.DataError, match="non-finite coordinate in point 17"):
        fk.read_points_file_device(p3)
    with open(p3, "wb") as f:
        f.write(b"FKDT" + (1).to_bytes(4, "little") + (3).to_bytes(4, "little") + (5000).to_bytes(8, "little"))
    with pytest.raises(fk.DataError, match="payload size does not match header"):
        fk.read_points_file_device(p3)


def test_multi_replica_sharding(oracle, monkeypatch):
    """fkd_tree_create with a device list shards a host batch across the
    replicas (capi.cu fkd_run_batch); two replicas on GPU 0 exercise the
    per-device workspaces, streams and result placement on a 1-GPU box."""
    monkeypatch.setenv("FKD_CHUNK", "3000")
    pts = oracle.random_points(12, 40000, 3)
    nodes = oracle.build_tree(pts)
    qs = oracle.random_points(13, 25001, 3)
    one = fk.KdTree.from_level_order(nodes, devices=[0])
    two = fk.KdTree.from_level_order(nodes, devices=[0, 0])
    three = fk.build_tree(pts, devices=[0, 0, 0])
    for kind, k, r in ((fk.QueryKind.fcp, 1, INF), (fk.QueryKind.knn, 8, 0.05), (fk.QueryKind.knn, 100, INF)):
        opt = fk.BatchOptions(kind=kind, k=k, max_radius=r, collect_stats=True)
        a, b, c = fk.run_batch(one, qs, opt), fk.run_batch(two, qs, opt), fk.run_batch(three, qs, opt)
        assert a.hits.tobytes() == b.hits.tobytes() == c.hits.tobytes()
        assert np.array_equal(a.counts, b.counts) and np.array_equal(a.counts, c.counts)
        assert a.stats == b.stats == c.stats
    bad = qs.copy()
    bad[20000, 2] = np.nan  # lands in the second replica's shard: global index reported
    with pytest.raises(fk.DataError, match="non-finite coordinate in point 20000"):
        fk.run_batch(two, bad)


def test_k_larger_than_tree_and_huge_k(oracle):
    nodes = oracle.build_tree(oracle.random_points(21, 37, 2))
    qs = oracle.random_points(22, 500, 2)
    tree = fk.KdTree.from_level_order(nodes)
    for k in (37, 38, 64, 65, 200, 1000):
        res = fk.run_batch(tree, qs, fk.BatchOptions(kind=fk.QueryKind.knn, k=k))
        c, h, _, _ = oracle.run_batch(nodes, qs, "knn", k)
        assert np.array_equal(res.counts, c) and res.hits.tobytes() == h.tobytes()


@pytest.mark.parametrize("shape", ["identical", "collinear", "two_values", "pow2"])
def test_degenerate_trees(oracle, shape, monkeypatch):
    """All-tie inputs: every distance equal (identical points) or planes that
    never separate (collinear, two values).  Every subtree stays in range, so
    walks are long (budget -> overflow / resume passes) and every answer is
    decided by the node-index tie rule (traverse.hpp:80-83)."""
    rng = np.random.default_rng(7)
    if shape == "identical":
        pts = np.full((3000, 3), 0.25, np.float32)
    elif shape == "collinear":
        t = rng.random(4000, dtype=np.float32)
        pts = np.stack([t, np.full_like(t, 0.5), np.full_like(t, 0.5)], 1)
    elif shape == "two_values":
        pts = rng.integers(0, 2, size=(4000, 2)).astype(np.float32)
    else:
        pts = rng.random((4095, 4), dtype=np.float32)
    nodes = oracle.build_tree(pts)
    qs = np.concatenate([pts[:50], rng.random((250, pts.shape[1]), dtype=np.float32)])
    tree = fk.KdTree.from_level_order(nodes)
    for budget in ("-1", "5"):
        monkeypatch.setenv("FKD_BUDGET", budget)
        for k, r in ((0, INF), (8, INF), (64, 0.1), (100, INF)):
            res = fk.run_batch(tree, qs, fk.BatchOptions(kind=_kind(k), k=max(k, 1), max_radius=r))
            c, h, _, _ = oracle.run_batch(nodes, qs, "knn" if k else "fcp", max(k, 1), r)
            assert np.array_equal(res.counts, c), (shape, budget, k)
            assert res.hits.tobytes() == h.tobytes(), (shape, budget, k)
    pts2 = rng.random((4096, 3), dtype=np.float32)  # exactly 2^12 nodes: one node on the last level
    nodes2 = oracle.build_tree(pts2)
    q3 = np.ascontiguousarray(qs[:, :3]) if qs.shape[1] >= 3 else rng.random((300, 3), dtype=np.float32)
    res = fk.run_batch(fk.KdTree.from_level_order(nodes2), q3,
                       fk.BatchOptions(kind=fk.QueryKind.knn, k=4, collect_stats=True))
    c, h, st, _ = oracle.run_batch(nodes2, q3, "knn", 4)
    assert res.hits.tobytes() == h.tobytes() and res.stats.nodes_processed == int(st["nodes_processed"])


def test_concurrent_callers_share_one_tree(oracle):
    """any number of concurrent callers may share a tree.  Host
    threads (ctypes drops the GIL) run different batches at once through the
    host path and the single-query entry points; each gets its own pooled
    workspace and stream."""
    import threading

    nodes = oracle.build_tree(oracle.random_points(61, 50000, 3))
    tree = fk.KdTree.from_level_order(nodes)
    jobs = []
    for t in range(8):
        qs = oracle.random_points(100 + t, 20000 + 997 * t, 3)
        k = (0, 1, 4, 8, 16, 20, 50, 100)[t]
        jobs.append((qs, k, oracle.run_batch(nodes, qs, "knn" if k else "fcp", max(k, 1), 0.2)))
    errors = []

    def worker(i):
        qs, k, (c, h, _, _) = jobs[i]
        try:
            for _ in range(3):
                res = fk.run_batch(tree, qs, fk.BatchOptions(kind=_kind(k), k=max(k, 1), max_radius=0.2))
                assert np.array_equal(res.counts, c) and res.hits.tobytes() == h.tobytes()
                q0 = qs[i]
                one = fk.knn(tree, q0, max(k, 1), 0.2) if k else fk.fcp(tree, q0, 0.2)
                assert one is not None or k == 0
        except Exception as e:  # noqa: BLE001
            errors.append((i, repr(e)))

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(8)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors


@pytest.mark.parametrize("staging,streams,chunk_div,budget,first_div,ramp", [
    ("1", "4", "8", "-1", "1", "2,2"),     # defaults: full staging, graduated chunks
    ("0", "4", "8", "-1", "1", "2,2"),     # ring staging (slot reuse waits)
    ("1", "2", "16", "40", "4", "2,2"),    # forced overflow in every chunk, smaller first budget
    ("0", "3", "5", "7", "1", "2,2"),      # ring + forced overflow + resume
    ("1", "4", "2", "-1", "1", "5,1"),     # deep head ramp, short tail ramp
    ("0", "2", "2", "40", "1", "0,6"),     # no head ramp, deep tail ramp, ring staging
])
def test_host_pipeline_chunks_exact(oracle, staging, streams, chunk_div, budget, first_div, ramp, monkeypatch):
    """fkd_run_batch's chunked pipeline (capi.cu: copy-in stream, slot streams,
    high-priority tail stream, copy-out stream; full or ring staging) returns
    exactly the oracle's results and the device path's, with over-budget
    queries finished inside the chunks."""
    import torch
    monkeypatch.setenv("FKD_FULL_STAGING", staging)
    monkeypatch.setenv("FKD_STREAMS", streams)
    monkeypatch.setenv("FKD_CHUNK_DIV", chunk_div)
    monkeypatch.setenv("FKD_BUDGET", budget)
    monkeypatch.setenv("FKD_FIRST_BUDGET_DIV", first_div)
    monkeypatch.setenv("FKD_RESUME_MIN", "50")
    monkeypatch.setenv("FKD_RAMP_HEAD", ramp.split(",")[0])
    monkeypatch.setenv("FKD_RAMP_TAIL", ramp.split(",")[1])
    pts = fk.clustered_points(5, 1, 60_000, 3)
    # 650,001 queries: > 2 x the 256k minimum full chunk, so the graduated schedule (ramps) is used
    qs = fk.clustered_points(5, 2, 2_600_001, 3)[::4].copy()
    nodes = oracle.build_tree(pts)
    tree = fk.KdTree.from_level_order(nodes)
    for kind, k, r in ((fk.QueryKind.fcp, 1, INF), (fk.QueryKind.knn, 8, INF), (fk.QueryKind.knn, 20, 0.01)):
        res = fk.run_batch(tree, qs, fk.BatchOptions(kind=kind, k=k, max_radius=r))
        sample = np.arange(0, len(qs), 97)
        ref = oracle.run_batch(nodes, qs[sample], "knn" if kind == fk.QueryKind.knn else "fcp", k, r)
        assert np.array_equal(res.counts[sample], ref[0])
        assert res.hits.reshape(len(qs), -1)[sample].tobytes() == ref[1].reshape(len(sample), -1).tobytes()
        dq = torch.from_numpy(qs).cuda()
        c = torch.empty(len(qs), dtype=torch.int32, device="cuda")
        h = torch.empty(len(qs) * k, dtype=torch.int64, device="cuda")
        fk.run_batch_device(tree, dq, c, h, fk.BatchOptions(kind=kind, k=k, max_radius=r))
        assert np.array_equal(c.cpu().numpy(), res.counts)
        assert h.cpu().numpy().tobytes() == res.hits.tobytes()


@pytest.mark.parametrize("mode", ["pageable-staged", "pageable-direct", "pinned"])
def test_host_buffers_pinned_and_pageable(oracle, mode, monkeypatch):
    """fkd_run_batch with pinned caller buffers, with pageable ones staged
    through the library's pinned pool (CopyPool, capi.cu), and with pageable
    ones handed to cudaMemcpyAsync directly (FKD_PAGEABLE_STAGING=0): the
    same bytes as the device path in every mode."""
    import ctypes as C
    import torch
    monkeypatch.setenv("FKD_PAGEABLE_STAGING", "0" if mode == "pageable-direct" else "1")
    pts = fk.clustered_points(6, 1, 50_000, 3)
    qs = fk.clustered_points(6, 2, 700_001, 3)
    tree = fk.KdTree.from_level_order(oracle.build_tree(pts))
    m = len(qs)
    for kind, k in ((fk.QueryKind.fcp, 1), (fk.QueryKind.knn, 8)):
        o = fk.BatchOptions(kind=kind, k=k).to_c()
        if mode == "pinned":
            hq = fk.LIB.fkd_host_alloc(qs.nbytes)
            C.memmove(hq, qs.ctypes.data, qs.nbytes)
            hc, hh = fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * k * 8)
            qa, ca, ha = hq, hc, hh
        else:
            counts = np.full(m, -7, np.int32)
            hits = np.full(m * k, -7, np.int64)
            qa, ca, ha = qs.ctypes.data, counts.ctypes.data, hits.ctypes.data
        rc = fk.LIB.fkd_run_batch(tree.handle, C.c_void_p(qa), m, 3, C.byref(o), C.c_void_p(ca),
                                  C.c_void_p(ha), None)
        assert rc == 0, fk.LIB.fkd_last_error()
        got_c = np.ctypeslib.as_array(C.cast(C.c_void_p(ca), C.POINTER(C.c_int32)), shape=(m,)).copy()
        got_h = np.ctypeslib.as_array(C.cast(C.c_void_p(ha), C.POINTER(C.c_int64)), shape=(m * k,)).copy()
        if mode == "pinned":
            for p in (hq, hc, hh):
                fk.LIB.fkd_host_free(p)
        dq = torch.from_numpy(qs).cuda()
        c = torch.empty(m, dtype=torch.int32, device="cuda")
        h = torch.empty(m * k, dtype=torch.int64, device="cuda")
        fk.run_batch_device(tree, dq, c, h, fk.BatchOptions(kind=kind, k=k))
        assert np.array_equal(got_c, c.cpu().numpy())
        assert np.array_equal(got_h, h.cpu().numpy())


def test_knn8_rounds_large_batch(oracle):
    """kNN8 batches of >= 2^22 queries take the continuation rounds (capi.cu
    rounds_on); the same queries through the host pipeline's chunks (< 2^22
    each: one budgeted walk) and the oracle on a sample must give the same bytes."""
    import torch
    pts = fk.clustered_points(8, 1, 300_000, 3)
    m = (1 << 22) + 1000
    qs = fk.clustered_points(8, 2, m, 3)
    nodes = fk.build_level_order(pts)
    tree = fk.KdTree.from_level_order(nodes)
    for k in (8, 5):
        opt = fk.BatchOptions(kind=fk.QueryKind.knn, k=k)
        dq = torch.from_numpy(qs).cuda()
        c = torch.empty(m, dtype=torch.int32, device="cuda")
        h = torch.empty(m * k, dtype=torch.int64, device="cuda")
        fk.run_batch_device(tree, dq, c, h, opt)
        res = fk.run_batch(tree, qs, opt)
        assert np.array_equal(c.cpu().numpy(), res.counts)
        assert h.cpu().numpy().tobytes() == res.hits.tobytes()
        sample = np.arange(0, m, 211)
        rc, rh = oracle.run_batch(nodes, qs[sample], "knn", k, INF)[:2]
        assert np.array_equal(res.counts[sample], rc)
        assert res.hits.reshape(m, -1)[sample].tobytes() == rh.reshape(len(sample), -1).tobytes()


@pytest.mark.parametrize("budget,resume_min,resume_trips,rounds", [
    ("-1", "0", "0", "-"), ("0", "0", "0", "-"),    # defaults; no budget (one walk, STATS too)
    ("3", "0", "0", "0"), ("40", "1", "5", "0"),    # CTA pass; budgeted resume -> CTA pass
    ("2", "1", "-1", "0"), ("2", "0", "0", "1,2"),  # unbounded resume; rounds -> CTA pass
])
def test_slot_list_walk_high_dim(oracle, budget, resume_min, resume_trips, rounds, monkeypatch):
    """8-D walks with 16 slots keep their sorted list in the output slot
    (LaneWalk::kSlot): insertion, parking, resuming, the CTA pass's bound and
    the final count all go through the slot.  Runtime k below the bucket
    (9, 12), bounded radii (short lists), grid-snapped ties, duplicates."""
    monkeypatch.setenv("FKD_BUDGET", budget)
    monkeypatch.setenv("FKD_RESUME_TRIPS", resume_trips)
    monkeypatch.setenv("FKD_RESUME_MIN", resume_min if resume_min != "0" else str(1 << 40))
    if rounds != "-":
        monkeypatch.setenv("FKD_RROUNDS_KNN", rounds)
    rng = oracle.instance_rng(8088)
    for t in range(6):
        n = (0, 1, 17, 3000, 6000, 12000)[t]
        pts = rng.random_point_set(n, 8, 8 if t % 2 else 0, 0.2 if t % 3 == 0 else 0.0)
        nodes = oracle.build_tree(pts) if n else pts
        qs = np.stack([rng.random_query(8, pts) for _ in range(400)])
        for k in (9, 12, 16):
            for r in (INF, 0.6, 0.0):
                res, ref = _run_both(oracle, nodes.reshape(n, 8), qs, k, r, morton=bool(t % 2))
                _assert_same(res, ref, f"n={n} k={k} r={r} budget={budget}")
                tree = fk.KdTree.from_level_order(nodes.reshape(n, 8))
                fast = fk.run_batch(tree, qs, fk.BatchOptions(kind=fk.QueryKind.knn, k=k, max_radius=r))
                assert np.array_equal(fast.counts, ref[0]) and fast.hits.tobytes() == ref[1].tobytes(), \
                    f"budgeted n={n} k={k} r={r} budget={budget}"


@pytest.mark.parametrize("budget,rounds", [("-1", "-"), ("2", "0"), ("40", "1,2")])
def test_register_walks_9_to_16d(oracle, budget, rounds, monkeypatch):
    """9..16-D batches run the compile-time register walks (padded 12/16-float
    store with the split plane, box pruning, buckets 1/8/16/32/64, Morton keys
    over the first 8 axes, budget / rounds / CTA pass): every bucket, k below
    the bucket, bounded radii, ties and duplicates equal the reference; STATS
    and unordered batches (the heap kernel there) too; a non-finite last
    coordinate rejects the batch with its index."""
    import torch

    monkeypatch.setenv("FKD_BUDGET", budget)
    if rounds != "-":
        monkeypatch.setenv("FKD_RROUNDS_KNN", rounds)
        monkeypatch.setenv("FKD_RROUNDS_FCP", rounds)
    rng = oracle.instance_rng(9016)
    for dim in range(9, 17):
        n = (0, 1, 7, 2500, 9000)[dim % 5]
        pts = rng.random_point_set(n, dim, 8 if dim % 2 else 0, 0.2 if dim % 3 == 0 else 0.0)
        nodes = (oracle.build_tree(pts) if n else pts).reshape(n, dim)
        qs = np.stack([rng.random_query(dim, pts) for _ in range(300)])
        tree = fk.KdTree.from_level_order(nodes)
        for k in (0, 3, 8, 12, 16, 25, 32, 40, 64):
            for r in (INF, 0.5):
                what = f"dim={dim} n={n} k={k} r={r} budget={budget}"
                opt = fk.BatchOptions(kind=_kind(k), k=max(k, 1), max_radius=r)
                res = fk.run_batch(tree, qs, opt)
                c, h = oracle.run_batch(nodes, qs, "knn" if k else "fcp", max(k, 1), r)[:2]
                assert np.array_equal(res.counts, c) and res.hits.tobytes() == h.tobytes(), what
                cd = torch.empty(len(qs), dtype=torch.int32, device="cuda")
                hd = torch.empty(len(qs) * opt.stride, dtype=torch.int64, device="cuda")
                fk.run_batch_device(tree, torch.from_numpy(qs).cuda(), cd, hd, opt)
                assert np.array_equal(cd.cpu().numpy(), c) and hd.cpu().numpy().tobytes() == h.tobytes(), what
        if n:
            for k in (1, 8):
                res, ref = _run_both(oracle, nodes, qs, k, INF)  # STATS: the reference's counters
                _assert_same(res, ref, f"stats dim={dim} k={k}")
                uo = fk.run_batch(tree, qs, fk.BatchOptions(kind=fk.QueryKind.knn, k=k, unordered=True))
                assert np.array_equal(uo.counts, ref[0]) and uo.hits.tobytes() == ref[1].tobytes()
            bad = qs.copy()
            bad[77, dim - 1] = np.nan  # an axis the Morton key does not read
            with pytest.raises(fk.DataError, match="non-finite coordinate in point 77"):
                fk.run_batch(tree, bad, fk.BatchOptions(kind=fk.QueryKind.knn, k=8))


def test_register_walks_high_dim_against_reference(reference):
    """9..16-D against the unmodified reference library (oracle/_ref) itself,
    at a scale where the walks park and resume (N = 200k, 4000 queries from the
    reference's own generator): fcp, kNN 8 / 16 / 40, unbounded and bounded
    radii — counts, hit nodes and dist2 bits, and the reference's result hash."""
    for dim in (9, 11, 12, 16):
        pts = reference.stream_points(3, 1, 200_000, dim)
        nodes = reference.build_tree(pts)
        qs = reference.stream_points(3, 2, 4000 if dim < 16 else 1000, dim)  # the reference's 16-D walks are long
        tree = fk.KdTree.from_level_order(nodes)
        for kind, k, r in (("fcp", 1, INF), ("knn", 8, INF), ("knn", 16, 0.4), ("knn", 40, INF)):
            c, h, _, _ = reference.run_batch(nodes, qs, kind, k, r)
            got = fk.run_batch(tree, qs, fk.BatchOptions(kind=fk.QueryKind[kind], k=k, max_radius=r))
            what = f"dim={dim} {kind} k={k} r={r}"
            assert np.array_equal(got.counts, c) and got.hits.tobytes() == h.tobytes(), what
            assert got.result_hash() == reference.result_hash(c, h, k if kind == "knn" else 1), what


def test_rejected_batch_writes_no_output(oracle, monkeypatch):
    """A non-finite query rejects the batch before any slot is written, as
    the reference throws before its BatchResult exists (batch.cpp:79 before
    :82-86): device outputs (key pass / scan flag + walk-entry exit) and
    pageable host outputs (host check fused into the staging copy, or up front)
    keep their previous bytes; the reported id is the first bad query."""
    import ctypes as C
    import torch

    monkeypatch.setenv("FKD_CHUNK_DIV", "16")
    pts = fk.clustered_points(8, 1, 40_000, 3)
    nodes = oracle.build_tree(pts)
    qs = fk.clustered_points(8, 2, 600_001, 3)
    qs[512_345, 1] = np.nan
    qs[590_000, 0] = np.inf
    for devices in ([0], [0, 0]):
        tree = fk.KdTree.from_level_order(nodes, devices=devices)
        for kind, k in ((fk.QueryKind.fcp, 1), (fk.QueryKind.knn, 8)):
            opts = fk.BatchOptions(kind=kind, k=k)
            # pageable in, pageable out (fused host check)
            counts = np.full(len(qs), -7, np.int32)
            hits = np.full(len(qs) * k, -7, np.int64)
            o = opts.to_c()
            rc = fk.LIB.fkd_run_batch(tree.handle, qs.ctypes.data, len(qs), 3, C.byref(o), counts.ctypes.data,
                                      hits.ctypes.data, None)
            assert rc == 2 and "non-finite coordinate in point 512345" in fk.LIB.fkd_last_error().decode()
            assert (counts == -7).all() and (hits == -7).all()
            # pinned in, pageable out (up-front host check)
            hq = fk.LIB.fkd_host_alloc(qs.nbytes)
            C.memmove(hq, qs.ctypes.data, qs.nbytes)
            rc = fk.LIB.fkd_run_batch(tree.handle, C.c_void_p(hq), len(qs), 3, C.byref(o), counts.ctypes.data,
                                      hits.ctypes.data, None)
            fk.LIB.fkd_host_free(hq)
            assert rc == 2 and "point 512345" in fk.LIB.fkd_last_error().decode()
            assert (counts == -7).all() and (hits == -7).all()
        # device-resident batch (Morton key pass and the unsorted scan)
        dq = torch.from_numpy(qs).cuda()
        for morton in (True, False):
            c = torch.full((len(qs),), -7, dtype=torch.int32, device="cuda")
            h = torch.full((len(qs) * 8,), -7, dtype=torch.int64, device="cuda")
            with pytest.raises(fk.DataError, match="point 512345"):
                fk.run_batch_device(tree, dq, c, h, fk.BatchOptions(kind=fk.QueryKind.knn, k=8, morton=morton))
            assert (c == -7).all().item() and (h == -7).all().item()


def test_add_replicas_fanout(oracle):
    """fkd_tree_add_replicas (pipelined device-to-device chain) gives
    byte-identical replicas: a batch sharded over them equals the one-replica
    batch, through both host-buffer modes."""
    pts = oracle.random_points(21, 70_000, 4)
    nodes = oracle.build_tree(pts)
    qs = oracle.random_points(22, 90_001, 4)
    one = fk.KdTree.from_level_order(nodes, devices=[0])
    many = fk.KdTree.from_level_order(nodes, devices=[0])
    many.add_replicas([0, 0, 0])
    assert many.replica_devices() == [0, 0, 0, 0]
    for kind, k in ((fk.QueryKind.fcp, 1), (fk.QueryKind.knn, 16)):
        opt = fk.BatchOptions(kind=kind, k=k, collect_stats=True)
        a, b = fk.run_batch(one, qs, opt), fk.run_batch(many, qs, opt)
        assert a.hits.tobytes() == b.hits.tobytes() and np.array_equal(a.counts, b.counts)
        assert a.stats == b.stats


def test_run_batch_device_rejects_bad_tensors(oracle):
    import torch

    tree = fk.KdTree.from_level_order(oracle.build_tree(oracle.random_points(31, 1000, 3)))
    q = torch.rand(100, 3, device="cuda")
    c = torch.empty(100, dtype=torch.int32, device="cuda")
    h = torch.empty(100 * 8, dtype=torch.int64, device="cuda")
    knn8 = fk.BatchOptions(kind=fk.QueryKind.knn, k=8)
    with pytest.raises(fk.DataError, match="expected an"):
        fk.run_batch_device(tree, q.reshape(-1), c, h, knn8)
    with pytest.raises(fk.DataError, match="contiguous"):
        fk.run_batch_device(tree, torch.rand(3, 100, device="cuda").t(), c, h, knn8)
    with pytest.raises(fk.DataError, match="dtype"):
        fk.run_batch_device(tree, q.double(), c, h, knn8)
    with pytest.raises(fk.DataError, match="hits: holds"):
        fk.run_batch_device(tree, q, c, h[:799], knn8)
    with pytest.raises(fk.DataError, match="counts"):
        fk.run_batch_device(tree, q, c.long(), h, knn8)
    with pytest.raises(fk.DataError, match="CUDA"):
        fk.run_batch_device(tree, q.cpu(), c, h, knn8)
    fk.run_batch_device(tree, q, c, h, knn8)  # the well-formed call goes through


def test_run_batches_device_concurrent_exact(oracle):
    """fkd_run_batches_device: several batches in one submission (forked
    streams, priorities, one shared Morton order for batches over the same
    query array) give exactly what separate run_batch_device calls give;
    statuses are per batch."""
    import torch

    pts = fk.clustered_points(41, 1, 200_000, 3)
    tree = fk.KdTree.from_level_order(oracle.build_tree(pts))
    qa = torch.from_numpy(fk.clustered_points(41, 2, 300_001, 3)).cuda()
    qb = torch.from_numpy(fk.random_points(41, 3, 120_000, 3)).cuda()
    specs = [(qa, fk.BatchOptions(kind=fk.QueryKind.fcp)),
             (qa, fk.BatchOptions(kind=fk.QueryKind.knn, k=8)),
             (qa, fk.BatchOptions(kind=fk.QueryKind.knn, k=20, max_radius=0.05)),
             (qa, fk.BatchOptions(kind=fk.QueryKind.knn, k=4, morton=False)),
             (qb, fk.BatchOptions(kind=fk.QueryKind.knn, k=8, collect_stats=True))]
    outs = [(torch.full((q.shape[0],), -7, dtype=torch.int32, device="cuda"),
             torch.full((q.shape[0] * o.stride,), -7, dtype=torch.int64, device="cuda")) for q, o in specs]
    res = fk.run_batches_device(tree, [(q, c, h, o) for (q, o), (c, h) in zip(specs, outs)], timings=True)
    for (q, o), (c, h), (st, tm) in zip(specs, outs, res):
        c2 = torch.empty_like(c)
        h2 = torch.empty_like(h)
        st2, _ = fk.run_batch_device(tree, q, c2, h2, o)
        assert torch.equal(c, c2) and torch.equal(h, h2), o
        assert tm["walk_launches"] >= 1
        if o.collect_stats:
            assert st == st2 and st.nodes_processed > 0
    # a rejected batch leaves its own slots (and only its own) untouched
    bad = qa.clone()
    bad[1234, 2] = float("nan")
    c_ok, h_ok = torch.empty(qb.shape[0], dtype=torch.int32, device="cuda"), \
        torch.empty(qb.shape[0] * 8, dtype=torch.int64, device="cuda")
    c_bad = torch.full((bad.shape[0],), -7, dtype=torch.int32, device="cuda")
    h_bad = torch.full((bad.shape[0] * 8,), -7, dtype=torch.int64, device="cuda")
    c_bad2 = torch.full((bad.shape[0],), -7, dtype=torch.int32, device="cuda")
    with pytest.raises(fk.DataError, match="point 1234"):
        fk.run_batches_device(tree, [(bad, c_bad, h_bad, fk.BatchOptions(kind=fk.QueryKind.knn, k=8)),
                                     (bad, c_bad2, torch.empty_like(c_bad2).long(), fk.BatchOptions()),
                                     (qb, c_ok, h_ok, fk.BatchOptions(kind=fk.QueryKind.knn, k=8))])
    assert (c_bad == -7).all().item() and (h_bad == -7).all().item() and (c_bad2 == -7).all().item()
    c_ref, h_ref = torch.empty_like(c_ok), torch.empty_like(h_ok)
    fk.run_batch_device(tree, qb, c_ref, h_ref, fk.BatchOptions(kind=fk.QueryKind.knn, k=8))
    assert torch.equal(c_ok, c_ref) and torch.equal(h_ok, h_ref)


@pytest.mark.parametrize("knobs", ["", "FKD_FULL_STAGING=0", "FKD_STREAMS=2;FKD_CHUNK_DIV=5",
                                   "FKD_FULL_STAGING=0;FKD_STREAMS=3;FKD_BUDGET=40;FKD_RESUME_MIN=50",
                                   "FKD_PAGEABLE_STAGING=0", "FKD_HOST_COUNTS=0"])
def test_run_batches_host_groups_exact(oracle, knobs, monkeypatch):
    """fkd_run_batches: batches over one query array run as one pipeline
    (shared upload, check and Morton order per chunk; full and ring device
    staging; pageable and pinned buffers); each equals its own fkd_run_batch."""
    import ctypes as C

    for kv in filter(None, knobs.split(";")):
        k_, v_ = kv.split("=")
        monkeypatch.setenv(k_, v_)
    pts = fk.clustered_points(51, 1, 80_000, 3)
    tree = fk.KdTree.from_level_order(oracle.build_tree(pts), devices=[0, 0])
    qa = fk.clustered_points(51, 2, 700_001, 3)
    qb = fk.random_points(51, 3, 50_000, 3)
    specs = [(qa, fk.BatchOptions(kind=fk.QueryKind.fcp, collect_stats=True)),
             (qa, fk.BatchOptions(kind=fk.QueryKind.knn, k=8, collect_stats=True)),
             (qb, fk.BatchOptions(kind=fk.QueryKind.knn, k=4)),
             (qa, fk.BatchOptions(kind=fk.QueryKind.knn, k=20, max_radius=0.02, morton=False))]
    got = fk.run_batches(tree, specs)
    for (q, o), r in zip(specs, got):
        ref = fk.run_batch(tree, q, o)
        assert np.array_equal(r.counts, ref.counts) and r.hits.tobytes() == ref.hits.tobytes(), o
        assert r.stats == ref.stats
    # pinned caller buffers through the C ABI
    m = len(qa)
    hq = fk.LIB.fkd_host_alloc(qa.nbytes)
    C.memmove(hq, qa.ctypes.data, qa.nbytes)
    arr = (fk._lib.fkd_host_batch * 2)()
    bufs = []
    for i, o in enumerate((fk.BatchOptions(kind=fk.QueryKind.knn, k=8), fk.BatchOptions())):
        hc, hh = fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * o.stride * 8)
        bufs.append((hc, hh, o))
        arr[i].queries, arr[i].m, arr[i].dim, arr[i].opt = hq, m, 3, o.to_c()
        arr[i].counts, arr[i].hits, arr[i].stats = hc, hh, None
    assert fk.LIB.fkd_run_batches(tree.handle, arr, 2) == 0, fk.LIB.fkd_last_error()
    for hc, hh, o in bufs:
        ref = fk.run_batch(tree, qa, o)
        gc = np.ctypeslib.as_array(C.cast(C.c_void_p(hc), C.POINTER(C.c_int32)), shape=(m,))
        gh = np.ctypeslib.as_array(C.cast(C.c_void_p(hh), C.POINTER(C.c_int64)), shape=(m * o.stride,))
        assert np.array_equal(gc, ref.counts) and gh.tobytes() == ref.hits.tobytes()
        fk.LIB.fkd_host_free(hc)
        fk.LIB.fkd_host_free(hh)
    fk.LIB.fkd_host_free(hq)


@pytest.mark.parametrize("knobs", ["", "FKD_FULL_STAGING=0;FKD_STREAMS=3", "FKD_PAGEABLE_STAGING=0"])
def test_host_written_counts_unbounded_radius(oracle, knobs, monkeypatch):
    """An unbounded-radius batch through the host pipeline: every count is
    min(k, n), written on the host while only the hits are copied (the device
    checks the walked counts); counts and hits equal the reference's with k
    below and above n, for an infinite radius and one whose square overflows."""
    import ctypes as C

    for kv in filter(None, knobs.split(";")):
        k_, v_ = kv.split("=")
        monkeypatch.setenv(k_, v_)
    q = fk.random_points(61, 2, 300_001, 3)
    for n in (5, 3000):
        nodes = oracle.build_tree(fk.random_points(61, 1, n, 3))
        tree = fk.KdTree.from_level_order(nodes)
        for kind, k, r in (("fcp", 1, INF), ("knn", 8, INF), ("knn", 3, 1e30), ("knn", 8, 0.05)):
            o = fk.BatchOptions(kind=fk.QueryKind[kind], k=k, max_radius=r)
            c, h, _, _ = oracle.run_batch(nodes, q, kind, k, r)
            got = fk.run_batch(tree, q, o)  # pageable (NumPy) buffers
            assert np.array_equal(got.counts, c) and got.hits.tobytes() == h.tobytes(), (n, kind, k, r)
            m = len(q)  # pinned caller buffers
            hq, hc, hh = fk.LIB.fkd_host_alloc(q.nbytes), fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * k * 8)
            C.memmove(hq, q.ctypes.data, q.nbytes)
            co = o.to_c()
            assert fk.LIB.fkd_run_batch(tree.handle, hq, m, 3, C.byref(co), hc, hh, None) == 0
            gc = np.ctypeslib.as_array(C.cast(C.c_void_p(hc), C.POINTER(C.c_int32)), shape=(m,))
            gh = np.ctypeslib.as_array(C.cast(C.c_void_p(hh), C.POINTER(C.c_int64)), shape=(m * k,))
            assert np.array_equal(gc, c) and gh.tobytes() == h.tobytes(), (n, kind, k, r)
            for p in (hq, hc, hh):
                fk.LIB.fkd_host_free(p)


def test_submit_batches_jobs_in_flight(oracle):
    """fkd_submit_batches / fkd_wait: several jobs in flight on one tree
    (their pipelines overlap on the device) each return exactly what
    run_batches does; a job with a non-finite query fails at wait with the
    reference's message, the others are unaffected; a job waits only once."""
    pts = fk.clustered_points(71, 1, 60_000, 3)
    tree = fk.KdTree.from_level_order(oracle.build_tree(pts))
    qs = [fk.clustered_points(71, 2 + i, 400_000 + 1000 * i, 3) for i in range(3)]
    bad = qs[1].copy()
    bad[1234, 2] = np.inf
    specs = [[(q, fk.BatchOptions(kind=fk.QueryKind.knn, k=8)), (q, fk.BatchOptions())] for q in qs]
    jobs = [fk.submit_batches(tree, sp) for sp in specs]
    bad_job = fk.submit_batches(tree, [(bad, fk.BatchOptions())])
    more = fk.submit_batches(tree, [(qs[2], fk.BatchOptions(kind=fk.QueryKind.knn, k=20, max_radius=0.03))])
    with pytest.raises(fk.DataError, match="non-finite coordinate in point 1234"):
        bad_job.wait()
    for sp, job in zip(specs, jobs):
        got = job.wait()
        ref = fk.run_batches(tree, sp)
        for g, r in zip(got, ref):
            assert np.array_equal(g.counts, r.counts) and g.hits.tobytes() == r.hits.tobytes()
    (g,) = more.wait()
    c, h, _, _ = oracle.run_batch(oracle.build_tree(pts), qs[2], "knn", 20, 0.03)
    assert np.array_equal(g.counts, c) and g.hits.tobytes() == h.tobytes()
    with pytest.raises(fk.InvalidArgument):
        more.wait()


def test_run_batches_rejected_group_and_many_batches(oracle):
    """A non-finite query rejects its whole group (same queries) with the
    first bad id and leaves pageable outputs untouched; another group's
    batch still completes; more batches than one pipeline holds are split."""
    import ctypes as C

    tree = fk.KdTree.from_level_order(oracle.build_tree(oracle.random_points(61, 30_000, 3)))
    bad = oracle.random_points(62, 400_000, 3)
    bad[333_333, 0] = np.inf
    good = oracle.random_points(63, 20_000, 3)
    arr = (fk._lib.fkd_host_batch * 3)()
    outs = []
    for i, (q, o) in enumerate(((bad, fk.BatchOptions(kind=fk.QueryKind.knn, k=8)), (bad, fk.BatchOptions()),
                                (good, fk.BatchOptions(kind=fk.QueryKind.knn, k=2)))):
        c = np.full(len(q), -7, np.int32)
        h = np.full(len(q) * o.stride, -7, np.int64)
        outs.append((c, h, q, o))
        arr[i].queries, arr[i].m, arr[i].dim, arr[i].opt = q.ctypes.data, len(q), 3, o.to_c()
        arr[i].counts, arr[i].hits, arr[i].stats = c.ctypes.data, h.ctypes.data, None
    assert fk.LIB.fkd_run_batches(tree.handle, arr, 3) == 2
    assert "point 333333" in fk.LIB.fkd_last_error().decode()
    assert [arr[i].status for i in range(3)] == [2, 2, 0]
    for c, h, q, o in outs[:2]:
        assert (c == -7).all() and (h == -7).all()
    c, h, q, o = outs[2]
    ref = fk.run_batch(tree, q, o)
    assert np.array_equal(c, ref.counts) and h.tobytes() == ref.hits.tobytes()
    many = [(good, fk.BatchOptions(kind=fk.QueryKind.knn, k=1 + i % 5)) for i in range(19)]
    for (q, o), r in zip(many, fk.run_batches(tree, many)):
        ref = fk.run_batch(tree, q, o)
        assert np.array_equal(r.counts, ref.counts) and r.hits.tobytes() == ref.hits.tobytes()


def test_bench_matrix_csv_matches_reference(reference):
    """bench_matrix.write_bench_csv (bench.cpp:119-133 schema) on the B200
    path against the reference's own run_bench_matrix + write_bench_csv on
    the same seeds: identical rows except engine/threads and the timings."""
    import io

    from paper_2210_12859_b200 import bench_matrix as bm

    for kind, ks, rs in (("fcp", (8,), (INF,)), ("knn", (1, 8, 20), (INF, 0.05))):
        base = bm.BenchConfig(n_queries=20_000, k_dim=3, kind=fk.QueryKind[kind], reps=2)
        rows = bm.run_bench_matrix(base, [1000, 7000], ks, rs)
        buf = io.StringIO()
        bm.write_bench_csv(buf, rows)
        ours = [line.split(",") for line in buf.getvalue().strip().splitlines()]
        ref = [line.split(",") for line in
               reference.bench_matrix_csv(20_000, 3, kind, 2, [1000, 7000], ks, rs).strip().splitlines()]
        assert ours[0] == ref[0] and len(ours) == len(ref)
        keep = [0, 1, 2, 3, 6, 7, 10, 11, 12]  # n query k max_r reps total nodes/q steps/q hash
        for a, b in zip(ours[1:], ref[1:]):
            assert [a[i] for i in keep] == [b[i] for i in keep], (a, b)
            assert a[4] == "b200" and b[4] == "stackfree"


def test_morton_keys_and_exchange_single_rank(oracle):
    """fkd_morton_keys = the batch ordering's key over the tree's box (24
    bits); the Morton-range exchange at world size 1 is the identity and the
    walk over its local queries returns the unpartitioned answer."""
    import torch

    from paper_2210_12859_b200.shard import MortonExchange

    nodes = oracle.build_tree(oracle.random_points(71, 50_000, 3))
    tree = fk.KdTree.from_level_order(nodes)
    qs = oracle.random_points(72, 30_000, 3) * np.float32(1.2) - np.float32(0.1)
    q = torch.from_numpy(qs).cuda()
    keys, bits = fk.morton_keys(tree, q)
    assert bits == 24
    lo, hi = nodes.min(0), nodes.max(0)
    top = np.float32((1 << 8) - 1)
    scale = (np.float64(top) / (hi.astype(np.float64) - lo.astype(np.float64))).astype(np.float32)
    t = np.minimum(np.maximum((qs - lo) * scale, np.float32(0)), top).astype(np.int64)
    ref = np.zeros(len(qs), np.int64)
    for b in range(7, -1, -1):
        for d in range(3):
            ref = (ref << 1) | ((t[:, d] >> b) & 1)
    assert np.array_equal(keys.cpu().numpy(), ref)
    ex = MortonExchange(q, keys, bits, 1)
    c = torch.empty(len(qs), dtype=torch.int32, device="cuda")
    h = torch.empty(len(qs) * 8, dtype=torch.int64, device="cuda")
    fk.run_batch_device(tree, ex.local_queries, c, h, fk.BatchOptions(kind=fk.QueryKind.knn, k=8))
    rc, rh = ex.return_results(c, h, 8)
    ref_c, ref_h, _, _ = oracle.run_batch(nodes, qs, "knn", 8)
    assert np.array_equal(rc.cpu().numpy(), ref_c) and rh.cpu().numpy().tobytes() == ref_h.tobytes()
    bad = q.clone()
    bad[17, 1] = float("nan")
    with pytest.raises(fk.DataError, match="point 17"):
        fk.morton_keys(tree, bad)


def test_concurrent_grouped_and_device_submissions(oracle):
    """Several host threads at once through the grouped host pipeline
    (pageable buffers: staging rings + drain threads) and the concurrent
    device submission, sharing one tree with two replicas: every result equals
    the single-caller answer (pooled workspaces, staging pool, copy pool and
    per-device threads under contention)."""
    import threading

    import torch

    nodes = oracle.build_tree(oracle.random_points(81, 60_000, 3))
    tree = fk.KdTree.from_level_order(nodes, devices=[0, 0])
    work = []
    for t in range(6):
        qs = fk.clustered_points(82 + t, 2, 300_000 + 7919 * t, 3)
        specs = [(qs, fk.BatchOptions(kind=fk.QueryKind.knn, k=8)), (qs, fk.BatchOptions()),
                 (qs, fk.BatchOptions(kind=fk.QueryKind.knn, k=3, max_radius=0.05))]
        work.append((qs, specs, [fk.run_batch(tree, q, o) for q, o in specs]))
    errors = []

    def worker(i):
        qs, specs, refs = work[i]
        try:
            for rep in range(3):
                if (i + rep) % 2 == 0:
                    got = fk.run_batches(tree, specs)
                    for g, r in zip(got, refs):
                        assert np.array_equal(g.counts, r.counts) and g.hits.tobytes() == r.hits.tobytes()
                else:
                    dq = torch.from_numpy(qs).cuda()
                    outs = [(torch.empty(len(qs), dtype=torch.int32, device="cuda"),
                             torch.empty(len(qs) * o.stride, dtype=torch.int64, device="cuda")) for _, o in specs]
                    stream = torch.cuda.Stream()
                    fk.run_batches_device(tree, [(dq, c, h, o) for (c, h), (_, o) in zip(outs, specs)], stream=stream)
                    for (c, h), r in zip(outs, refs):
                        assert np.array_equal(c.cpu().numpy(), r.counts)
                        assert h.cpu().numpy().tobytes() == r.hits.tobytes()
        except Exception as e:  # noqa: BLE001
            errors.append((i, repr(e)))

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(6)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
