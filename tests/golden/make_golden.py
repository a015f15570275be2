"""Generates tests/golden/golden.json from the UNMODIFIED reference library
(oracle/_ref/libflatkd_ref.so, compiled from /root/reference/proj by
oracle/Makefile).  Run here (where /root/reference exists):

    python tests/golden/make_golden.py

The fixtures pin the oracle restatement (tests/test_oracle.py, CPU) and the
GPU path (tests/test_gpu_parity.py) without needing the reference at run time.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import Reference  # noqa: E402

INF = float("inf")


def main():
    r = Reference()
    g = {"source": "reference flatkd built by oracle/Makefile (-O3 -ffp-contract=off)"}
    # Fig. 1 (selfcheck.cpp:268-274)
    pts = np.array([[2, 3], [5, 4], [9, 6], [4, 7], [8, 1], [7, 2]], np.float32)
    tree = r.build_tree(pts)
    fig = {"points": pts.tolist(), "level_order": tree.tolist(), "queries": []}
    for q in ([9, 2], [2, 3], [5, 5], [0, 0], [7.5, 2.5]):
        for kind, k, rad in (("fcp", 1, INF), ("fcp", 1, 1.0), ("knn", 2, INF), ("knn", 3, INF), ("knn", 6, 3.0)):
            hits, st, tr = r.query(tree, q, kind, k, rad, trace_cap=64)
            fig["queries"].append({"q": q, "kind": kind, "k": k, "max_radius": rad,
                                   "hits": [[int(h["node"]), float(h["dist2"])] for h in hits],
                                   "stats": [int(x) for x in st], "trace": [int(x) for x in tr]})
    c, h, _, _ = r.run_batch(tree, np.array([[9, 2], [2, 3]], np.float32), "knn", 3)
    fig["batch_knn3_text"] = r.write_results(c, h, 3)
    g["figure1"] = fig
    # rng streams (rng.hpp:26-53)
    g["random_points_seed1_stream1_first12"] = r.random_points(r.derive_stream_seed(1, 1), 4, 3).reshape(-1).tolist()
    g["derive_stream_seed"] = {str(s): str(r.derive_stream_seed(1, s)) for s in (1, 2, 3)}
    # small batches over all query configurations, hashes + stats
    cases = []
    for dim in (1, 2, 3, 4, 5, 8):
        pts = r.random_points(r.derive_stream_seed(11 + dim, 1), 3000, dim)
        qs = r.random_points(r.derive_stream_seed(11 + dim, 2), 500, dim) * np.float32(1.5) - np.float32(0.25)
        nodes = r.build_tree(pts)
        for kind, k in (("fcp", 1), ("knn", 1), ("knn", 4), ("knn", 8), ("knn", 20), ("knn", 50)):
            for rad in (INF, 0.25, 0.01, 0.0):
                c, h, st, _ = r.run_batch(nodes, qs, kind, k, rad, collect_stats=True)
                _, _, st_rec, _ = r.run_batch(nodes, qs, kind, k, rad, engine=1, collect_stats=True)
                cases.append({"dim": dim, "seed": 11 + dim, "n": 3000, "m": 500, "kind": kind, "k": k,
                              "max_radius": rad, "hash": f"{r.result_hash(c, h, k if kind == 'knn' else 1):016x}",
                              "stats": [int(x) for x in st], "stats_recursive": [int(x) for x in st_rec]})
    g["batches"] = cases
    # tie-heavy instancegen instances (instancegen.cpp:12-48)
    inst = []
    rng = r.instance_rng(2024)
    for t in range(30):
        n = 1 + (rng.next_u64() % 700)
        dim = 1 + (rng.next_u64() % 4)
        grid = 8 if t % 3 == 0 else (16 if t % 3 == 1 else 0)
        dup = 0.2 if t % 2 == 0 else 0.0
        pts = rng.random_point_set(int(n), int(dim), grid, dup)
        qs = np.stack([rng.random_query(int(dim), pts) for _ in range(40)])
        nodes = r.build_tree(pts)
        entry = {"n": int(n), "dim": int(dim), "grid": grid, "dup": dup,
                 "points": pts.tolist(), "queries": qs.tolist(), "results": []}
        for kind, k, rad in (("fcp", 1, INF), ("fcp", 1, 0.25), ("knn", 4, INF), ("knn", 8, 0.25), ("knn", 20, 0.0)):
            c, h, st, _ = r.run_batch(nodes, qs, kind, k, rad, collect_stats=True)
            entry["results"].append({"kind": kind, "k": k, "max_radius": rad, "counts": c.tolist(),
                                     "hits": [[int(x["node"]), float(x["dist2"])] for x in h],
                                     "stats": [int(x) for x in st]})
        entry["level_order"] = nodes.tolist()
        inst.append(entry)
    g["instances"] = inst
    # survey-time large hashes, recomputed here
    data = r.random_points(r.derive_stream_seed(1, 1), 1_000_000, 3)
    qs = r.random_points(r.derive_stream_seed(1, 2), 1_000_000, 3)
    nodes = r.build_tree(data)
    big = {}
    for name, kind, k, rad in (("c1_fcp", "fcp", 1, INF), ("c2_knn8_inf", "knn", 8, INF), ("c2_knn8_r001", "knn", 8, 0.01)):
        c, h, st, _ = r.run_batch(nodes, qs, kind, k, rad, collect_stats=True)
        big[name] = {"hash": f"{r.result_hash(c, h, k if kind == 'knn' else 1):016x}", "stats": [int(x) for x in st]}
    g["c1_c2"] = big
    # reference suites (selfcheck.cpp): the reference's own property tests pass
    g["suites"] = {"structure": r.structure_suite(1024, 100000)[:2],
                   "trace": r.trace_suite(1, 2000, 1024, 20)[:2],
                   "oracle": r.oracle_suite(1, 300, 2000, 20)[:2]}
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(out, "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
