"""Generates tests/golden/scale.json: the reference's own answers at the
BASELINE.json scales (N = 10M / 100M trees), computed by the UNMODIFIED
reference library (oracle/_ref/libflatkd_ref.so, built from /root/reference
by oracle/Makefile).  Run here, where /root/reference exists (~10 min on 8
cores; the 100M single-threaded reference build alone takes ~155 s):

    python tests/golden/make_golden_scale.py

Each entry: the workload (seed 1; data stream 1, query stream 2 — exactly
flatkd::run_bench_matrix's inputs, bench.cpp:64-90), the reference's
BatchResult::result_hash over the whole batch (batch.cpp:30-48), its
QueryStats totals, and a SHA-256 of the reference builder's level-order
array (tree.cpp:80-89) so the GPU builder's output is pinned at this scale
too.  SURVEY.md §8(c) recorded the uniform hashes at survey time; this
script recomputes them (and asserts they agree) and adds the clustered C3
workload (full M = 10M, fcp + kNN8), which the survey has no hash for.

tests/test_gpu_scale.py (-m gpu) checks the B200 path against this file;
nothing on the GPU box reads /root/reference.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import Reference  # noqa: E402

INF = float("inf")
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scale.json")

# name: (generator, dim, N, M, kind, k, max_radius, SURVEY §8(c) hash or None)
CASES = [
    ("fcp_3d_n10m_m1m", "uniform", 3, 10_000_000, 1_000_000, "fcp", 1, INF, "0cca445a11013618"),
    ("knn8_3d_n10m_m1m", "uniform", 3, 10_000_000, 1_000_000, "knn", 8, INF, "5a71a6a204bbe790"),
    ("fcp_4d_n10m_m1m", "uniform", 4, 10_000_000, 1_000_000, "fcp", 1, INF, "11d43fd7c68c62e6"),
    ("knn8_4d_n10m_m1m_r0.01", "uniform", 4, 10_000_000, 1_000_000, "knn", 8, 0.01, "7c5c62b9b41500e3"),
    ("knn16_2d_n10m_m200k", "uniform", 2, 10_000_000, 200_000, "knn", 16, INF, "6a39ab1bb32b6cb2"),
    ("knn16_4d_n10m_m200k", "uniform", 4, 10_000_000, 200_000, "knn", 16, INF, "563944befa0aff8b"),
    ("knn16_8d_n10m_m200k", "uniform", 8, 10_000_000, 200_000, "knn", 16, INF, "10a6147e5f8a5a07"),
    ("fcp_3d_n100m_m200k", "uniform", 3, 100_000_000, 200_000, "fcp", 1, INF, "1fc44d5457a0fee4"),
    ("c3_fcp_clustered_n10m_m10m", "clustered", 3, 10_000_000, 10_000_000, "fcp", 1, INF, None),
    ("c3_knn8_clustered_n10m_m10m", "clustered", 3, 10_000_000, 10_000_000, "knn", 8, INF, None),
]


def points(r, gen, stream, count, dim):
    if gen == "clustered":
        return r.clustered_points(1, stream, count, dim, 64, 0.02)
    return r.stream_points(1, stream, count, dim)


def main():
    r = Reference()
    only = set(sys.argv[1:])
    out = {"source": "reference flatkd (oracle/_ref, -O3 -ffp-contract=off), run_batch over the whole batch",
           "threads": r.hardware_threads(), "cases": {}}
    if os.path.exists(OUT):
        out["cases"] = json.load(open(OUT)).get("cases", {})
    trees = {}
    for name, gen, dim, n, m, kind, k, rad, survey in CASES:
        if only and name not in only:
            continue
        key = (gen, dim, n)
        t0 = time.time()
        if key not in trees:
            trees.clear()  # one big tree at a time
            nodes = r.build_tree(points(r, gen, 1, n, dim))
            trees[key] = (nodes, hashlib.sha256(nodes.tobytes()).hexdigest())
        nodes, tree_sha = trees[key]
        qs = points(r, gen, 2, m, dim)
        c, h, st, secs = r.run_batch(nodes, qs, kind, k, rad, collect_stats=True)
        got = f"{r.result_hash(c, h, k if kind == 'knn' else 1):016x}"
        if survey is not None and got != survey:
            raise SystemExit(f"{name}: reference hash {got} != SURVEY §8(c) {survey}")
        out["cases"][name] = {"generator": gen, "seed": 1, "data_stream": 1, "query_stream": 2, "dim": dim,
                              "n": n, "m": m, "kind": kind, "k": k, "max_radius": rad, "hash": got,
                              "survey_hash": survey, "stats": [int(x) for x in st],
                              "tree_sha256": tree_sha, "reference_seconds_with_stats": round(secs, 3)}
        print(f"{name}: {got} stats={list(st)} ({time.time() - t0:.1f} s)", flush=True)
        json.dump(out, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()
