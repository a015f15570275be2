"""Table-1 style benchmark grid on the B200 path, in the reference's schema.

Mirrors the reference's bench API (``/root/reference/proj/include/flatkd/
bench.hpp:13-52``, ``src/bench.cpp:35-133``) over :func:`run_batch`:

* :class:`BenchConfig` / :class:`BenchRow`  — bench.hpp:13-33, same fields;
* :func:`run_bench` / :func:`run_bench_matrix` — bench.cpp:56-90: data from
  ``derive_stream_seed(seed, 1)``, queries from ``(seed, 2)``, the tree built
  once per n (untimed, bench.hpp:35-37), ``reps`` timed full passes of the
  query batch, the result hash of the first pass, node counters from one
  extra untimed counted pass (run_cell, bench.cpp:23-53);
* :func:`print_bench_table` / :func:`write_bench_csv` — bench.cpp:102-133,
  the same columns and number formats.  ``engine`` reads ``b200`` and
  ``threads`` the number of GPUs holding the tree, so a B200 CSV diffs
  row-for-row against the reference's (``oracle.Reference.bench_matrix_csv``)
  on every column but the timings.

Each timed pass is one drop-in ``run_batch`` call: host buffers in and out,
H2D, Morton order, walk and D2H inside the clock, as the reference times
its whole ``run_batch`` (bench.cpp:36-39).

CLI: ``python -m paper_2210_12859_b200.bench_matrix --dim 3 --m 1000000
--n 1000000 --kind knn --k 1,4,8,16 --maxr inf,0.01 --reps 3 --csv out.csv``
"""
from __future__ import annotations

import argparse
import io
import math
import sys
import time
from dataclasses import dataclass, field, replace
from typing import List, Sequence

import numpy as np

from . import BatchOptions, Engine, KdTree, QueryKind, build_tree, random_points, run_batch

INF = float("inf")


@dataclass
class BenchConfig:
    """flatkd::BenchConfig (bench.hpp:13-24)."""

    n_data: int = 1000
    n_queries: int = 10_000_000
    k_dim: int = 4
    kind: QueryKind = QueryKind.fcp
    k: int = 8
    max_radius: float = INF
    seed: int = 1
    reps: int = 100
    threads: int = 0          # GPUs in the reference's "threads" column (0: the tree's replica count)
    engine: Engine = Engine.stack_free
    devices: Sequence[int] = field(default_factory=lambda: [0])


@dataclass
class BenchRow:
    """flatkd::BenchRow (bench.hpp:26-33)."""

    config: BenchConfig
    total_queries: int = 0
    wall_time: float = 0.0
    queries_per_second: float = 0.0
    nodes_processed_per_query: float = 0.0
    steps_per_query: float = 0.0
    result_hash: int = 0


def _validate(cfg: BenchConfig) -> None:  # bench.cpp:14-21, same messages
    from . import DataError

    if cfg.n_data < 0:
        raise DataError("bench: n must be >= 0")
    if cfg.n_queries < 1:
        raise DataError("bench: m must be >= 1")
    if cfg.k_dim < 1:
        raise DataError("bench: k-dim must be >= 1")
    if cfg.reps < 1:
        raise DataError("bench: reps must be >= 1")
    if cfg.kind == QueryKind.knn and cfg.k < 1:
        raise DataError("bench: k must be >= 1")
    if not cfg.max_radius > 0.0:
        raise DataError("bench: max radius must be > 0 or inf")


def _run_cell(tree: KdTree, queries, cfg: BenchConfig) -> BenchRow:
    """run_cell (bench.cpp:23-53)."""
    opts = BatchOptions(kind=cfg.kind, k=cfg.k, max_radius=cfg.max_radius, engine=cfg.engine)
    # one untimed pass first: the library grows its device workspaces and
    # pinned staging lazily on first use, a one-time cost per process that
    # a reference run_batch has no counterpart of
    run_batch(tree, queries, opts)
    wall, h = 0.0, 0
    for rep in range(cfg.reps):
        t0 = time.perf_counter()
        res = run_batch(tree, queries, opts)
        wall += time.perf_counter() - t0
        if rep == 0:
            h = res.result_hash()
    counted = run_batch(tree, queries, replace(opts, collect_stats=True))
    row = BenchRow(config=cfg)
    row.total_queries = cfg.n_queries * cfg.reps
    row.wall_time = wall
    row.queries_per_second = row.total_queries / wall if wall > 0 else 0.0
    m = float(cfg.n_queries)
    row.nodes_processed_per_query = counted.stats.nodes_processed / m
    row.steps_per_query = counted.stats.steps / m
    row.result_hash = h
    return row


def run_bench(cfg: BenchConfig) -> BenchRow:
    """run_bench (bench.cpp:56-63)."""
    _validate(cfg)
    tree = build_tree(random_points(cfg.seed, 1, cfg.n_data, cfg.k_dim), devices=list(cfg.devices))
    queries = random_points(cfg.seed, 2, cfg.n_queries, cfg.k_dim)
    return _run_cell(tree, queries, cfg)


def run_bench_matrix(base: BenchConfig, n_list: Sequence[int], k_list: Sequence[int] = (8,),
                     maxr_list: Sequence[float] = (INF,)) -> List[BenchRow]:
    """run_bench_matrix (bench.cpp:64-90): one row per (n, cell); fcp
    collapses the cell list to one column, knn crosses k_list x maxr_list."""
    rows = []
    queries = random_points(base.seed, 2, base.n_queries, base.k_dim)
    for n in n_list:
        cfg = replace(base, n_data=int(n))
        _validate(cfg)
        tree = build_tree(random_points(cfg.seed, 1, cfg.n_data, cfg.k_dim), devices=list(cfg.devices))
        if cfg.kind == QueryKind.fcp:
            rows.append(_run_cell(tree, queries, cfg))
            continue
        for k in k_list:
            for maxr in maxr_list:
                c = replace(cfg, k=int(k), max_radius=float(maxr))
                _validate(c)
                rows.append(_run_cell(tree, queries, c))
    return rows


def _format_float(v: float) -> str:  # io::format_float (io.cpp:163-167): "%.9g" of the float32 value
    return "%.9g" % float(np.float32(v))


def _maxr_text(v: float) -> str:  # bench.cpp:95-97
    return "inf" if math.isinf(v) else _format_float(v)


def _threads(c: BenchConfig) -> int:
    return c.threads if c.threads > 0 else len(c.devices)


def _kind(c: BenchConfig) -> str:
    return "fcp" if c.kind == QueryKind.fcp else "knn"


def print_bench_table(out, rows: Sequence[BenchRow]) -> None:
    """print_bench_table (bench.cpp:102-117)."""
    out.write("%10s %5s %4s %8s %10s %4s %5s %14s %12s %16s\n" % (
        "n", "query", "k", "maxR", "engine", "thr", "reps", "q/s", "nodes/query", "result-hash"))
    for r in rows:
        c = r.config
        out.write("%10d %5s %4d %8s %10s %4d %5d %14.0f %12.1f %016x\n" % (
            c.n_data, _kind(c), c.k if c.kind == QueryKind.knn else 1, _maxr_text(c.max_radius), "b200",
            _threads(c), c.reps, r.queries_per_second, r.nodes_processed_per_query, r.result_hash))


def write_bench_csv(out, rows: Sequence[BenchRow]) -> None:
    """write_bench_csv (bench.cpp:119-133)."""
    out.write("n,query,k,max_r,engine,threads,reps,total_queries,wall_time_s,queries_per_second,"
              "nodes_processed_per_query,steps_per_query,result_hash\n")
    for r in rows:
        c = r.config
        out.write("%d,%s,%d,%s,%s,%d,%d,%d,%.6f,%.1f,%.3f,%.3f,%016x\n" % (
            c.n_data, _kind(c), c.k if c.kind == QueryKind.knn else 1, _maxr_text(c.max_radius), "b200",
            _threads(c), c.reps, r.total_queries, r.wall_time, r.queries_per_second,
            r.nodes_processed_per_query, r.steps_per_query, r.result_hash))


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--dim", type=int, default=4)
    ap.add_argument("--m", type=int, default=10_000_000)
    ap.add_argument("--n", default="1000")
    ap.add_argument("--kind", choices=["fcp", "knn"], default="fcp")
    ap.add_argument("--k", default="8")
    ap.add_argument("--maxr", default="inf")
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--devices", default="0")
    ap.add_argument("--csv", default=None, help="write the CSV here (default: the table on stdout)")
    a = ap.parse_args(argv)
    base = BenchConfig(n_queries=a.m, k_dim=a.dim, kind=QueryKind[a.kind], reps=a.reps, seed=a.seed,
                       devices=[int(x) for x in a.devices.split(",")])
    rows = run_bench_matrix(base, [int(x) for x in a.n.split(",")], [int(x) for x in a.k.split(",")],
                            [float(x) for x in a.maxr.split(",")])
    if a.csv:
        with open(a.csv, "w") as f:
            write_bench_csv(f, rows)
    buf = io.StringIO()
    print_bench_table(buf, rows)
    sys.stdout.write(buf.getvalue())


if __name__ == "__main__":
    main()
