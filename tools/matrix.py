"""Config matrix of BASELINE.json (C1..C5) on one B200, with the reference's
run_batch timed on the host cores on a sample and a parity hash per config.

    python tools/matrix.py [--only c1,c4] > profiles/rNN_matrix.jsonl

Every line: config, walk ms (device-resident, Morton order, CUDA events),
queries/s, P-bar, algorithmic bytes/query, HBM roofline fraction, reference
q/s (16 host threads, sample), parity of the sample's result hash.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2210_12859_b200 as fk  # noqa: E402
from oracle import Reference  # noqa: E402

INF = float("inf")


def _hbm_peak() -> float:
    """Measured HBM GB/s (MEASURED_PEAKS.json, driver-written), else the
    B200_PROFILING.md fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


HBM = _hbm_peak()


def gen(kind, stream, count, dim):
    if kind == "clustered":
        return fk.clustered_points(1, stream, count, dim, 64, 0.02)
    return fk.random_points(1, stream, count, dim)


def bq(dim, p, stride):
    return 4 * dim + p * 4 * dim + 4 + 8 * stride


def run(ref, name, n, m, dim, data, batches, cpu_sample, unordered=(False,), reps=3, unordered_m=100_000):
    pts = gen(data, 1, n, dim)
    nodes_d = fk.build_level_order_device(torch.from_numpy(pts).cuda())
    del pts
    tree = fk.KdTree.from_device(nodes_d)
    qs = gen(data, 2, m, dim)
    dq = torch.from_numpy(qs).cuda()
    nodes_h = nodes_d.cpu().numpy() if cpu_sample else None
    del nodes_d
    for kind, k, r in batches:
        stride = k if kind == "knn" else 1
        counts = torch.empty(m, dtype=torch.int32, device="cuda")
        hits = torch.empty(m * stride, dtype=torch.int64, device="cuda")
        for uo in unordered:
            # the unordered walk is measured as itself (no step budget /
            # overflow pass, which would finish it with ordered subtree walks)
            os.environ["FKD_BUDGET"] = "0" if uo else os.environ.get("FKD_BUDGET_ORDERED", "-1")
            mm = m if not uo else min(m, unordered_m)
            opt = fk.BatchOptions(kind=fk.QueryKind[kind], k=k, max_radius=r, unordered=uo)
            dqm, cm, hm = dq[:mm], counts[:mm], hits[: mm * stride]
            fk.run_batch_device(tree, dqm, cm, hm, opt)
            walk, order, tail = [], [], []
            for _ in range(reps):
                _, tm = fk.run_batch_device(tree, dqm, cm, hm, opt, timings=True)
                walk.append(tm["walk_ms"]); order.append(tm["order_ms"]); tail.append(tm["tail_ms"])
            st, _ = fk.run_batch_device(tree, dqm, cm, hm, fk.BatchOptions(
                kind=fk.QueryKind[kind], k=k, max_radius=r, unordered=uo, collect_stats=True))
            w = float(np.median(walk)); o = float(np.median(order))
            p = st.nodes_processed / mm
            rec = {"config": name, "n": n, "m": mm, "dim": dim, "data": data, "kind": kind, "k": k,
                   "max_radius": r, "unordered": uo, "walk_ms": w, "order_ms": o,
                   "tail_ms": float(np.median(tail)), "walk_qps": mm / w * 1e3,
                   "batch_qps": mm / (w + o) * 1e3, "P_bar": p, "steps_per_query": st.steps / mm,
                   "bytes_per_query": bq(dim, p, stride),
                   "hbm_frac": mm * bq(dim, p, stride) / (w * 1e-3) / 1e9 / HBM,
                   "note": ("P_bar is the reference walk's (STATS pass); from 5-D the production walk "
                            "prunes by cell box and processes fewer nodes") if dim >= 5 else ""}
            if cpu_sample and not uo:
                s = min(m, cpu_sample)
                qsam = np.ascontiguousarray(qs[:s])
                c, h, _, secs = ref.run_batch(nodes_h, qsam, kind, k, r, threads=0)
                res = fk.run_batch(tree, qsam, fk.BatchOptions(kind=fk.QueryKind[kind], k=k, max_radius=r))
                rec.update({"cpu_ref_qps": s / secs, "cpu_sample": s, "cpu_threads": ref.hardware_threads(),
                            "parity_sample_hash_equal": res.result_hash() == ref.result_hash(c, h, stride),
                            "gpu_vs_cpu": (m / (w + o) * 1e3) / (s / secs)})
            print(json.dumps(rec), flush=True)
        del counts, hits
    del dq, tree
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c2,c3,c4,c5")  # also: paper, hd
    ap.add_argument("--c5-queries", type=int, default=1_000_000_000)
    args = ap.parse_args()
    ref = Reference()
    only = set(args.only.split(","))
    if "c1" in only:
        run(ref, "C1", 1_000_000, 1_000_000, 3, "uniform", [("fcp", 1, INF)], 1_000_000)
    if "c2" in only:
        run(ref, "C2", 1_000_000, 1_000_000, 3, "uniform", [("knn", 8, 0.01), ("knn", 8, INF)], 1_000_000)
    if "c3" in only:
        run(ref, "C3", 10_000_000, 10_000_000, 3, "clustered", [("fcp", 1, INF), ("knn", 8, INF)], 1_000_000)
        run(ref, "C3-uniform", 10_000_000, 10_000_000, 3, "uniform", [("fcp", 1, INF), ("knn", 8, INF)], 1_000_000)
    if "c4" in only:
        for dim, m, sample, um in ((2, 10_000_000, 200_000, 20_000), (4, 10_000_000, 100_000, 5_000),
                                   (8, 1_000_000, 20_000, 2_000)):
            run(ref, f"C4-{dim}D", 10_000_000, m, dim, "uniform", [("knn", 16, INF)], sample,
                unordered=(False, True), reps=2, unordered_m=um)
    if "paper" in only:  # PAPER.md Table 1 setting: 4-D uniform, N=10M, M=10M (RTX 3090 Ti numbers)
        run(ref, "paper-4D", 10_000_000, 10_000_000, 4, "uniform",
            [("fcp", 1, INF), ("knn", 4, INF), ("knn", 8, INF), ("knn", 20, INF), ("knn", 50, INF),
             ("knn", 4, 0.01), ("knn", 8, 0.01), ("knn", 20, 0.01), ("knn", 50, 0.01)], 100_000, reps=2)
    if "hd" in only:  # beyond the BASELINE configs: 9..16-D register walks (N = M = 1M uniform)
        for dim, sample in ((10, 20_000), (12, 10_000), (16, 2_000)):
            run(ref, f"HD-{dim}D", 1_000_000, 1_000_000, dim, "uniform", [("fcp", 1, INF), ("knn", 8, INF)], sample,
                reps=1)
    if "c5" in only:
        t0 = time.time()
        run(ref, "C5", 100_000_000, args.c5_queries, 3, "uniform", [("fcp", 1, INF)], 2_000_000, reps=2)
        print(json.dumps({"config": "C5", "wall_s": time.time() - t0}), flush=True)


if __name__ == "__main__":
    main()
