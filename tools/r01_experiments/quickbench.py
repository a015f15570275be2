"""Quick device-resident timing sweep (development aid, not the bench contract)."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--m", type=int, default=10_000_000)
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--clustered", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--configs", default="fcp,knn8,knn8r01")
    ap.add_argument("--sorted-only", action="store_true")
    args = ap.parse_args()
    gen = (lambda s, c: fk.clustered_points(1, s, c, args.dim)) if args.clustered else \
        (lambda s, c: fk.random_points(1, s, c, args.dim))
    t0 = time.time()
    pts = gen(1, args.n)
    qs = gen(2, args.m)
    t1 = time.time()
    nodes = fk.build_level_order(pts)
    t2 = time.time()
    tree = fk.KdTree.from_level_order(nodes)
    print(f"gen {t1-t0:.2f}s build {t2-t1:.2f}s layout={os.environ.get('FKD_LAYOUT','padded')}", flush=True)
    dq = torch.from_numpy(qs).cuda()
    cfgs = {"fcp": (fk.QueryKind.fcp, 1, float("inf")), "knn8": (fk.QueryKind.knn, 8, float("inf")),
            "knn8r01": (fk.QueryKind.knn, 8, 0.01), "knn16": (fk.QueryKind.knn, 16, float("inf")),
            "knn4": (fk.QueryKind.knn, 4, float("inf")), "knn50": (fk.QueryKind.knn, 50, float("inf")),
            "knn20": (fk.QueryKind.knn, 20, float("inf")), "knn32": (fk.QueryKind.knn, 32, float("inf")),
            "knn64": (fk.QueryKind.knn, 64, float("inf"))}
    for name in args.configs.split(","):
        kind, k, r = cfgs[name]
        counts = torch.empty(args.m, dtype=torch.int32, device="cuda")
        hits = torch.empty(args.m * k, dtype=torch.int64, device="cuda")
        for morton in ((True,) if args.sorted_only else (True, False)):
            opt = fk.BatchOptions(kind=kind, k=k, max_radius=r, morton=morton)
            fk.run_batch_device(tree, dq, counts, hits, opt)
            walk, order, tail, ovf = [], [], [], 0
            for _ in range(args.reps):
                _, tm = fk.run_batch_device(tree, dq, counts, hits, opt, timings=True)
                walk.append(tm["walk_ms"])
                order.append(tm["order_ms"])
                tail.append(tm["tail_ms"])
                ovf = tm["overflowed"]
            st, _ = fk.run_batch_device(tree, dq, counts, hits,
                                        fk.BatchOptions(kind=kind, k=k, max_radius=r, morton=morton,
                                                        collect_stats=True))
            w = float(np.median(walk))
            o = float(np.median(order))
            print(json.dumps({"cfg": name, "morton": morton, "walk_ms": round(w, 3), "order_ms": round(o, 3), "tail_ms": round(float(np.median(tail)), 3), "overflowed": ovf,
                              "walk_qps": round(args.m / w * 1e3 / 1e6, 1), "total_qps_M": round(args.m / (w + o) * 1e3 / 1e6, 1),
                              "P": st.nodes_processed / args.m, "steps": st.steps / args.m}), flush=True)


if __name__ == "__main__":
    main()
