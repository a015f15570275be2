"""Device walk time of one batch configuration under knob variants.
    python tools/kernel_ab.py --dim 8 --k 16 --m 1000000 '' 'FKD_BUDGET=1;FKD_RESUME_MIN=1000000000'
Each variant: warm-up + `--reps` timed calls (median); results must be identical."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="*", default=[""])
    ap.add_argument("--dim", type=int, default=4)
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--r", type=float, default=float("inf"))
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--m", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--clustered", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    gen = (lambda s, n: fk.clustered_points(1, s, n, a.dim)) if a.clustered else (lambda s, n: fk.random_points(1, s, n, a.dim))
    nodes = fk.build_level_order_device(torch.from_numpy(gen(1, a.n)).to(dev))
    tree = fk.KdTree.from_device(nodes)
    q = torch.from_numpy(gen(2, a.m)).to(dev)
    kind = fk.QueryKind.knn if a.k > 1 else fk.QueryKind.fcp
    c = torch.empty(a.m, dtype=torch.int32, device=dev)
    h = torch.empty(a.m * a.k, dtype=torch.int64, device=dev)
    ref = None
    for v in a.variants:
        env = dict(p.split("=", 1) for p in v.split(";") if p)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        ts = []
        for i in range(a.reps + 1):
            _, tm = fk.run_batch_device(tree, q, c, h, fk.BatchOptions(kind=kind, k=a.k, max_radius=a.r), timings=True)
            ts.append(tm)
        got = fk.result_hash(c.cpu().numpy(), h.cpu().numpy().view(fk.HIT_DTYPE), a.k)
        ref = ref if ref is not None else got
        walk = float(np.median([t["walk_ms"] for t in ts[1:]]))
        print(json.dumps({"variant": v or "default", "dim": a.dim, "k": a.k, "m": a.m, "walk_ms": walk,
                          "qps": a.m / walk * 1e3, "tail_ms": float(np.median([t["tail_ms"] for t in ts[1:]])),
                          "overflowed": ts[-1]["overflowed"], "same": got == ref, "hash": f"{got:016x}"}), flush=True)
        for k_, v_ in old.items():
            if v_ is None:
                os.environ.pop(k_, None)
            else:
                os.environ[k_] = v_


if __name__ == "__main__":
    main()
