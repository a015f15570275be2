"""What the Morton-range partition buys one GPU at C5 (N = 100M uniform
tree, fcp), measured on ONE B200: a rank's share of G-way block sharding is
M/G queries spread over the whole cube; under the Morton-range partition it
is M/G queries inside the rank's 1/G key range — for uniform queries the
region where the top log2(G) Morton bits (x, then y, then z) are fixed, i.e.
x < 1/2 (G = 2), x, y < 1/2 (G = 4), the octant (G = 8).  Both are walked as
one device batch (Morton order, CUDA events); the ratio is the per-GPU walk
gain the exchange has to pay for.
    python tools/partition_locality.py [--m 125000000]"""
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
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--m", type=int, default=125_000_000)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    nodes = fk.build_level_order_device(torch.from_numpy(fk.random_points(1, 1, a.n, 3)).to(dev))
    tree = fk.KdTree.from_device(nodes)
    del nodes
    base = torch.from_numpy(fk.random_points(1, 2, a.m, 3)).to(dev)
    c = torch.empty(a.m, dtype=torch.int32, device=dev)
    h = torch.empty(a.m, dtype=torch.int64, device=dev)
    for g, dims in ((1, 0), (2, 1), (4, 2), (8, 3)):
        q = base.clone()
        q[:, :dims] *= 0.5  # the rank's Morton range for uniform queries
        ts = []
        for _ in range(a.reps + 1):
            _, tm = fk.run_batch_device(tree, q, c, h, fk.BatchOptions(), timings=True)
            ts.append(tm["order_ms"] + tm["walk_ms"])
        ms = float(np.median(ts[1:]))
        print(json.dumps({"G": g, "region": ["cube", "x<1/2", "x,y<1/2", "octant"][dims], "m": a.m,
                          "ms": ms, "qps": a.m / ms * 1e3}), flush=True)
        del q


if __name__ == "__main__":
    main()
