"""Cost of walking a batch in slices (what the host pipeline's chunks do):
C3 (10M clustered), kNN8 and fcp, the batch cut into 1..16 slices walked one
after another, slices taken (a) in input order — each a random sample of the
whole distribution, as the host pipeline's chunks are — and (b) in global
Morton order — each a compact region at full query density.  Sum of per-slice
order + walk ms (CUDA events).  python tools/slice_ab.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk  # noqa: E402

dev = torch.device("cuda", 0)
n = m = 10_000_000
nodes = fk.build_level_order_device(torch.from_numpy(fk.clustered_points(1, 1, n, 3)).to(dev))
tree = fk.KdTree.from_device(nodes)
q = torch.from_numpy(fk.clustered_points(1, 2, m, 3)).to(dev)
keys, _ = fk.morton_keys(tree, q)
qs = q[torch.argsort(keys)].contiguous()
for kind, k in ((fk.QueryKind.knn, 8), (fk.QueryKind.fcp, 1)):
    for name, src in (("input-order", q), ("morton-order", qs)):
        for parts in (1, 2, 4, 8, 16):
            per = m // parts
            c = torch.empty(per, dtype=torch.int32, device=dev)
            h = torch.empty(per * k, dtype=torch.int64, device=dev)
            tot = []
            for rep in range(3):
                s = 0.0
                for p in range(parts):
                    _, tm = fk.run_batch_device(tree, src[p * per:(p + 1) * per], c, h, fk.BatchOptions(kind=kind, k=k),
                                                timings=True)
                    s += tm["order_ms"] + tm["walk_ms"]
                tot.append(s)
            print(f"{kind.name}{k if k > 1 else ''} {name:13s} slices {parts:2d} sum ms {np.median(tot):.3f}", flush=True)
