"""Per-batch timeline inside one concurrent C3 step (fkd_run_batches_device):
for each batch, ms from the fork to its order end, tail start and walk end.
python tools/step_timeline.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk  # noqa: E402

dev = torch.device("cuda", 0)
n = m = 10_000_000
tree = fk.KdTree.from_device(fk.build_level_order_device(torch.from_numpy(fk.clustered_points(1, 1, n, 3)).to(dev)))
q = torch.from_numpy(fk.clustered_points(1, 2, m, 3)).to(dev)
outs = [(torch.empty(m, dtype=torch.int32, device=dev), torch.empty(m, dtype=torch.int64, device=dev)),
        (torch.empty(m, dtype=torch.int32, device=dev), torch.empty(m * 8, dtype=torch.int64, device=dev))]
opts = [fk.BatchOptions(kind=fk.QueryKind.fcp), fk.BatchOptions(kind=fk.QueryKind.knn, k=8)]
st = torch.cuda.current_stream()
for rep in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    res = fk.run_batches_device(tree, [(q, c, h, o) for (c, h), o in zip(outs, opts)], stream=st, timings=True)
    e1.record(st)
    e1.synchronize()
    if rep >= 3:
        line = [f"step {e0.elapsed_time(e1):.3f} ms"]
        for name, (_, tm) in zip(("fcp", "knn8"), res):
            end = tm["order_ms"] + tm["walk_ms"]
            line.append(f"{name}: order {tm['order_ms']:.3f} tail_start {end - tm['tail_ms']:.3f} end {end:.3f}")
        print(" | ".join(line), flush=True)
