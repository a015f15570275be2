"""D2H rate into pinned memory alone vs while the C3 kNN8 walk runs on another
stream (does kernel activity slow the copy engine?).
    python tools/micro/d2h_under_walk.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2210_12859_b200 as fk  # noqa: E402

MB = 1 << 20
dev = torch.device("cuda", 0)
m = 10_000_000
tree = fk.KdTree.from_device(fk.build_level_order_device(torch.from_numpy(fk.clustered_points(1, 1, m, 3)).to(dev)))
q = torch.from_numpy(fk.clustered_points(1, 2, m, 3)).to(dev)
c = torch.empty(m, dtype=torch.int32, device=dev)
h = torch.empty(m * 8, dtype=torch.int64, device=dev)
opt = fk.BatchOptions(kind=fk.QueryKind.knn, k=8)
src = torch.empty(640 * MB, dtype=torch.uint8, device=dev)
dst = torch.empty(640 * MB, dtype=torch.uint8, pin_memory=True)
cs, ws = torch.cuda.Stream(), torch.cuda.Stream()
fk.run_batch_device(tree, q, c, h, opt, stream=ws)
torch.cuda.synchronize()
for label, with_walk in (("alone", False), ("under the kNN8 walk", True), ("alone", False), ("under the kNN8 walk", True)):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(cs):
        e0.record(cs)
        for i in range(8):
            dst[i * 80 * MB:(i + 1) * 80 * MB].copy_(src[i * 80 * MB:(i + 1) * 80 * MB], non_blocking=True)
        e1.record(cs)
    if with_walk:
        fk.run_batch_device(tree, q, c, h, opt, stream=ws)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"D2H 640 MB in 80 MB pieces {label}: {ms:.2f} ms, {640 * MB / ms / 1e6:.1f} GB/s", flush=True)
    torch.cuda.synchronize()
