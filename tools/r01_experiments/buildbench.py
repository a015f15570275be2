"""GPU vs host tree-build timing (development aid; results go to DESIGN.md)."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk

for n in (1_000_000, 10_000_000, 100_000_000):
    pts = fk.random_points(1, 1, n, 3)
    d = torch.from_numpy(pts).cuda()
    out = fk.build_level_order_device(d)  # warm
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fk.build_level_order_device(d, out); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    rec = {"n": n, "gpu_build_ms": min(ts)}
    if n <= 10_000_000:
        t0 = time.perf_counter(); host = fk.build_level_order(pts); rec["host_build_ms"] = (time.perf_counter() - t0) * 1e3
        rec["equal"] = bool(np.array_equal(host, out.cpu().numpy()))
    print(json.dumps(rec), flush=True)
