"""Per-call latency of small host batches (the drop-in as a request/response
server uses it): fk.run_batch (pageable NumPy buffers) and the pinned C ABI
call, M = 1 .. 100k queries, C3 tree (N = 10M clustered), fcp and kNN8;
the reference's run_batch (16 threads) on the same batch for comparison.
    python tools/latency.py"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2210_12859_b200 as fk  # noqa: E402
from oracle import Reference  # noqa: E402

ref = Reference()
n = 10_000_000
pts = fk.clustered_points(1, 1, n, 3)
tree = fk.build_tree(pts)
nodes = None
qs_all = fk.clustered_points(1, 2, 100_000, 3)
for kind, k in (("fcp", 1), ("knn", 8)):
    opt = fk.BatchOptions(kind=fk.QueryKind[kind], k=k)
    for m in (1, 10, 100, 1000, 10_000, 100_000):
        qs = np.ascontiguousarray(qs_all[:m])
        for _ in range(3):
            fk.run_batch(tree, qs, opt)
        reps = 50 if m <= 1000 else 10
        t0 = time.perf_counter()
        for _ in range(reps):
            fk.run_batch(tree, qs, opt)
        t_pg = (time.perf_counter() - t0) / reps
        hq, hc, hh = fk.LIB.fkd_host_alloc(qs.nbytes), fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * k * 8)
        C.memmove(hq, qs.ctypes.data, qs.nbytes)
        co = opt.to_c()
        for _ in range(3):
            fk.LIB.fkd_run_batch(tree.handle, hq, m, 3, C.byref(co), hc, hh, None)
        t0 = time.perf_counter()
        for _ in range(reps):
            fk.LIB.fkd_run_batch(tree.handle, hq, m, 3, C.byref(co), hc, hh, None)
        t_pin = (time.perf_counter() - t0) / reps
        for p in (hq, hc, hh):
            fk.LIB.fkd_host_free(p)
        if nodes is None:
            nodes = fk.build_level_order(pts)
        _, _, _, secs = ref.run_batch(nodes, qs, kind, k, float("inf"), threads=0)
        print(json.dumps({"kind": kind, "k": k, "m": m, "pageable_us": t_pg * 1e6, "pinned_us": t_pin * 1e6,
                          "reference_us": secs * 1e6}), flush=True)
