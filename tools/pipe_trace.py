"""Per-job timeline of one C3 host-path call (FKD_PIPE_TRACE=1): fcp + kNN8
grouped (fkd_run_batches) with pinned buffers, or NumPy (pageable) outputs
with --pageable (then also the drain thread's per-job wait / copy times).
Usage: python tools/pipe_trace.py [--pageable] [knobs...]"""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk  # noqa: E402

m, dim = 10_000_000, 3
tree = fk.build_tree(fk.clustered_points(1, 1, m, dim))
qs = fk.clustered_points(1, 2, m, dim)
hq = fk.LIB.fkd_host_alloc(qs.nbytes)
C.memmove(hq, qs.ctypes.data, qs.nbytes)
arr = (fk._lib.fkd_host_batch * 2)()
pageable = "--pageable" in sys.argv
keep = []
for i, o in enumerate((fk.BatchOptions(kind=fk.QueryKind.knn, k=8), fk.BatchOptions())):
    arr[i].queries, arr[i].m, arr[i].dim, arr[i].opt = hq, m, dim, o.to_c()
    if pageable:
        c, h = np.ones(m, np.int32), np.ones(m * o.stride, np.int64)
        keep += [c, h]
        arr[i].counts, arr[i].hits = c.ctypes.data, h.ctypes.data
    else:
        arr[i].counts, arr[i].hits = fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * o.stride * 8)
for kv in (a for a in sys.argv[1:] if a != "--pageable"):
    k, v = kv.split("=")
    os.environ[k] = v
for rep in range(3):
    if rep == 2:
        os.environ["FKD_PIPE_TRACE"] = "1"
    t0 = time.perf_counter()
    assert fk.LIB.fkd_run_batches(tree.handle, arr, 2) == 0
    print(f"rep {rep}: {(time.perf_counter() - t0) * 1e3:.2f} ms", file=sys.stderr, flush=True)
