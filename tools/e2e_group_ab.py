"""C3 grouped host call (fkd_run_batches, fcp + kNN8, pinned and pageable)
under knob variants: python tools/e2e_group_ab.py '' 'FKD_ROUNDS_MIN_M=1000000' ..."""
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
opts = (fk.BatchOptions(kind=fk.QueryKind.knn, k=8), fk.BatchOptions())
arrs = {}
for mode in ("pinned", "pageable"):
    arr = (fk._lib.fkd_host_batch * 2)()
    for i, o in enumerate(opts):
        if mode == "pinned":
            c, h = fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * o.stride * 8)
            q = hq
        else:
            ca, ha = np.zeros(m, np.int32), np.zeros(m * o.stride, np.int64)
            ca.fill(1)
            ha.fill(1)
            arrs.setdefault("keep", []).extend([ca, ha])
            c, h, q = ca.ctypes.data, ha.ctypes.data, qs.ctypes.data
        arr[i].queries, arr[i].m, arr[i].dim, arr[i].opt = q, m, dim, o.to_c()
        arr[i].counts, arr[i].hits = c, h
    arrs[mode] = arr
for variant in sys.argv[1:] or [""]:
    env = dict(p.split("=", 1) for p in variant.split(";") if p)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    out = []
    for mode in ("pinned", "pageable"):
        ts = []
        for rep in range(5):
            t = time.perf_counter()
            assert fk.LIB.fkd_run_batches(tree.handle, arrs[mode], 2) == 0, fk.LIB.fkd_last_error()
            ts.append(time.perf_counter() - t)
        best = min(ts[1:])
        out.append(f"{mode} {best * 1e3:.2f} ms ({2 * m / best / 1e9:.3f} G q/s)")
    print(f"{variant or 'default':45s} " + "  ".join(out), flush=True)
    for key, val in old.items():
        if val is None:
            os.environ.pop(key, None)
        else:
            os.environ[key] = val
