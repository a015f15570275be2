"""Host-path latency of a small batch (C1-size: 1M queries, N = 1M / 10M),
pinned vs pageable buffers, per knob variant:
    python tools/small_call.py '' 'FKD_CHUNK=1000000' ..."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk  # noqa: E402

for n in (1_000_000, 10_000_000):
    tree = fk.build_tree(fk.random_points(1, 1, n, 3))
    m = 1_000_000
    qs = fk.random_points(1, 2, m, 3)
    hq = fk.LIB.fkd_host_alloc(qs.nbytes)
    C.memmove(hq, qs.ctypes.data, qs.nbytes)
    for kind, k in (("fcp", 1), ("knn", 8)):
        hc, hh = fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * k * 8)
        pc, ph = np.zeros(m, np.int32), np.zeros(m * k, np.int64)
        o = fk.BatchOptions(kind=fk.QueryKind[kind], k=k).to_c()
        for variant in sys.argv[1:] or [""]:
            env = dict(p.split("=", 1) for p in variant.split(";") if p)
            old = {kk: os.environ.get(kk) for kk in env}
            os.environ.update(env)
            out = []
            for mode, (qa, ca, ha) in (("pinned", (hq, hc, hh)), ("pageable", (qs.ctypes.data, pc.ctypes.data, ph.ctypes.data))):
                ts = []
                for rep in range(6):
                    t = time.perf_counter()
                    rc = fk.LIB.fkd_run_batch(tree.handle, C.c_void_p(qa), m, 3, C.byref(o), C.c_void_p(ca), C.c_void_p(ha), None)
                    ts.append(time.perf_counter() - t)
                    assert rc == 0
                out.append(f"{mode} {min(ts[1:]) * 1e3:.2f} ms")
            t = time.perf_counter()
            res = fk.run_batch(tree, qs, fk.BatchOptions(kind=fk.QueryKind[kind], k=k))
            out.append(f"fk.run_batch {1e3 * (time.perf_counter() - t):.2f} ms")
            print(f"N={n} {kind}{k if k > 1 else ''} {variant or 'default':28s} " + "  ".join(out), flush=True)
            for kk, vv in old.items():
                if vv is None:
                    os.environ.pop(kk, None)
                else:
                    os.environ[kk] = vv
