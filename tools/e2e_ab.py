"""fkd_run_batch end to end on C3 (fcp + kNN8, 10M clustered) under knob
variants, pinned and pageable caller buffers.  Usage:
    python tools/e2e_ab.py '' 'FKD_HOST_RING=8' 'FKD_HOST_RING=2;FKD_CHUNK_DIV=16' ...
Prints ms per call (min of 4 after a warm-up) for each kind and buffer mode."""
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
bufs = {}
for kind, k in (("fcp", 1), ("knn", 8)):
    pc, ph = np.empty(m, np.int32), np.empty(m * k, np.int64)
    pc.fill(0)
    ph.fill(0)
    bufs[kind] = (k, fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * k * 8), pc, ph)
for variant in sys.argv[1:] or [""]:
    env = dict(p.split("=", 1) for p in variant.split(";") if p)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    out = []
    for kind in ("fcp", "knn"):
        k, hc, hh, pc, ph = bufs[kind]
        o = fk.BatchOptions(kind=fk.QueryKind[kind], k=k).to_c()
        for mode, (qa, ca, ha) in (("pinned", (hq, hc, hh)), ("pageable", (qs.ctypes.data, pc.ctypes.data, ph.ctypes.data))):
            ts = []
            for rep in range(5):
                t = time.perf_counter()
                rc = fk.LIB.fkd_run_batch(tree.handle, C.c_void_p(qa), m, dim, C.byref(o), C.c_void_p(ca),
                                          C.c_void_p(ha), None)
                ts.append(time.perf_counter() - t)
                assert rc == 0, fk.LIB.fkd_last_error()
            out.append(f"{kind}/{mode} {min(ts[1:]) * 1e3:.2f}")
    print(f"{variant or 'default':40s} " + "  ".join(out), flush=True)
    for key, val in old.items():
        if val is None:
            os.environ.pop(key, None)
        else:
            os.environ[key] = val
