"""C3 (fcp + kNN8, clustered, N=M=10M): the two batches back to back (bench.py's
step) against both in flight at once from two host threads, each on its own
stream (the C ABI is re-entrant; each call takes its own workspace).  Device-
resident (events on a join stream) and end to end (pinned host buffers)."""
import ctypes as C
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk  # noqa: E402

n = m = 10_000_000
pts = fk.clustered_points(1, 1, n, 3, 64, 0.02)
qs = fk.clustered_points(1, 2, m, 3, 64, 0.02)
tree = fk.KdTree.from_level_order(fk.build_level_order(pts))
dq = torch.from_numpy(qs).cuda()
batches = [(fk.QueryKind.fcp, 1), (fk.QueryKind.knn, 8)]
outs = [(torch.empty(m, dtype=torch.int32, device="cuda"), torch.empty(m * k, dtype=torch.int64, device="cuda"))
        for _, k in batches]
opts = [fk.BatchOptions(kind=kd, k=k) for kd, k in batches]
streams = [torch.cuda.Stream() for _ in batches]
main = torch.cuda.current_stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def seq():
    for (c, h), o in zip(outs, opts):
        fk.run_batch_device(tree, dq, c, h, o, stream=main)


def conc():
    ev = torch.cuda.Event()
    ev.record(main)
    done = [torch.cuda.Event() for _ in batches]

    def one(i):
        streams[i].wait_event(ev)
        fk.run_batch_device(tree, dq, outs[i][0], outs[i][1], opts[i], stream=streams[i])
        done[i].record(streams[i])
    ts = [threading.Thread(target=one, args=(i,)) for i in range(len(batches))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for d in done:
        main.wait_event(d)


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        fn()
        e1.record(main)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out)), float(np.min(out))


ref = None
for name, fn in (("sequential", seq), ("concurrent", conc), ("sequential", seq), ("concurrent", conc)):
    med, mn = timed(fn)
    got = [(c.cpu().numpy().tobytes(), h.cpu().numpy().tobytes()) for c, h in outs]
    ref = ref or got
    print(f"device {name}: {med:.3f} ms (min {mn:.3f}) -> {2 * m / med / 1e6:.0f} M q/s, same={got == ref}", flush=True)

# end to end, pinned host buffers
hq = fk.LIB.fkd_host_alloc(qs.nbytes)
C.memmove(hq, qs.ctypes.data, qs.nbytes)
hout = [(fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * k * 8)) for _, k in batches]
copts = [o.to_c() for o in opts]


def e2e_one(i):
    rc = fk.LIB.fkd_run_batch(tree.handle, hq, m, 3, C.byref(copts[i]), hout[i][0], hout[i][1], None)
    assert rc == 0, fk.LIB.fkd_last_error()


def e2e_seq():
    for i in range(len(batches)):
        e2e_one(i)


def e2e_conc():
    ts = [threading.Thread(target=e2e_one, args=(i,)) for i in range(len(batches))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


for name, fn in (("sequential", e2e_seq), ("concurrent", e2e_conc), ("sequential", e2e_seq), ("concurrent", e2e_conc)):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(8):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    med = float(np.median(ts)) * 1e3
    print(f"e2e {name}: {med:.2f} ms -> {2 * m / med / 1e3:.0f} M q/s", flush=True)
