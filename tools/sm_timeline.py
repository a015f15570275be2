"""SM occupancy of the C3 bench step, reconstructed from per-block timestamps.

Needs a profiling build of the library (block records on):
    make -C paper_2210_12859_b200/csrc OUT=../libfkd_trace.so OBJDIR=/tmp/obj_trace EXTRA=-DFKD_BLOCK_TRACE=1
    FKD_LIB=paper_2210_12859_b200/libfkd_trace.so python tools/sm_timeline.py

For the serial step (fcp call, then kNN8 call) and the one-submission step,
every walk / round / CTA-pass block records {tag, SM, start, end}; per SM the
union of its blocks' intervals is the time it had work.  Reported: the step
span, the fraction of SM-time with at least one resident walk block over the
whole step and over its last 25% (the tail), and per tag (list length x phase)
the block count and SM-time.  ncu cannot show this: it serialises kernels."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk  # noqa: E402

REC = np.dtype([("tag", "<u4"), ("sm", "<u4"), ("t0", "<u8"), ("t1", "<u8")])
PHASE = {0: "walk", 3: "round/resume", 1: "CTA pass"}


def busy(intervals):
    """Total length of the union of [t0, t1) intervals."""
    tot, end = 0, None
    for a, b in sorted(intervals):
        if end is None or a > end:
            tot += b - a
            end = b
        elif b > end:
            tot += b - end
            end = b
    return tot


def analyse(recs, sms, t_lo, t_hi):
    per_sm = {}
    for r in recs:
        per_sm.setdefault(int(r["sm"]), []).append((int(r["t0"]), int(r["t1"])))
    span = t_hi - t_lo
    tail_lo = t_hi - span // 4
    full = sum(busy([(max(a, t_lo), min(b, t_hi)) for a, b in iv if b > t_lo and a < t_hi]) for iv in per_sm.values())
    tail = sum(busy([(max(a, tail_lo), min(b, t_hi)) for a, b in iv if b > tail_lo and a < t_hi]) for iv in per_sm.values())
    tags = {}
    for r in recs:
        key = f"k{int(r['tag']) >> 8} {PHASE.get(int(r['tag']) & 0xff, '?')}"
        d = tags.setdefault(key, [0, 0])
        d[0] += 1
        d[1] += int(r["t1"]) - int(r["t0"])
    return {"span_ms": span / 1e6, "sm_busy_frac": full / (sms * span), "tail_sm_busy_frac": tail / (sms * (t_hi - tail_lo)),
            "blocks": {k: {"n": v[0], "block_ms": v[1] / 1e6} for k, v in sorted(tags.items())}}


def main():
    dev = torch.device("cuda", 0)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    n = m = 10_000_000
    tree = fk.KdTree.from_device(fk.build_level_order_device(torch.from_numpy(fk.clustered_points(1, 1, n, 3)).to(dev)))
    q = torch.from_numpy(fk.clustered_points(1, 2, m, 3)).to(dev)
    outs = [(torch.empty(m, dtype=torch.int32, device=dev), torch.empty(m, dtype=torch.int64, device=dev)),
            (torch.empty(m * 1, dtype=torch.int32, device=dev), torch.empty(m * 8, dtype=torch.int64, device=dev))]
    opts = [fk.BatchOptions(kind=fk.QueryKind.fcp), fk.BatchOptions(kind=fk.QueryKind.knn, k=8)]
    cap = 2_000_000
    buf = torch.zeros(cap * REC.itemsize // 8, dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream()
    # the host path: one fkd_run_batches call, pinned buffers (bench.py's e2e)
    qs_host = q.cpu().numpy()
    hq = fk.LIB.fkd_host_alloc(qs_host.nbytes)
    C.memmove(hq, qs_host.ctypes.data, qs_host.nbytes)
    arr = (fk._lib.fkd_host_batch * 2)()
    for i, o in enumerate(opts[::-1]):
        arr[i].queries, arr[i].m, arr[i].dim, arr[i].opt = hq, m, 3, o.to_c()
        arr[i].counts, arr[i].hits = fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * o.stride * 8)
    for mode in ("serial", "concurrent", "host-grouped"):
        def step():
            if mode == "serial":
                for (c, h), o in zip(outs, opts):
                    fk.run_batch_device(tree, q, c, h, o, stream=st)
            elif mode == "concurrent":
                fk.run_batches_device(tree, [(q, c, h, o) for (c, h), o in zip(outs, opts)], stream=st)
            else:
                assert fk.LIB.fkd_run_batches(tree.handle, arr, 2) == 0
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        cnt.zero_()
        rc = fk.LIB.fkd_debug_block_trace(C.c_void_p(buf.data_ptr()), C.c_void_p(cnt.data_ptr()), cap)
        if rc != 0:
            raise SystemExit(fk.LIB.fkd_last_error().decode())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        step()
        e1.record(st)
        e1.synchronize()
        fk.LIB.fkd_debug_block_trace(None, None, 0)
        k = min(int(cnt.item()), cap)
        recs = np.frombuffer(buf.cpu().numpy().tobytes(), dtype=REC)[:k]
        t_lo, t_hi = int(recs["t0"].min()), int(recs["t1"].max())
        res = analyse(recs, sms, t_lo, t_hi)
        res.update({"mode": mode, "step_ms_events": e0.elapsed_time(e1), "records": k})
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
