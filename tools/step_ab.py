"""A/B of the C3 bench step (fcp + kNN8 over N = M = 10M clustered) on one
GPU: serial run_batch_device calls vs one run_batches_device submission,
and FKD_* knob settings.  Usage:
    python tools/step_ab.py 'serial' 'concurrent' 'concurrent;FKD_BUDGET=512' ...
Each variant: 3 warm-up steps, then `--steps` timed steps (L2 flushed between
steps), interleaved over `--reps` rounds; prints ms/step (mean of the reps)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--workload", default="clustered")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    gen = fk.clustered_points if args.workload == "clustered" else (lambda s, st, n, d, *a: fk.random_points(s, st, n, d))
    n = m = 10_000_000
    nodes = fk.build_level_order_device(torch.from_numpy(gen(1, 1, n, 3, 64, 0.02)).to(dev))
    tree = fk.KdTree.from_device(nodes)
    q = torch.from_numpy(gen(1, 2, m, 3, 64, 0.02)).to(dev)
    outs = [(torch.empty(m, dtype=torch.int32, device=dev), torch.empty(m, dtype=torch.int64, device=dev)),
            (torch.empty(m, dtype=torch.int32, device=dev), torch.empty(m * 8, dtype=torch.int64, device=dev))]
    opts = [fk.BatchOptions(kind=fk.QueryKind.fcp), fk.BatchOptions(kind=fk.QueryKind.knn, k=8)]
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    ref = None
    res = {v: [] for v in args.variants}
    for rep in range(args.reps):
        for v in args.variants:
            parts = v.split(";")
            mode = parts[0]
            env = dict(p.split("=", 1) for p in parts[1:])
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)

            def step():
                if mode == "serial":
                    for (c, h), o in zip(outs, opts):
                        fk.run_batch_device(tree, q, c, h, o, stream=stream)
                else:
                    fk.run_batches_device(tree, [(q, c, h, o) for (c, h), o in zip(outs, opts)], stream=stream)

            for _ in range(3):
                step()
            ts = []
            for _ in range(args.steps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[v].append(float(np.mean(ts)))
            got = [fk.result_hash(c.cpu().numpy(), h.cpu().numpy().view(fk.HIT_DTYPE), 1 if i == 0 else 8)
                   for i, (c, h) in enumerate(outs)]
            if ref is None:
                ref = got
            assert got == ref, f"{v}: results differ"
            for k, val in old.items():
                if val is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = val
    for v in args.variants:
        print(f"{v:50s} ms/step {np.mean(res[v]):.3f}  reps {['%.3f' % x for x in res[v]]}  "
              f"q/s {2 * m / np.mean(res[v]) * 1e3 / 1e9:.3f} G", flush=True)


if __name__ == "__main__":
    main()
