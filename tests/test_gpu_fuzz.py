"""Randomised GPU parity sweep (bounded to ~1 minute): random tree sizes up
to 200k, dims 1..10, k in 1..100, random radii, grid snapping and duplicates,
Morton on/off, both engines' counters — every batch bit-exact against the
oracle (counts, hit nodes, dist2 bits, batch stats)."""
import os
import time

import numpy as np
import pytest

import paper_2210_12859_b200 as fk

pytestmark = pytest.mark.gpu


def test_random_sweep(oracle):
    # FKD_FUZZ_SEED / FKD_FUZZ_SECONDS widen the sweep for a long run
    rng = oracle.instance_rng(int(os.environ.get("FKD_FUZZ_SEED", "20261018")))
    seconds = float(os.environ.get("FKD_FUZZ_SECONDS", "60"))
    t0 = time.time()
    cases = 0
    while time.time() - t0 < seconds and (cases < 400 or seconds > 60):
        n = rng.next_int(1, 200_000) if rng.chance(0.3) else rng.next_int(1, 5000)
        dim = rng.next_int(1, 16)
        grid = (0, 4, 8, 16, 1024)[rng.next_int(0, 4)]
        dup = (0.0, 0.05, 0.3)[rng.next_int(0, 2)]
        pts = rng.random_point_set(n, dim, grid, dup)
        nodes = oracle.build_tree(pts)
        m = rng.next_int(1, 3000)
        qs = np.stack([rng.random_query(dim, pts) for _ in range(min(m, 300))])
        if m > 300:
            qs = np.concatenate([qs, oracle.random_points(cases + 1, m - 300, dim) * np.float32(1.4) - np.float32(0.2)])
        kind = "knn" if rng.chance(0.7) else "fcp"
        k = 1 if kind == "fcp" else (rng.next_int(1, 20) if rng.chance(0.8) else rng.next_int(21, 100))
        r = (float("inf"), 0.0, 1e-3, 0.05, 0.3, 2.0)[rng.next_int(0, 5)]
        tree = fk.KdTree.from_level_order(nodes)
        morton = rng.chance(0.8)
        engine = fk.Engine.recursive if rng.chance(0.2) else fk.Engine.stack_free
        res = fk.run_batch(tree, qs, fk.BatchOptions(kind=fk.QueryKind[kind], k=k, max_radius=r, morton=morton,
                                                      engine=engine, collect_stats=rng.chance(0.3)))
        c, h, st, _ = oracle.run_batch(nodes, qs, kind, k, r, recursive=engine == fk.Engine.recursive)
        what = (cases, n, dim, grid, dup, m, kind, k, r, morton)
        assert np.array_equal(res.counts, c), what
        assert res.hits.tobytes() == h.tobytes(), what
        if cases % 3 == 0:  # the device-resident entry point on the same batch
            import torch

            opts = fk.BatchOptions(kind=fk.QueryKind[kind], k=k, max_radius=r, morton=morton, engine=engine)
            cd = torch.empty(len(qs), dtype=torch.int32, device="cuda")
            hd = torch.empty(len(qs) * opts.stride, dtype=torch.int64, device="cuda")
            fk.run_batch_device(tree, torch.from_numpy(qs).cuda(), cd, hd, opts)
            assert np.array_equal(cd.cpu().numpy(), c), what
            assert hd.cpu().numpy().tobytes() == h.tobytes(), what
        if res.stats.steps:
            assert (res.stats.steps, res.stats.nodes_visited, res.stats.nodes_processed) == \
                (int(st["steps"]), int(st["nodes_visited"]), int(st["nodes_processed"])), what
        cases += 1
    assert cases >= 20
