"""World-size-2 gloo run of the multi-GPU host logic on CPU: tree replicated
by broadcast from rank 0, queries sharded into warp-aligned blocks, per-rank
results (computed here by the oracle — the CPU stand-in for each GPU) land in
disjoint slots and reproduce the single-process result hash; timing reduced
as the max over ranks."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2210_12859_b200.shard import shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    import paper_2210_12859_b200 as fk
    from oracle import Oracle
    from paper_2210_12859_b200.shard import max_over_ranks, replicate_tree, shard_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, dim, m = 20000, 3, 5003
    nodes = fk.build_level_order(fk.random_points(1, 1, n, dim)) if rank == 0 else None
    t = replicate_tree(nodes, n, dim, "cpu")
    local = t.numpy()
    qs = fk.random_points(1, 2, m, dim)
    lo, hi = shard_range(m, world, rank)
    o = Oracle()
    c, h, _, _ = o.run_batch(local, qs[lo:hi], "knn", 4, 0.2)
    # gather shards to rank 0 (host-side result assembly)
    counts = torch.zeros(m, dtype=torch.int32)
    hits = torch.zeros(m * 4, dtype=torch.int64)
    counts[lo:hi] = torch.from_numpy(c)
    hits[lo * 4: hi * 4] = torch.from_numpy(h.view(np.int64))
    dist.all_reduce(counts)
    dist.all_reduce(hits)
    tmax = max_over_ranks(0.5 + rank, "cpu")
    if rank == 0:
        hc = counts.numpy()
        hh = hits.numpy().view(fk.HIT_DTYPE)
        out.put((fk.result_hash(hc, hh, 4), tmax, local.tobytes() == nodes.tobytes()))
    else:
        out.put(None)
    dist.destroy_process_group()


def test_shard_range_covers_disjointly():
    for m in (0, 1, 31, 32, 1000, 10_000_001):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            assert all(lo % 32 == 0 or lo == m for lo, _ in spans)


def test_gloo_world2_matches_single_process():
    import paper_2210_12859_b200 as fk
    from oracle import Oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = [r for r in res if r is not None][0]
    nodes = fk.build_level_order(fk.random_points(1, 1, 20000, 3))
    c, h, _, _ = Oracle().run_batch(nodes, fk.random_points(1, 2, 5003, 3), "knn", 4, 0.2)
    assert got[0] == fk.result_hash(c, h, 4)
    assert got[1] == 1.5 and got[2]
