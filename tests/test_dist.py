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


def _np_morton(qs, bits=8):
    """Test-side Morton key (any key consistent across ranks partitions
    correctly; the GPU path uses fkd_morton_keys)."""
    c = np.clip((qs * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)
    key = np.zeros(len(qs), np.int64)
    for b in range(bits - 1, -1, -1):
        for d in range(qs.shape[1]):
            key = (key << 1) | ((c[:, d] >> b) & 1)
    return key, bits * qs.shape[1]


def _morton_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    import paper_2210_12859_b200 as fk
    from oracle import Oracle
    from paper_2210_12859_b200.shard import MortonExchange

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    nodes = fk.build_level_order(fk.random_points(3, 1, 30000, 3))
    # each rank's own batch (weak scaling), clustered so the ranges are uneven
    qs = fk.clustered_points(3, 100 + rank, 4000 + 777 * rank, 3, 8, 0.05)
    keys, kbits = _np_morton(np.clip(qs, 0, 0.999999))
    ex = MortonExchange(torch.from_numpy(qs), torch.from_numpy(keys), kbits, world)
    local = ex.local_queries.numpy()
    c, h, _, _ = o.run_batch(nodes, local, "knn", 5, 0.3)  # this rank's key range
    rc, rh = ex.return_results(torch.from_numpy(c), torch.from_numpy(h.view(np.int64)), 5)
    c0, h0, _, _ = o.run_batch(nodes, qs, "knn", 5, 0.3)  # the unpartitioned answer
    ok = np.array_equal(rc.numpy(), c0) and rh.numpy().tobytes() == h0.tobytes()
    sizes = [None] * world
    dist.all_gather_object(sizes, (len(qs), len(local)))
    out.put((rank, ok, sizes))
    dist.destroy_process_group()


def test_morton_range_partition_world2():
    """shard.MortonExchange over gloo, world size 2: every query goes to the
    rank owning its Morton range (histogram all-reduce + all-to-all), the
    answers come back to their original slots byte-identical to an
    unpartitioned run, and the ranges hold about equal shares."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_morton_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res)
    sizes = res[0][2]
    total = sum(s[0] for s in sizes)
    assert sum(s[1] for s in sizes) == total
    assert all(abs(s[1] - total / 2) < 0.1 * total for s in sizes)
