#!/usr/bin/env python3
"""Benchmark: fcp + kNN(k=8) queries/s on B200 (BASELINE.json metric).

Workload (default ``c3``, BASELINE.json configs[2]): 3-D float, N = 10M
points from 64 Gaussian blobs (sigma 0.02), M = 10M queries from the same
mixture, walked in Morton order.  One *step* = one fcp batch over the M
queries + one unbounded kNN(k=8) batch over the same M queries, each a full
``fkd_run_batch_device`` call (Morton keys + radix sort + walk).  ``value``
= 2*M*N_gpus / step time with inputs resident in HBM; ``e2e`` = the same
through the host-buffer C ABI call ``fkd_run_batch`` (H2D + walk + D2H
inside the timed region, pinned host buffers).

Multi-GPU (torchrun): one rank per GPU, the tree is built on rank 0 and
replicated with an NCCL broadcast; every rank walks its own M queries
(weak scaling, no per-query communication); time = max over ranks.

``--impl reference`` times the reference's own ``flatkd::run_batch``
(oracle/_ref, compiled unmodified from the reference sources) with all
host threads over the same full batches (C5's 1B queries: a 10M sample),
generating the identical inputs with the reference's own RNG; it never
loads the product library.  ``e2e_pageable`` times the drop-in with
NumPy (pageable) buffers, the way a reference caller's std::vectors arrive.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (description, N, M, dim, generator, [(kind, k, max_radius), ...])
    "c3": ("fcp + kNN8 3D, N=10M clustered (64 Gaussian blobs, sigma=0.02), M=10M queries "
           "from the same mixture, Morton-ordered", 10_000_000, 10_000_000, 3, "clustered",
           [("fcp", 1, float("inf")), ("knn", 8, float("inf"))]),
    "c3u": ("fcp + kNN8 3D, N=10M uniform, M=10M uniform queries, Morton-ordered",
            10_000_000, 10_000_000, 3, "uniform", [("fcp", 1, float("inf")), ("knn", 8, float("inf"))]),
    "c1": ("fcp 3D, N=1M uniform, M=1M uniform queries", 1_000_000, 1_000_000, 3, "uniform",
           [("fcp", 1, float("inf"))]),
    "c2": ("kNN8 3D, N=1M uniform, M=1M queries, maxR=0.01", 1_000_000, 1_000_000, 3, "uniform",
           [("knn", 8, 0.01)]),
    # C5 is strong scaling in the BASELINE (1B queries over 1/2/4/8 GPUs); run
    # per rank as 1B / world queries with --workload c5
    "c5": ("fcp 3D, N=100M uniform replicated tree, 1B uniform queries sharded over the GPUs",
           100_000_000, 1_000_000_000, 3, "uniform", [("fcp", 1, float("inf"))]),
}
SEED = 1
METRIC = "fcp & kNN(k=8) queries/sec, 3D float, N=10M, 1/2/4/8 B200 vs host CPU"


def gen_points(gen, kind: str, stream: int, count: int, dim: int) -> np.ndarray:
    """Workload points from `gen`: the product's host generators (B200 arm)
    or the reference library's (reference arm, oracle/ref_capi.cpp) — the
    two are byte-identical (tests/test_host.py), so both arms walk the same
    inputs while the reference arm never loads the product library."""
    if kind == "clustered":
        return gen.clustered_points(SEED, stream, count, dim, 64, 0.02)
    if hasattr(gen, "stream_points"):
        return gen.stream_points(SEED, stream, count, dim)
    return gen.random_points(SEED, stream, count, dim)


def query_stream(rank: int) -> int:
    """RNG stream of a rank's queries (weak scaling): rank 0 uses the
    reference's query stream (rng.hpp:24), other ranks private streams
    (same rule as paper_2210_12859_b200.shard.query_stream)."""
    return 2 if rank == 0 else 1000 + rank


def workload_config(workload: str, world: int) -> dict:
    """The `config` object of the JSON line — identical in both arms."""
    desc, n, m, dim, gkind, batches = WORKLOADS[workload]
    strong = workload == "c5"
    return {"workload": desc, "tree_n": n, "queries_per_gpu": (m // world if strong else m), "dim": dim,
            "batches_per_step": [("fcp" if kk == "fcp" else f"knn{k2}") for kk, k2, _ in batches],
            "max_radius": [rr for _, _, rr in batches], "parallelism": f"query-sharded x{world}",
            "l2": "flushed: the B200 arm writes a 256 MB buffer (> 126 MB L2) between timed steps "
                  f"(untimed); inputs {m * dim * 4 / 1e6:.0f} MB of queries + {n * 16 / 1e6:.0f} MB tree store",
            "morton": True, "seed": SEED}


def host_cpu() -> dict:
    """Host cores and CPU model of this box (BASELINE.md §3 asks for both)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count() or 1, "cpu_model": model}


def repo_native_libs() -> list:
    """In-repo shared libraries mapped into this process (which native code ran)."""
    libs = set()
    try:
        for line in open("/proc/self/maps"):
            path = line.split()[-1] if len(line.split()) >= 6 else ""
            if path.endswith(".so") and path.startswith(ROOT):
                libs.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(libs)


def bytes_per_query(dim: int, p_bar: float, stride: int) -> float:
    """Algorithmic bytes: query + every processed point once
    + count + hit slots."""
    return 4 * dim + p_bar * 4 * dim + 4 + 8 * stride


def measured_peaks() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = f"/tmp/fkd_clocks_{os.getpid()}.csv"

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) == 6 and parts[0].isdigit():
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(statistics.median(float(r[0]) for r in rows)),
                "sm_max_mhz": float(max(float(r[1]) for r in rows)), "reasons": reasons,
                "samples": len(rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------- reference arm

def run_reference(args) -> None:
    """The reference's own flatkd::run_batch (oracle/_ref, built unmodified
    from /root/reference by oracle/Makefile) over the FULL batch of every
    step, timed exactly as run_cell does (bench.cpp:35-41: run_batch only).
    Nothing from the product package is imported or loaded here."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import Reference

    desc, n, m, dim, gkind, batches = WORKLOADS[args.workload]
    ref = Reference()
    threads = ref.hardware_threads()
    # the tree is input, not the path: flatkd::build_tree, untimed (bench.hpp:35-37)
    nodes = ref.build_tree(gen_points(ref, gkind, 1, n, dim))
    strong = args.workload == "c5"
    m_rank = m // world if strong else m
    sample = m_rank if args.ref_sample <= 0 else min(m_rank, args.ref_sample)
    qs = gen_points(ref, gkind, 2 if strong else query_stream(0), sample, dim)
    times, hashes = [], {}
    for it in range(args.warmup + args.steps):
        t = 0.0
        for kind, k, r in batches:
            c, h, _, secs = ref.run_batch(nodes, qs, kind, k, r, threads=0)
            t += secs
            if it == 0:
                hashes[kind if kind == "fcp" else f"knn{k}"] = f"{ref.result_hash(c, h, k if kind == 'knn' else 1):016x}"
        if it >= args.warmup:
            times.append(t)
    step = float(np.mean(times))
    value = len(batches) * sample / step
    cpu = host_cpu()
    what = "every query of the batch" if sample == m_rank else f"first {sample} of the {m_rank} queries"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic", "config": workload_config(args.workload, world),
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": threads, "kind": "reference",
                         **cpu, "sample": f"{what}, each batch of the step, flatkd::run_batch "
                                          "(Engine::stack_free, OpenMP, all host threads), rank 0 only"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "result_hash": hashes,
        "native_libs": repo_native_libs(),
    }
    assert not any("libfkd_b200" in x for x in line["native_libs"]), "reference arm loaded the product"
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- B200 arm

def cpu_baseline_leg(nodes, qs_host, batches, sample, gpu_hashes) -> dict:
    """The reference's run_batch on this box's host cores over the same tree
    and queries (the whole batch unless --cpu-sample caps it), timed as
    run_cell does (bench.cpp:35-41), plus its result hashes against the
    B200 path's (the device-resident outputs of the timed steps)."""
    from oracle import REF_SO, Oracle, Reference

    kind_name = "reference" if os.path.exists(REF_SO) else "port"
    impl = Reference() if kind_name == "reference" else Oracle()
    q = np.ascontiguousarray(qs_host[:sample])
    total_t = 0.0
    parity = True
    for kind, k, r in batches:
        if kind_name == "reference":
            c, h, _, secs = impl.run_batch(nodes, q, kind, k, r, threads=0)
        else:
            t0 = time.perf_counter()
            c, h, _, _ = impl.run_batch(nodes, q, kind, k, r, threads=0)
            secs = time.perf_counter() - t0
        total_t += secs
        name = kind if kind == "fcp" else f"knn{k}"
        if sample == len(qs_host):
            parity &= f"{impl.result_hash(c, h, k if kind == 'knn' else 1):016x}" == gpu_hashes[name]
    cpu = host_cpu()
    threads = impl.hardware_threads() if kind_name == "reference" else cpu["nproc"]
    what = "every query of rank 0's batch" if sample == len(qs_host) else f"first {sample} queries of rank 0"
    line = {"value": len(batches) * sample / total_t, "unit": "queries/s", "cores": threads,
            "kind": kind_name, **cpu,
            "sample": f"{what}, every batch of the step, "
                      f"{'flatkd::run_batch from oracle/_ref' if kind_name == 'reference' else 'oracle port'}"
                      f" with {threads} OpenMP threads"}
    if sample == len(qs_host):
        line["parity_hash_equal"] = bool(parity)
    return line


def run_b200(args) -> None:
    import ctypes as C

    import torch

    import paper_2210_12859_b200 as fk
    from paper_2210_12859_b200.shard import MortonExchange, max_over_ranks, replicate_tree, shard_range

    world, rank, local = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    desc, n, m, dim, gkind, batches = WORKLOADS[args.workload]

    # ---- tree: built on rank 0 (GPU builder, byte-identical to
    # flatkd::build_tree), replicated by NCCL broadcast
    if rank == 0:
        nodes_dev = fk.build_level_order_device(torch.from_numpy(gen_points(fk, gkind, 1, n, dim)).to(dev))
        nodes_host = nodes_dev.cpu().numpy()
    else:
        nodes_host = None
        nodes_dev = None
    nodes_dev = replicate_tree(nodes_host, n, dim, dev) if world > 1 else nodes_dev
    tree = fk.KdTree.from_device(nodes_dev)

    strong = args.workload == "c5"
    if strong:  # 1B queries split across the ranks (contiguous blocks of one stream)
        lo, hi = shard_range(m, world, rank)
        m = hi - lo
        qs_host = gen_points(fk, gkind, 2, hi, dim)[lo:hi].copy() if world > 1 else gen_points(fk, gkind, 2, m, dim)
    else:
        qs_host = gen_points(fk, gkind, query_stream(rank), m, dim)
    qs_dev = torch.from_numpy(qs_host).to(dev)
    outs = {}
    for kind, k, _ in batches:
        outs[(kind, k)] = (torch.empty(m, dtype=torch.int32, device=dev),
                           torch.empty(m * k, dtype=torch.int64, device=dev))
    opts = [fk.BatchOptions(kind=fk.QueryKind[kind], k=k, max_radius=r) for kind, k, r in batches]

    # ---- untimed stats pass: P-bar per batch (algorithmic bytes)
    pbar = {}
    for (kind, k, r), o in zip(batches, opts):
        c, h = outs[(kind, k)]
        st, _ = fk.run_batch_device(tree, qs_dev, c, h, fk.BatchOptions(kind=o.kind, k=k, max_radius=r,
                                                                        collect_stats=True))
        pbar[(kind, k)] = st.nodes_processed / m

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > L2
    stream = torch.cuda.current_stream()

    def step(timing: bool):
        """One step: every batch of the workload over the step's queries.
        Default: one fkd_run_batches_device submission (the batches run
        concurrently, the costliest at the highest stream priority, sharing
        one Morton order of the common query array); --serial: back-to-back
        fkd_run_batch_device calls."""
        if args.partition == "morton" and world > 1:
            # Morton-range partition: keys, histogram
            # all-reduce, all-to-all of the queries, the local walk of this
            # rank's key range, all-to-all of the answers back to their slots
            keys, kbits = fk.morton_keys(tree, qs_dev, stream=stream)
            ex = MortonExchange(qs_dev, keys, kbits, world)
            local = []
            for (kind, k, _), o in zip(batches, opts):
                lm = ex.local_queries.shape[0]
                local.append((torch.empty(lm, dtype=torch.int32, device=dev),
                              torch.empty(lm * k, dtype=torch.int64, device=dev)))
            res = fk.run_batches_device(tree, [(ex.local_queries, c, h, o) for (c, h), o in zip(local, opts)],
                                        stream=stream, timings=timing)
            for (kind, k, _), (c, h) in zip(batches, local):
                rc, rh = ex.return_results(c, h, k)
                outs[(kind, k)][0].copy_(rc)
                outs[(kind, k)][1].copy_(rh)
            return [tm for _, tm in res]
        if args.serial:
            tms = []
            for (kind, k, _), o in zip(batches, opts):
                c, h = outs[(kind, k)]
                _, tm = fk.run_batch_device(tree, qs_dev, c, h, o, stream=stream, timings=timing)
                tms.append(tm)
            return tms
        res = fk.run_batches_device(tree, [(qs_dev, *outs[(kind, k)], o) for (kind, k, _), o in zip(batches, opts)],
                                    stream=stream, timings=timing)
        return [tm for _, tm in res]

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, walk_ms, launches = [], {b: [] for b in range(len(batches))}, 0
    sampler = ClockSampler(dev.index)
    with sampler:
        for _ in range(args.steps):
            flush.zero_()  # untimed L2 flush between timed steps
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            tms = step(True)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            for b, tm in enumerate(tms):
                walk_ms[b].append(tm["walk_ms"])
                launches += tm["launches"]
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t_step = max_over_ranks(sum(step_ms), dev) / args.steps / 1e3  # seconds, max over ranks
    m_total = WORKLOADS[args.workload][2] if strong else world * m
    value = len(batches) * m_total / t_step
    gpu_hashes = {}
    for kind, k, _ in batches:
        c, h = outs[(kind, k)]
        gpu_hashes[kind if kind == "fcp" else f"knn{k}"] = \
            f"{fk.result_hash(c.cpu().numpy(), h.cpu().numpy().view(fk.HIT_DTYPE), k):016x}"

    # ---- e2e through the host-buffer C ABI, same metric: H2D of the step's
    # queries, the walk and D2H of every result slot inside the timed region.
    # Pinned caller buffers (fkd_host_alloc) -> `e2e`; the drop-in as a
    # reference caller makes it (NumPy / std::vector, pageable) -> `e2e_pageable`.
    h2d = m * dim * 4 * (len(batches) if args.serial else 1)  # one upload per step when grouped
    # an unbounded-radius batch's counts are min(k, n) for every query: the
    # library writes them on the host (checked against the walked counts on
    # the device) and copies only the hits
    d2h = 0
    for kind, k, r in batches:
        d2h += (m * 4 if math.isfinite(r) else 0) + m * k * 8

    def host_buffers(pinned: bool):
        bufs = {}
        if pinned:
            hq = fk.LIB.fkd_host_alloc(qs_host.nbytes)
            C.memmove(hq, qs_host.ctypes.data, qs_host.nbytes)
            for kind, k, _ in batches:
                bufs[(kind, k)] = (fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * k * 8))
            return hq, bufs
        keep = [qs_host]
        for kind, k, _ in batches:
            c_arr, h_arr = np.empty(m, np.int32), np.empty(m * k, np.int64)
            c_arr.fill(0)  # pages touched, as a reference BatchResult's are (batch.cpp:82-86)
            h_arr.fill(-1)
            keep += [c_arr, h_arr]
            bufs[(kind, k)] = (c_arr.ctypes.data, h_arr.ctypes.data)
        bufs["keep"] = keep
        return qs_host.ctypes.data, bufs

    def e2e_run(pinned: bool) -> tuple[float, bool]:
        hq, bufs = host_buffers(pinned)

        arr = (fk._lib.fkd_host_batch * len(batches))()
        for i, ((kind, k, _), o) in enumerate(zip(batches, opts)):
            hc, hh = bufs[(kind, k)]
            arr[i].queries, arr[i].m, arr[i].dim, arr[i].opt = hq, m, dim, o.to_c()
            arr[i].counts, arr[i].hits, arr[i].stats = hc, hh, None

        def e2e_step():
            if args.serial:  # one fkd_run_batch call per batch
                for (kind, k, _), o in zip(batches, opts):
                    hc, hh = bufs[(kind, k)]
                    co = o.to_c()
                    rc = fk.LIB.fkd_run_batch(tree.handle, hq, m, dim, C.byref(co), hc, hh, None)
                    if rc != 0:
                        raise RuntimeError(fk.LIB.fkd_last_error().decode())
                return
            # one fkd_run_batches call: the step's batches share the query
            # array, so they run as one pipeline (one upload per chunk)
            rc = fk.LIB.fkd_run_batches(tree.handle, arr, len(batches))
            if rc != 0:
                raise RuntimeError(fk.LIB.fkd_last_error().decode())

        for _ in range(max(1, args.warmup)):
            e2e_step()
        if dist is not None:
            dist.barrier()
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            e2e_step()
            times.append(time.perf_counter() - t0)
        val = len(batches) * m_total / (max_over_ranks(sum(times), dev) / args.steps)
        # results of the e2e path must equal the device path (same queries)
        same = True
        for kind, k, _ in batches:
            hc, hh = bufs[(kind, k)]
            c, h = outs[(kind, k)]
            got_c = np.ctypeslib.as_array(C.cast(hc, C.POINTER(C.c_int32)), shape=(m,))
            got_h = np.ctypeslib.as_array(C.cast(hh, C.POINTER(C.c_int64)), shape=(m * k,))
            same &= bool(np.array_equal(got_c, c.cpu().numpy()))
            same &= bool(np.array_equal(got_h, h.view(torch.int64).cpu().numpy()))
        if pinned:
            for key, (hc, hh) in bufs.items():
                fk.LIB.fkd_host_free(hc)
                fk.LIB.fkd_host_free(hh)
            fk.LIB.fkd_host_free(hq)
        return val, same

    def e2e_pipelined_run(depth: int = 3) -> tuple[float, bool]:
        # a serving loop: step s+1 is submitted (fkd_submit_batches) before
        # step s is collected (fkd_wait), so one step's uploads and walks
        # overlap the previous step's result copies; every step still moves
        # its own queries in and results out (pinned, one buffer set per
        # job in flight)
        hq = fk.LIB.fkd_host_alloc(qs_host.nbytes)
        C.memmove(hq, qs_host.ctypes.data, qs_host.nbytes)
        sets = []
        for _ in range(depth):
            bufs = {(kind, k): (fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * k * 8)) for kind, k, _ in batches}
            arr = (fk._lib.fkd_host_batch * len(batches))()
            for i, ((kind, k, _), o) in enumerate(zip(batches, opts)):
                hc, hh = bufs[(kind, k)]
                arr[i].queries, arr[i].m, arr[i].dim, arr[i].opt = hq, m, dim, o.to_c()
                arr[i].counts, arr[i].hits, arr[i].stats = hc, hh, None
            sets.append((bufs, arr))

        def run(nsteps):
            pending = []
            for s_ in range(nsteps):
                h = C.c_void_p()
                if fk.LIB.fkd_submit_batches(tree.handle, sets[s_ % depth][1], len(batches), C.byref(h)) != 0:
                    raise RuntimeError(fk.LIB.fkd_last_error().decode())
                pending.append(h)
                if len(pending) == depth:
                    if fk.LIB.fkd_wait(pending.pop(0)) != 0:
                        raise RuntimeError(fk.LIB.fkd_last_error().decode())
            for h in pending:
                if fk.LIB.fkd_wait(h) != 0:
                    raise RuntimeError(fk.LIB.fkd_last_error().decode())

        # the first jobs in flight size their own workspaces (full-batch
        # device staging per concurrent job): warm up past that
        run(2 * depth + args.warmup)
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        run(args.steps)
        val = len(batches) * m_total / (max_over_ranks(time.perf_counter() - t0, dev) / args.steps)
        same = True
        for bufs, _ in sets:
            for kind, k, _ in batches:
                hc, hh = bufs[(kind, k)]
                c, h = outs[(kind, k)]
                same &= bool(np.array_equal(np.ctypeslib.as_array(C.cast(hc, C.POINTER(C.c_int32)), shape=(m,)),
                                            c.cpu().numpy()))
                same &= bool(np.array_equal(np.ctypeslib.as_array(C.cast(hh, C.POINTER(C.c_int64)), shape=(m * k,)),
                                            h.view(torch.int64).cpu().numpy()))
        for bufs, _ in sets:
            for hc, hh in bufs.values():
                fk.LIB.fkd_host_free(hc)
                fk.LIB.fkd_host_free(hh)
        fk.LIB.fkd_host_free(hq)
        return val, same

    e2e_value, e2e_parity = e2e_run(True)
    e2e_pg_value, e2e_pg_parity = e2e_run(False) if not args.no_pageable else (None, None)
    # the serving loop is for batches a server pipelines; two 1B-query C5
    # jobs in flight hold twice the full-batch staging and measured slower
    # than one (2.35 vs 2.93 G q/s, profiles/r02/r02bc_bench_c5.json)
    pipelined = not args.serial and m <= (1 << 27)
    e2e_pp_value, e2e_pp_parity = e2e_pipelined_run() if pipelined else (None, None)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # ---- roofline.  The step's batches run concurrently, so the walk kernels
    # of one batch share the SMs with the other's: the primary figure is the
    # whole step — every batch's algorithmic bytes over the step time (Morton
    # ordering included).  The dominant batch is also timed ALONE (untimed
    # serial calls after the timed region, CUDA events on its stream) for
    # the per-kernel fraction.
    peak, peak_src = measured_peaks()
    dom = max(range(len(batches)), key=lambda b: bytes_per_query(dim, pbar[batches[b][:2]],
                                                                    batches[b][1] if batches[b][0] == "knn" else 1))
    kind, k, r = batches[dom]
    stride = k if kind == "knn" else 1
    bq = bytes_per_query(dim, pbar[(kind, k)], stride)
    step_bytes = sum(m * bytes_per_query(dim, pbar[(kk, k2)], k2 if kk == "knn" else 1) for kk, k2, _ in batches)
    achieved = step_bytes / (sum(step_ms) / args.steps / 1e3) / 1e9
    alone = []
    c_d, h_d = outs[(kind, k)]
    for _ in range(5):
        flush.zero_()
        _, tm = fk.run_batch_device(tree, qs_dev, c_d, h_d, opts[dom], stream=stream, timings=True)
        alone.append(tm["walk_ms"])
    t_walk = float(np.median(alone)) / 1e3
    traffic = ncu_traffic(args.workload)
    issue = ncu_traffic(args.workload + "_issue")
    per_batch = {}
    for b, (kk, k2, r2) in enumerate(batches):
        name = kk if kk == "fcp" else f"knn{k2}"
        tw = float(np.mean(walk_ms[b])) / 1e3
        bpq = bytes_per_query(dim, pbar[(kk, k2)], k2 if kk == "knn" else 1)
        per_batch[name] = {"walk_ms_in_step": tw * 1e3, "P_bar": pbar[(kk, k2)],
                           "bytes_per_query": bpq, "result_hash": gpu_hashes[name]}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        sample = m if args.cpu_sample <= 0 else min(m, args.cpu_sample)
        cpu = cpu_baseline_leg(nodes_host, qs_host, batches, sample, gpu_hashes)

    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args.workload, world),
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "results_equal_device_path": bool(e2e_parity),
                "path": ("fkd_run_batch per batch" if args.serial else "one fkd_run_batches call per step (the "
                         "batches share the query array: one chunked pipeline, one upload)") +
                        " (C ABI, pinned host buffers from fkd_host_alloc, chunked H2D/walk/D2H; counts of "
                        "unbounded-radius batches written on the host, verified on the device)"},
        "gpu_launches": launches // args.steps,
        "gpu_launches_note": "own kernels per timed step (per batch: Morton keys, walk, continuation "
                             "rounds (fcp: 3), resume pass, CTA overflow pass); CUB sort kernels excluded",
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "the step's walk kernels (" + " + ".join(per_batch) + " batches, one concurrent "
                               "submission): algorithmic bytes of every batch / step time",
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_step": step_bytes},
        "roofline_dominant_alone": {
            "kernel": f"walk {kind}{'' if kind == 'fcp' else k} batch alone (walk + rounds + tail passes)",
            "achieved": m * bq / t_walk / 1e9, "peak": peak, "unit": "GB/s",
            "frac": m * bq / t_walk / 1e9 / peak, "walk_ms": t_walk * 1e3,
            "algorithmic_bytes_per_query": bq, "traffic": traffic,
            "timing": "median of 5 untimed single-batch calls after the timed region, CUDA events on its stream"},
        "issue_roofline": None if not issue else {
            "bound": "issue (warp instructions; the walk is ALU/issue-bound, see DESIGN.md §6)",
            "achieved": issue["knn8_warp_insts_per_launch"] / t_walk,
            "peak": 4 * torch.cuda.get_device_properties(dev).multi_processor_count * float(
                (sampler.summary().get("sm_mhz") or 1965.0)) * 1e6,
            "unit": "warp-instructions/s", "kernel": "walk knn8",
            "source": "instruction count per launch from profiles/traffic.json (ncu), time live"},
        "per_batch": per_batch,
        "partition": (args.partition if world > 1 else "single GPU"),
        "submission": ("serial: one fkd_run_batch_device call per batch" if args.serial else
                       "one fkd_run_batches_device call per step: the batches run concurrently (costliest at "
                       "the highest stream priority) and share one Morton order of the common query array"),
        "clocks": sampler.summary(),
        "native_libs": repo_native_libs(),
    }
    if e2e_pp_value is not None:
        line["e2e_pipelined"] = {"value": e2e_pp_value, "unit": "queries/s", "h2d_bytes_per_step": h2d,
                                 "d2h_bytes_per_step": d2h, "results_equal_device_path": bool(e2e_pp_parity),
                                 "path": "a serving loop over the same C ABI: fkd_submit_batches for step s+1 "
                                         "before fkd_wait for step s - 2 (3 jobs in flight, one pinned buffer set each); "
                                         "every step still uploads its queries and copies its results back"}
    if e2e_pg_value is not None:
        line["e2e_pageable"] = {"value": e2e_pg_value, "unit": "queries/s", "h2d_bytes_per_step": h2d,
                                "d2h_bytes_per_step": d2h, "results_equal_device_path": bool(e2e_pg_parity),
                                "path": "same call with NumPy (pageable) buffers, as flatkd::b200::run_batch "
                                        "passes a reference BatchResult's std::vectors"}
    if line.get("issue_roofline"):
        line["issue_roofline"]["frac"] = line["issue_roofline"]["achieved"] / line["issue_roofline"]["peak"]
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--cpu-sample", type=int, default=-1,
                    help="queries of the cpu_baseline leg (<=0: the whole batch; default: whole "
                         "batch up to 20M queries, else 10M)")
    ap.add_argument("--ref-sample", type=int, default=-1,
                    help="queries per batch of the reference arm (same rule as --cpu-sample)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pageable", action="store_true", help="skip the e2e_pageable measurement")
    ap.add_argument("--partition", choices=["block", "morton"], default="block",
                    help="multi-GPU query partition: contiguous blocks (no data-path collective) or Morton "
                         "key ranges (histogram all-reduce + two all-to-alls per step)")
    ap.add_argument("--serial", action="store_true",
                    help="submit the step's batches as back-to-back calls instead of one concurrent submission")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    m_rank = WORKLOADS[args.workload][2] // (int(os.environ.get("WORLD_SIZE", "1")) if args.workload == "c5" else 1)
    for attr in ("cpu_sample", "ref_sample"):  # whole batch where the host finishes it in seconds
        if getattr(args, attr) < 0:
            setattr(args, attr, 0 if m_rank <= 20_000_000 else 10_000_000)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
