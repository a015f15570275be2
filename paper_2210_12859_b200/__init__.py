"""B200-native stack-free k-d tree queries (arXiv 2210.12859), Python face.

A thin ctypes mirror of the reference's C++ query API
(``/root/reference/proj/include/flatkd/{batch,traverse,tree,point}.hpp``)
over the C ABI in ``include/fkd_b200.h``.  Every query is answered by the
sm_100a kernels in ``libfkd_b200.so``; there is no CPU fallback — without
the library this package raises on import, and without a GPU the query
entry points raise :class:`DeviceError`.

Reference mapping:

=============================  ===========================================
reference                      here
=============================  ===========================================
``flatkd::run_batch``          :func:`run_batch`     (batch.cpp:71-134)
``flatkd::fcp`` / ``knn``      :func:`fcp` / :func:`knn` (traverse.cpp:25-39)
``KdTree::from_level_order``   :meth:`KdTree.from_level_order` (tree.cpp:71-78)
``flatkd::build_tree``         :func:`build_tree`    (tree.cpp:80-89)
``BatchOptions``               :class:`BatchOptions` (batch.hpp:16-23)
``BatchResult``                :class:`BatchResult`  (batch.hpp:27-41)
``Hit`` / ``QueryStats``       :data:`HIT_DTYPE` / :class:`QueryStats`
``write_query_results``        :func:`write_query_results` (batch.cpp:136-158)
``random_points``              :func:`random_points` (rng.hpp:46-53)
``DataError``                  :class:`DataError`    (error.hpp:9-12)
``std::invalid_argument``      :class:`InvalidArgument` (a ``ValueError``)
=============================  ===========================================
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._lib import LIB, LIB_PATH, fkd_batch_options, fkd_device_batch, fkd_host_batch, fkd_query_stats, fkd_timings

__all__ = [
    "BatchOptions", "BatchResult", "DataError", "DeviceError", "Engine", "HIT_DTYPE",
    "InvalidArgument", "InvariantError", "KdTree", "QueryKind", "QueryStats", "build_tree",
    "build_level_order", "build_level_order_device", "clustered_points", "fcp", "knn", "random_points", "result_hash", "run_batch",
    "run_batch_device", "run_batches", "run_batches_device", "submit_batches", "Job", "morton_keys",
    "write_query_results", "LIB_PATH",
]

HIT_DTYPE = np.dtype([("node", "<i4"), ("dist2", "<f4")])  # flatkd::Hit, 8 bytes
INF = float("inf")

FLAG_MORTON = 0x1
FLAG_UNORDERED = 0x2
FLAG_NO_MORTON = 0x4


class DataError(RuntimeError):
    """flatkd::DataError — bad or inconsistent input (error.hpp:9-12)."""


class InvariantError(RuntimeError):
    """flatkd::InvariantError (error.hpp:15-18)."""


class InvalidArgument(ValueError):
    """std::invalid_argument (e.g. knn k < 1, batch.cpp:72-73)."""


class DeviceError(RuntimeError):
    """CUDA failure or no usable B200 — there is no CPU fallback."""


_STATUS = {1: InvalidArgument, 2: DataError, 3: InvariantError, 4: DeviceError, 5: DeviceError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = LIB.fkd_last_error().decode()
        raise _STATUS.get(rc, DeviceError)(msg)


class QueryKind(enum.IntEnum):
    fcp = 0
    knn = 1


class Engine(enum.IntEnum):
    stack_free = 0
    recursive = 1


@dataclass
class BatchOptions:
    """flatkd::BatchOptions (batch.hpp:16-23) + B200 switches."""

    kind: QueryKind = QueryKind.fcp
    k: int = 1
    max_radius: float = INF
    engine: Engine = Engine.stack_free
    threads: int = 0            # accepted, ignored on the GPU
    collect_stats: bool = False
    morton: bool = True         # walk in Morton order (results stay in input order)
    unordered: bool = False     # left-first child order

    def to_c(self) -> fkd_batch_options:
        o = fkd_batch_options()
        o.kind = int(self.kind)
        o.k = int(self.k)
        o.max_radius = float(self.max_radius)
        o.engine = int(self.engine)
        o.threads = int(self.threads)
        o.collect_stats = int(bool(self.collect_stats))
        flags = FLAG_MORTON if self.morton else FLAG_NO_MORTON
        if self.unordered:
            flags |= FLAG_UNORDERED
        o.flags = flags
        return o

    @property
    def stride(self) -> int:
        return int(self.k) if self.kind == QueryKind.knn else 1


@dataclass
class QueryStats:
    """flatkd::QueryStats (traverse.hpp:46-54)."""

    steps: int = 0
    nodes_visited: int = 0
    nodes_processed: int = 0

    @classmethod
    def from_c(cls, s: fkd_query_stats) -> "QueryStats":
        return cls(int(s.steps), int(s.nodes_visited), int(s.nodes_processed))


@dataclass
class BatchResult:
    """flatkd::BatchResult (batch.hpp:27-41): fixed-stride slots in input order."""

    stride: int
    counts: np.ndarray                   # int32[m]
    hits: np.ndarray                     # HIT_DTYPE[m * stride], empty slots {-1, inf}
    stats: QueryStats = field(default_factory=QueryStats)

    def hits_for(self, query: int) -> np.ndarray:
        base = query * self.stride
        return self.hits[base: base + int(self.counts[query])]

    def result_hash(self) -> int:
        return result_hash(self.counts, self.hits, self.stride)


def _f32(a, dim: Optional[int] = None) -> np.ndarray:
    arr = np.ascontiguousarray(a, dtype=np.float32)
    if arr.ndim == 1 and dim is not None:
        arr = arr.reshape(-1, dim) if arr.size else arr.reshape(0, dim)
    return arr


class KdTree:
    """Device-resident level-order tree (the reference's KdTree, tree.hpp:41-65,
    round-robin split policy).  Immutable; safe to share between threads."""

    def __init__(self, handle, n: int, dim: int, nodes: Optional[np.ndarray]):
        self._h = handle
        self._n = n
        self._dim = dim
        self._nodes = nodes

    @classmethod
    def from_level_order(cls, nodes, devices: Optional[Sequence[int]] = None) -> "KdTree":
        """Adopt a level-order array without reordering it (tree.cpp:71-78)."""
        arr = _f32(nodes)
        if arr.ndim != 2:
            raise DataError("point set: expected an (n, dim) array")
        n, dim = arr.shape
        h = C.c_void_p()
        if devices:
            devs = (C.c_int32 * len(devices))(*devices)
            _check(LIB.fkd_tree_create(arr.ctypes.data, n, dim, devs, len(devices), C.byref(h)))
        else:
            _check(LIB.fkd_tree_create(arr.ctypes.data, n, dim, None, 0, C.byref(h)))
        return cls(h, n, dim, arr)

    @classmethod
    def from_device(cls, tensor, stream=None) -> "KdTree":
        """Adopt a level-order torch CUDA tensor (n, dim) float32 (copied)."""
        if not tensor.is_cuda or tensor.dtype.itemsize != 4 or tensor.dim() != 2:
            raise DataError("expected a CUDA float32 (n, dim) tensor")
        t = tensor.contiguous()
        n, dim = t.shape
        h = C.c_void_p()
        _check(LIB.fkd_tree_create_device(C.c_void_p(t.data_ptr()), n, dim, _stream_ptr(stream),
                                          C.byref(h)))
        return cls(h, n, dim, None)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                LIB.fkd_tree_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def size(self) -> int:
        return self._n

    def dim(self) -> int:
        return self._dim

    def empty(self) -> bool:
        return self._n == 0

    def nodes(self) -> Optional[np.ndarray]:
        return self._nodes

    def replica_devices(self) -> List[int]:
        """CUDA devices holding a replica of the tree store (shard order)."""
        n = int(LIB.fkd_tree_replicas(self._h, None, 0))
        out = (C.c_int32 * max(n, 1))()
        LIB.fkd_tree_replicas(self._h, out, n)
        return [int(out[i]) for i in range(n)]

    def add_replicas(self, devices: Sequence[int]) -> None:
        """Replicate the tree store onto more devices, device to device
        (pipelined chain over NVLink / NVSwitch); they join the shard order."""
        devs = (C.c_int32 * max(len(devices), 1))(*devices)
        _check(LIB.fkd_tree_add_replicas(self._h, devs, len(devices)))

    def replica_device(self) -> Optional[int]:
        """The device fkd_run_batch_device runs on (the first replica)."""
        devs = self.replica_devices()
        return devs[0] if devs else None

    @property
    def handle(self):
        return self._h


def build_tree(points, devices: Optional[Sequence[int]] = None) -> KdTree:
    """flatkd::build_tree (tree.cpp:80-89) on the GPU (csrc/build.cu) + the
    device tree store: the unique left-balanced tree, byte-identical to the
    reference's.  ``tree.nodes()`` holds the level-order array."""
    arr = _f32(points)
    if arr.ndim != 2:
        raise DataError("point set: expected an (n, dim) array")
    n, dim = arr.shape
    out = np.empty_like(arr)
    h = C.c_void_p()
    devs = (C.c_int32 * len(devices))(*devices) if devices else None
    _check(LIB.fkd_tree_build(arr.ctypes.data, n, dim, devs, len(devices) if devices else 0,
                              out.ctypes.data, C.byref(h)))
    return KdTree(h, n, dim, out)


def build_level_order_device(points, out=None, stream=None):
    """GPU build from a CUDA float32 (n, dim) tensor; returns the level-order
    tensor (``out`` if given)."""
    import torch

    if not points.is_cuda or points.dtype != torch.float32 or points.dim() != 2:
        raise DataError("expected a CUDA float32 (n, dim) tensor")
    p = points.contiguous()
    if out is None:
        out = torch.empty_like(p)
    _check(LIB.fkd_build_tree_device(C.c_void_p(p.data_ptr()), p.shape[0], p.shape[1],
                                     C.c_void_p(out.data_ptr()), _stream_ptr(stream)))
    return out


def build_level_order(points) -> np.ndarray:
    """Host (multi-threaded CPU) builder: the reference's level-order array
    (byte-identical).  Needs no GPU; for large sets prefer build_tree()."""
    arr = _f32(points)
    if arr.ndim != 2:
        raise DataError("point set: expected an (n, dim) array")
    out = np.empty_like(arr)
    _check(LIB.fkd_build_tree(arr.ctypes.data, arr.shape[0], arr.shape[1], out.ctypes.data))
    return out


def run_batch(tree: KdTree, queries, options: Optional[BatchOptions] = None) -> BatchResult:
    """flatkd::run_batch (batch.cpp:71-134) on the GPU, host buffers in and out."""
    options = options or BatchOptions()
    if options.kind == QueryKind.knn and options.k < 1:  # batch.cpp:72-73, checked first
        raise InvalidArgument("knn: k must be >= 1")
    q = _f32(queries, tree.dim())
    if q.ndim != 2:
        raise DataError("queries: expected an (m, dim) array")
    m, dim = q.shape
    stride = options.stride
    counts = np.zeros(m, np.int32)
    hits = np.empty(m * stride, HIT_DTYPE)
    st = fkd_query_stats()
    o = options.to_c()
    _check(LIB.fkd_run_batch(tree.handle, q.ctypes.data, m, dim, C.byref(o), counts.ctypes.data,
                             hits.ctypes.data, C.byref(st)))
    return BatchResult(stride, counts, hits, QueryStats.from_c(st) if options.collect_stats else QueryStats())


def _prepare_batches(tree: KdTree, batches):
    """The fkd_host_batch array of run_batches / submit_batches, the arrays it
    points into (kept alive by the caller) and the per-batch result parts."""
    n = len(batches)
    arr = (fkd_host_batch * max(n, 1))()
    keep, results = [], []
    converted = {}
    for i, (queries, opt) in enumerate(batches):
        opt = opt or BatchOptions()
        if opt.kind == QueryKind.knn and opt.k < 1:  # batch.cpp:72-73, checked first
            raise InvalidArgument("knn: k must be >= 1")
        q = converted.get(id(queries))
        if q is None:
            q = converted[id(queries)] = _f32(queries, tree.dim())
        if q.ndim != 2:
            raise DataError("queries: expected an (m, dim) array")
        m, dim = q.shape
        counts = np.zeros(m, np.int32)
        hits = np.empty(m * opt.stride, HIT_DTYPE)
        st = fkd_query_stats()
        keep.append((q, counts, hits, st))
        results.append((opt, counts, hits, st))
        b = arr[i]
        b.queries, b.m, b.dim, b.opt = q.ctypes.data, m, dim, opt.to_c()
        b.counts, b.hits, b.stats = counts.ctypes.data, hits.ctypes.data, C.addressof(st)
    return arr, keep, results


def _batch_results(results) -> List[BatchResult]:
    return [BatchResult(opt.stride, c, h, QueryStats.from_c(st) if opt.collect_stats else QueryStats())
            for opt, c, h, st in results]


def run_batches(tree: KdTree, batches) -> List[BatchResult]:
    """Several host-buffer batches in one call (fkd_run_batches): ``batches``
    is a list of (queries, BatchOptions).  Batches over the same query array
    (the same object) run as one pipeline — the queries are uploaded, checked
    and ordered once per chunk and walked by every batch.  Returns one
    BatchResult per batch; raises on the first failing batch."""
    arr, keep, results = _prepare_batches(tree, batches)
    _check(LIB.fkd_run_batches(tree.handle, arr, len(batches)))
    return _batch_results(results)


class Job:
    """A submission in flight (fkd_submit_batches); ``wait()`` returns its
    BatchResults (or raises) once, and keeps the inputs alive until then."""

    def __init__(self, tree, handle, arr, keep, results):
        self._tree, self._handle, self._arr, self._keep, self._results = tree, handle, arr, keep, results

    def wait(self) -> List[BatchResult]:
        if self._handle is None:
            raise InvalidArgument("job already waited for")
        h, self._handle = self._handle, None
        _check(LIB.fkd_wait(h))
        return _batch_results(self._results)

    def __del__(self):
        if getattr(self, "_handle", None) is not None and LIB is not None:
            LIB.fkd_wait(self._handle)  # never leave the library thread writing freed arrays


def submit_batches(tree: KdTree, batches) -> Job:
    """run_batches without waiting (fkd_submit_batches): returns a Job at
    once; several jobs in flight on one tree overlap on the device (a serving
    loop submits batch i+1 before collecting batch i)."""
    arr, keep, results = _prepare_batches(tree, batches)
    h = C.c_void_p()
    _check(LIB.fkd_submit_batches(tree.handle, arr, len(batches), C.byref(h)))
    return Job(tree, h, arr, keep, results)


def _stream_ptr(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


def _check_device_batch(tree: KdTree, queries, counts, hits, options: BatchOptions, per_query=None):
    """The C ABI takes raw pointers: shapes, dtypes, layout and device are
    checked here so a wrong tensor raises instead of reading or writing out
    of bounds.  Returns (m, dim)."""
    import torch

    if options.kind == QueryKind.knn and options.k < 1:  # batch.cpp:72-73, checked first
        raise InvalidArgument("knn: k must be >= 1")
    if queries.dim() != 2:
        raise DataError("queries: expected an (m, dim) tensor")
    m, dim = int(queries.shape[0]), int(queries.shape[1])
    stride = options.stride
    checks = ((queries, torch.float32, m * dim, "queries"), (counts, torch.int32, m, "counts"),
              (hits, None, m * stride, "hits"))
    for t, dt, need, what in checks:
        if not t.is_cuda:
            raise DataError(f"{what}: expected a CUDA tensor")
        if not t.is_contiguous():
            raise DataError(f"{what}: expected a contiguous tensor")
        if dt is not None and t.dtype != dt:
            raise DataError(f"{what}: expected dtype {dt}, got {t.dtype}")
        elems = t.numel() if dt is not None else t.numel() * t.element_size() // 8
        if elems < need:
            raise DataError(f"{what}: holds {elems} elements, the batch needs {need}")
    if hits.element_size() not in (8, 4) or (hits.numel() * hits.element_size()) % 8:
        raise DataError("hits: expected 8-byte Hit slots (int64 / float64 / 2 x int32 per slot)")
    if per_query is not None and (not per_query.is_cuda or not per_query.is_contiguous()
                                  or per_query.numel() * per_query.element_size() < 24 * m):
        raise DataError("per_query: expected a contiguous CUDA tensor of m x 24 bytes")
    dev = queries.device
    for t in (counts, hits) + ((per_query,) if per_query is not None else ()):
        if t.device != dev:
            raise DataError("queries, counts, hits and per_query must be on one device")
    if tree.replica_device() is not None and dev.index != tree.replica_device():
        raise DataError(f"queries are on cuda:{dev.index}, the tree's first replica on "
                        f"cuda:{tree.replica_device()}")
    return m, dim


def _timings_dict(tm: fkd_timings) -> dict:
    return {"order_ms": tm.order_ms, "walk_ms": tm.walk_ms, "tail_ms": tm.tail_ms, "launches": tm.launches,
            "walk_launches": tm.walk_launches, "overflowed": tm.overflowed}


def run_batch_device(tree: KdTree, queries, counts, hits, options: Optional[BatchOptions] = None,
                     stream=None, per_query=None, timings: bool = False):
    """Device-resident batch: torch CUDA tensors in and out, launched on `stream`
    (default: torch's current stream).  Returns (QueryStats, timings dict|None)."""
    import torch

    options = options or BatchOptions()
    m, dim = _check_device_batch(tree, queries, counts, hits, options, per_query)
    if stream is None:
        stream = torch.cuda.current_stream(queries.device)
    st = fkd_query_stats()
    tm = fkd_timings()
    o = options.to_c()
    _check(LIB.fkd_run_batch_device(
        tree.handle, C.c_void_p(queries.data_ptr()), m, dim, C.byref(o),
        C.c_void_p(counts.data_ptr()), C.c_void_p(hits.data_ptr()),
        C.byref(st) if options.collect_stats else None,
        C.c_void_p(per_query.data_ptr()) if per_query is not None else None,
        _stream_ptr(stream), C.byref(tm) if timings else None))
    return QueryStats.from_c(st), (_timings_dict(tm) if timings else None)


def run_batches_device(tree: KdTree, batches, stream=None, timings: bool = False):
    """Several independent device batches in one submission
    (fkd_run_batches_device): ``batches`` is a list of (queries, counts,
    hits, BatchOptions); each runs exactly as run_batch_device would, all
    concurrently (the costliest on the highest-priority stream).  Returns a
    list of (QueryStats, timings dict|None); raises on the first failing batch."""
    import torch

    n = len(batches)
    arr = (fkd_device_batch * max(n, 1))()
    keep = []
    for i, (q, c, h, opt) in enumerate(batches):
        opt = opt or BatchOptions()
        m, dim = _check_device_batch(tree, q, c, h, opt)
        st, tm = fkd_query_stats(), fkd_timings()
        keep.append((st, tm, opt))
        b = arr[i]
        b.d_queries, b.m, b.dim, b.opt = q.data_ptr(), m, dim, opt.to_c()
        b.d_counts, b.d_hits = c.data_ptr(), h.data_ptr()
        b.stats = C.addressof(st) if opt.collect_stats else None
        b.d_per_query = None
        b.timings = C.addressof(tm) if timings else None
    if stream is None and n:
        stream = torch.cuda.current_stream(batches[0][0].device)
    _check(LIB.fkd_run_batches_device(tree.handle, arr, n, _stream_ptr(stream)))
    return [(QueryStats.from_c(st), _timings_dict(tm) if timings else None) for st, tm, _ in keep]


def morton_keys(tree: KdTree, queries, stream=None):
    """Morton keys of device queries over the tree's bounding box (the batch
    ordering's key at full resolution) -> (uint32-valued int64 tensor, key
    bits); the multi-GPU Morton-range partition splits batches by them."""
    import torch

    if not queries.is_cuda or queries.dtype != torch.float32 or queries.dim() != 2 or not queries.is_contiguous():
        raise DataError("queries: expected a contiguous CUDA float32 (m, dim) tensor")
    m, dim = queries.shape
    keys = torch.empty(m, dtype=torch.int32, device=queries.device)
    bits = C.c_int32(0)
    if stream is None:
        stream = torch.cuda.current_stream(queries.device)
    _check(LIB.fkd_morton_keys(tree.handle, C.c_void_p(queries.data_ptr()), m, dim, C.c_void_p(keys.data_ptr()),
                               C.byref(bits), _stream_ptr(stream)))
    return keys.to(torch.int64) & 0xFFFFFFFF, int(bits.value)


def fcp(tree: KdTree, query, max_radius: float = INF, stats: bool = False):
    """Closest stored point within max_radius (inclusive), or None (traverse.cpp:25-30).
    Returns (node, dist2) or None; with stats=True returns (hit, QueryStats)."""
    q = _f32(query).reshape(-1)
    out = np.empty(1, HIT_DTYPE)
    cnt = C.c_int32(0)
    st = fkd_query_stats()
    _check(LIB.fkd_fcp(tree.handle, q.ctypes.data, len(q), C.c_float(max_radius), out.ctypes.data,
                       C.byref(cnt), C.byref(st) if stats else None))
    hit = (int(out[0]["node"]), float(out[0]["dist2"])) if cnt.value else None
    return (hit, QueryStats.from_c(st)) if stats else hit


def knn(tree: KdTree, query, k: int, max_radius: float = INF, stats: bool = False):
    """Up to k nearest within max_radius, ascending by (dist2, node) (traverse.cpp:32-39)."""
    q = _f32(query).reshape(-1)
    out = np.empty(max(int(k), 1), HIT_DTYPE)
    cnt = C.c_int32(0)
    st = fkd_query_stats()
    _check(LIB.fkd_knn(tree.handle, q.ctypes.data, len(q), int(k), C.c_float(max_radius),
                       out.ctypes.data, C.byref(cnt), C.byref(st) if stats else None))
    hits = [(int(h["node"]), float(h["dist2"])) for h in out[: cnt.value]]
    return (hits, QueryStats.from_c(st)) if stats else hits


def result_hash(counts, hits, stride: int) -> int:
    """BatchResult::result_hash (batch.cpp:30-48)."""
    c = np.ascontiguousarray(counts, np.int32)
    h = np.ascontiguousarray(hits, HIT_DTYPE)
    return int(LIB.fkd_result_hash(c.ctypes.data, h.ctypes.data, len(c), int(stride)))


def _format_float(v: np.float32) -> str:
    # io::format_float: "%.9g" (io.cpp:163-167); sqrt in float (traverse.hpp:74)
    f = float(v)
    if math.isinf(f):
        return "inf" if f > 0 else "-inf"
    if math.isnan(f):
        return "nan"
    return "%.9g" % f


def write_query_results(result: BatchResult) -> str:
    """Text form of write_query_results (batch.cpp:136-158)."""
    lines = []
    for qi in range(len(result.counts)):
        hs = result.hits_for(qi)
        dist = np.sqrt(hs["dist2"].astype(np.float32))
        if result.stride == 1:
            lines.append("-1,inf" if len(hs) == 0 else f"{int(hs[0]['node'])},{_format_float(dist[0])}")
        else:
            parts = [str(len(hs))]
            for h, d in zip(hs, dist):
                parts.append(str(int(h["node"])))
                parts.append(_format_float(d))
            lines.append(",".join(parts))
    return "".join(line + "\n" for line in lines)


def random_points(seed: int, stream: int, count: int, dim: int) -> np.ndarray:
    """random_points(derive_stream_seed(seed, stream), count, dim) (rng.hpp:26-53)."""
    out = np.empty(count * dim, np.float32)
    _check(LIB.fkd_random_points(seed, stream, count, dim, out.ctypes.data))
    return out.reshape(count, dim)


def clustered_points(seed: int, stream: int, count: int, dim: int, blobs: int = 64,
                     sigma: float = 0.02) -> np.ndarray:
    """Gaussian blobs (SURVEY §8(d) C3 workload; no reference counterpart)."""
    out = np.empty(count * dim, np.float32)
    _check(LIB.fkd_clustered_points(seed, stream, count, dim, blobs, C.c_float(sigma),
                                    out.ctypes.data))
    return out.reshape(count, dim)


# ---------------------------------------------------------------- debugging

STATS_DTYPE = np.dtype([("steps", "<i8"), ("nodes_visited", "<i8"), ("nodes_processed", "<i8")])


def trace(tree: KdTree, queries, kind: QueryKind = QueryKind.fcp, k: int = 1,
          max_radius: float = INF, cap: int = 4096):
    """Device trace of each query's walk (traverse.hpp:56-68): returns
    (counts, hits, stats, events) where events[i] lists node ids processed
    (>= 0) and ~node for bounces, exactly as flatkd's Trace records them."""
    q = _f32(queries, tree.dim())
    m, dim = q.shape
    kk = int(k) if kind == QueryKind.knn else 1
    counts = np.zeros(m, np.int32)
    hits = np.empty(m * kk, HIT_DTYPE)
    stats = np.zeros(m, STATS_DTYPE)
    ev = np.zeros(max(m * cap, 1), np.int32)
    lens = np.zeros(m, np.int64)
    _check(LIB.fkd_trace_batch(tree.handle, q.ctypes.data, m, dim, int(kind), int(k), C.c_float(max_radius),
                               counts.ctypes.data, hits.ctypes.data, stats.ctypes.data, ev.ctypes.data,
                               cap, lens.ctypes.data))
    events = [ev[i * cap: i * cap + min(int(lens[i]), cap)].copy() for i in range(m)]
    return counts, hits, stats, events


# ---------------------------------------------------------------- files

def write_points_file(path: str, points, tree: bool = False) -> None:
    """io::write_points / write_tree, binary format (io.cpp:50-99)."""
    arr = _f32(points)
    _check(LIB.fkd_write_file(path.encode(), int(tree), arr.ctypes.data, arr.shape[0], arr.shape[1]))


def read_points_file_device(path: str, tree: bool = False, device=None):
    """Binary points/tree file straight into a CUDA tensor (no host copy)."""
    import torch

    n = C.c_int64(0)
    d = C.c_int32(0)
    _check(LIB.fkd_file_info(path.encode(), int(tree), C.byref(n), C.byref(d)))
    out = torch.empty((n.value, d.value), dtype=torch.float32, device=device or "cuda")
    _check(LIB.fkd_read_file_device(path.encode(), int(tree), C.c_void_p(out.data_ptr()), n.value,
                                    C.byref(n), C.byref(d), None))
    return out


def load_tree(path: str, devices: Optional[Sequence[int]] = None) -> KdTree:
    """io::read_tree + KdTree::from_level_order onto the device(s)."""
    h = C.c_void_p()
    devs = (C.c_int32 * len(devices))(*devices) if devices else None
    _check(LIB.fkd_tree_load(path.encode(), devs, len(devices) if devices else 0, C.byref(h)))
    return KdTree(h, int(LIB.fkd_tree_size(h)), int(LIB.fkd_tree_dim(h)), None)
