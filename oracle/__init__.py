"""ctypes faces of the two CPU checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product
(``paper_2210_12859_b200``) never imports it and never falls back to it.

* :class:`Oracle`    — ``_build/libfkd_oracle.so``: the C restatement
  (``fkd_oracle.c``) of the reference's query path, each function citing the
  reference file:line it follows.
* :class:`Reference` — ``_ref/libflatkd_ref.so``: the UNMODIFIED reference
  sources (``/root/reference/proj``) compiled by ``oracle/Makefile``, driven
  through ``ref_capi.cpp``.  Present wherever ``build()`` ran in a container
  that had ``/root/reference``; the built ``.so`` travels to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libfkd_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libflatkd_ref.so")
REF_SRC = os.environ.get("FKD_REFERENCE_DIR", "/root/reference/proj")

HIT_DTYPE = np.dtype([("node", "<i4"), ("dist2", "<f4")])
STATS_DTYPE = np.dtype([("steps", "<i8"), ("nodes_visited", "<i8"), ("nodes_processed", "<i8")])

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_hitp = np.ctypeslib.ndpointer(dtype=HIT_DTYPE, flags="C_CONTIGUOUS")
_statp = np.ctypeslib.ndpointer(dtype=STATS_DTYPE, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def build(reference: bool = True) -> None:
    """Compile the checkers (make -C oracle).  The reference library is only
    (re)built when its sources exist (this container, not the GPU box)."""
    targets = ["oracle"]
    if reference and os.path.isdir(REF_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, f"REF={REF_SRC}", *targets], check=True)


def _null_or(arr):
    return None if arr is None else arr


class Oracle:
    """The C restatement (fkd_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run oracle.build()")
        L = self.lib = C.CDLL(path)
        L.fko_last_error.restype = C.c_char_p
        L.fko_derive_stream_seed.restype = C.c_uint64
        L.fko_derive_stream_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.fko_random_points.argtypes = [C.c_uint64, C.c_int64, C.c_int, _f32p]
        L.fko_rng_state_size.restype = C.c_int
        L.fko_mt_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.fko_mt_next.restype = C.c_uint64
        L.fko_mt_next.argtypes = [C.c_void_p]
        L.fko_mt_next_int.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.fko_mt_chance.argtypes = [C.c_void_p, C.c_double]
        L.fko_mt_float01.restype = C.c_float
        L.fko_mt_float01.argtypes = [C.c_void_p]
        L.fko_random_point_set.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, _f32p]
        L.fko_random_query.argtypes = [C.c_void_p, C.c_int, _f32p, C.c_int, _f32p]
        L.fko_left_subtree_size.argtypes = [C.c_int]
        L.fko_build_tree.argtypes = [_f32p, C.c_int, C.c_int, _f32p]
        L.fko_verify_tree.argtypes = [_f32p, C.c_int, C.c_int]
        L.fko_query.argtypes = [_f32p, C.c_int, C.c_int, _f32p, C.c_int, C.c_int, C.c_float,
                                C.c_int, _hitp, C.POINTER(C.c_int), C.c_void_p, C.c_void_p,
                                C.c_int64, C.POINTER(C.c_int64)]
        L.fko_run_batch.argtypes = [_f32p, C.c_int, C.c_int, _f32p, C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.c_float, C.c_int, C.c_int, _i32p, _hitp,
                                    C.c_void_p, C.c_void_p]
        L.fko_brute_batch.argtypes = [_f32p, C.c_int, C.c_int, _f32p, C.c_int, C.c_int, C.c_int,
                                      C.c_float, _i32p, _hitp]
        L.fko_result_hash.restype = C.c_uint64
        L.fko_result_hash.argtypes = [_i32p, _hitp, C.c_int64, C.c_int]

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.lib.fko_last_error().decode())

    # --- generators ---
    def derive_stream_seed(self, master: int, stream: int) -> int:
        return self.lib.fko_derive_stream_seed(master, stream)

    def random_points(self, seed: int, count: int, dim: int) -> np.ndarray:
        out = np.empty(count * dim, np.float32)
        self.lib.fko_random_points(seed, count, dim, out)
        return out.reshape(count, dim)

    def instance_rng(self, seed: int) -> "InstanceRng":
        return InstanceRng(self, seed)

    # --- tree ---
    def left_subtree_size(self, n: int) -> int:
        return self.lib.fko_left_subtree_size(n)

    def build_tree(self, points: np.ndarray) -> np.ndarray:
        pts = np.ascontiguousarray(points, np.float32)
        n, dim = pts.shape
        out = np.empty_like(pts)
        self._check(self.lib.fko_build_tree(pts.reshape(-1), n, dim, out.reshape(-1)))
        return out

    def verify_tree(self, nodes: np.ndarray) -> bool:
        nodes = np.ascontiguousarray(nodes, np.float32)
        return bool(self.lib.fko_verify_tree(nodes.reshape(-1), nodes.shape[0], nodes.shape[1]))

    # --- queries ---
    def query(self, nodes, q, kind="fcp", k=1, max_radius=float("inf"), recursive=False,
              trace_cap=0):
        nodes = np.ascontiguousarray(nodes, np.float32)
        n, dim = nodes.shape if nodes.ndim == 2 else (0, len(q))
        q = np.ascontiguousarray(q, np.float32)
        kk = k if kind == "knn" else 1
        hits = np.empty(max(kk, 1), HIT_DTYPE)
        cnt = C.c_int(0)
        st = np.zeros(1, STATS_DTYPE)
        tr = np.zeros(max(trace_cap, 1), np.int32)
        tlen = C.c_int64(0)
        self._check(self.lib.fko_query(nodes.reshape(-1), n, dim, q, int(kind == "knn"), k,
                                       max_radius, int(recursive), hits, C.byref(cnt),
                                       st.ctypes.data, tr.ctypes.data if trace_cap else None,
                                       trace_cap, C.byref(tlen)))
        return hits[: cnt.value].copy(), st[0], (tr[: tlen.value].copy() if trace_cap else None)

    def run_batch(self, nodes, queries, kind="fcp", k=1, max_radius=float("inf"),
                  recursive=False, threads=0, per_query=False):
        nodes = np.ascontiguousarray(nodes, np.float32)
        queries = np.ascontiguousarray(queries, np.float32)
        n, tdim = nodes.shape
        m, qdim = queries.shape
        stride = k if kind == "knn" else 1
        counts = np.zeros(m, np.int32)
        hits = np.empty(max(m * stride, 1), HIT_DTYPE)
        tot = np.zeros(1, STATS_DTYPE)
        pq = np.zeros(max(m, 1), STATS_DTYPE) if per_query else None
        self._check(self.lib.fko_run_batch(nodes.reshape(-1), n, tdim, queries.reshape(-1), m, qdim,
                                           int(kind == "knn"), k, max_radius, int(recursive),
                                           threads, counts, hits, tot.ctypes.data,
                                           pq.ctypes.data if pq is not None else None))
        return counts, hits[: m * stride], tot[0], (pq[:m] if pq is not None else None)

    def brute_batch(self, points, queries, kind="fcp", k=1, max_radius=float("inf")):
        points = np.ascontiguousarray(points, np.float32)
        queries = np.ascontiguousarray(queries, np.float32)
        n, dim = points.shape
        m = queries.shape[0]
        stride = k if kind == "knn" else 1
        counts = np.zeros(m, np.int32)
        hits = np.empty(max(m * stride, 1), HIT_DTYPE)
        self._check(self.lib.fko_brute_batch(points.reshape(-1), n, dim, queries.reshape(-1), m,
                                             int(kind == "knn"), k, max_radius, counts, hits))
        return counts, hits[: m * stride]

    def result_hash(self, counts, hits, stride) -> int:
        counts = np.ascontiguousarray(counts, np.int32)
        hits = np.ascontiguousarray(hits, HIT_DTYPE)
        if hits.size == 0:
            hits = np.empty(1, HIT_DTYPE)
        return self.lib.fko_result_hash(counts, hits, len(counts), stride)


class InstanceRng:
    """testing::InstanceRng restated (instancegen.hpp:16-27)."""

    def __init__(self, oracle: Oracle, seed: int):
        self.o = oracle
        self.state = C.create_string_buffer(oracle.lib.fko_rng_state_size())
        oracle.lib.fko_mt_seed(self.state, seed)

    def next_u64(self) -> int:
        return self.o.lib.fko_mt_next(self.state)

    def next_int(self, lo: int, hi: int) -> int:
        return self.o.lib.fko_mt_next_int(self.state, lo, hi)

    def next_float01(self) -> float:
        return self.o.lib.fko_mt_float01(self.state)

    def chance(self, p: float) -> bool:
        return bool(self.o.lib.fko_mt_chance(self.state, p))

    def random_point_set(self, n: int, dim: int, grid: int = 0, dup_fraction: float = 0.0):
        out = np.empty(max(n * dim, 1), np.float32)
        self.o.lib.fko_random_point_set(self.state, n, dim, grid, dup_fraction, out)
        return out[: n * dim].reshape(n, dim)

    def random_query(self, dim: int, points: np.ndarray) -> np.ndarray:
        pts = np.ascontiguousarray(points, np.float32).reshape(-1)
        if pts.size == 0:
            pts = np.zeros(1, np.float32)
        out = np.empty(dim, np.float32)
        self.o.lib.fko_random_query(self.state, dim, pts, points.shape[0], out)
        return out


class Reference:
    """The unmodified reference library (oracle/_ref/libflatkd_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run oracle.build() where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.fkr_last_error.restype = C.c_char_p
        L.fkr_random_points.argtypes = [C.c_uint64, C.c_longlong, C.c_int, _f32p]
        L.fkr_derive_stream_seed.restype = C.c_uint64
        L.fkr_derive_stream_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.fkr_build_tree.argtypes = [_f32p, C.c_longlong, C.c_int, _f32p]
        L.fkr_verify_tree.argtypes = [_f32p, C.c_longlong, C.c_int]
        L.fkr_left_subtree_size.argtypes = [C.c_int]
        L.fkr_run_batch.argtypes = [_f32p, C.c_longlong, C.c_int, _f32p, C.c_longlong, C.c_int,
                                    C.c_int, C.c_int, C.c_float, C.c_int, C.c_int, C.c_int,
                                    _i32p, _hitp, C.c_void_p, C.POINTER(C.c_double)]
        L.fkr_result_hash.restype = C.c_uint64
        L.fkr_result_hash.argtypes = [_i32p, _hitp, C.c_longlong, C.c_int]
        L.fkr_write_results.restype = C.c_size_t
        L.fkr_write_results.argtypes = [_i32p, _hitp, C.c_longlong, C.c_int, C.c_char_p, C.c_size_t]
        L.fkr_query.argtypes = [_f32p, C.c_longlong, C.c_int, _f32p, C.c_int, C.c_int, C.c_float,
                                _hitp, C.POINTER(C.c_int), C.c_void_p, C.c_void_p, C.c_longlong,
                                C.POINTER(C.c_longlong)]
        L.fkr_brute.argtypes = [_f32p, C.c_longlong, C.c_int, _f32p, C.c_int, C.c_int, C.c_float,
                                _hitp, C.POINTER(C.c_int)]
        L.fkr_instance_rng_new.restype = C.c_void_p
        L.fkr_instance_rng_new.argtypes = [C.c_uint64]
        L.fkr_instance_rng_free.argtypes = [C.c_void_p]
        L.fkr_instance_rng_u64.restype = C.c_uint64
        L.fkr_instance_rng_u64.argtypes = [C.c_void_p]
        L.fkr_random_point_set.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, _f32p]
        L.fkr_random_query.argtypes = [C.c_void_p, C.c_int, _f32p, C.c_int, _f32p]
        for fn in ("fkr_trace_suite", "fkr_oracle_suite"):
            getattr(L, fn).restype = C.c_longlong
            getattr(L, fn).argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_longlong)]
        L.fkr_structure_suite.restype = C.c_longlong
        L.fkr_structure_suite.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_longlong)]
        L.fkr_hardware_threads.restype = C.c_int
        L.fkr_write_file.argtypes = [C.c_char_p, C.c_int, _f32p, C.c_longlong, C.c_int]
        L.fkr_read_file.argtypes = [C.c_char_p, C.c_int, _f32p, C.c_longlong, C.POINTER(C.c_longlong),
                                    C.POINTER(C.c_int)]
        L.fkr_layout.argtypes = [C.POINTER(C.c_int)]
        L.fkr_clustered_points.argtypes = [C.c_uint64, C.c_uint64, C.c_longlong, C.c_int, C.c_int,
                                           C.c_float, _f32p]
        L.fkr_bench_matrix_csv.restype = C.c_longlong
        L.fkr_bench_matrix_csv.argtypes = [C.c_longlong, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                           C.c_int, C.c_char_p, C.c_longlong]

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.lib.fkr_last_error().decode())

    def last_error(self) -> str:
        return self.lib.fkr_last_error().decode()

    def write_file(self, path: str, points, tree: bool = False) -> None:
        pts = np.ascontiguousarray(points, np.float32)
        self._check(self.lib.fkr_write_file(path.encode(), int(tree), pts.reshape(-1) if pts.size else
                                            np.zeros(1, np.float32), pts.shape[0], pts.shape[1]))

    def read_file(self, path: str, tree: bool = False, cap_floats: int = 1 << 26) -> np.ndarray:
        out = np.empty(cap_floats, np.float32)
        n = C.c_longlong(0)
        d = C.c_int(0)
        self._check(self.lib.fkr_read_file(path.encode(), int(tree), out, cap_floats, C.byref(n), C.byref(d)))
        return out[: n.value * d.value].reshape(n.value, d.value)

    def hardware_threads(self) -> int:
        return self.lib.fkr_hardware_threads()

    def layout(self):
        out = (C.c_int * 5)()
        self.lib.fkr_layout(out)
        return list(out)

    def random_points(self, seed: int, count: int, dim: int) -> np.ndarray:
        out = np.empty(max(count * dim, 1), np.float32)
        self._check(self.lib.fkr_random_points(seed, count, dim, out))
        return out[: count * dim].reshape(count, dim)

    def derive_stream_seed(self, master: int, stream: int) -> int:
        return self.lib.fkr_derive_stream_seed(master, stream)

    def stream_points(self, master: int, stream: int, count: int, dim: int) -> np.ndarray:
        """random_points(derive_stream_seed(master, stream), count, dim) (rng.hpp:26-53)."""
        return self.random_points(self.derive_stream_seed(master, stream), count, dim)

    def clustered_points(self, master: int, stream: int, count: int, dim: int, blobs: int = 64,
                         sigma: float = 0.02) -> np.ndarray:
        """The C3 Gaussian-blob workload on the reference's RNG (ref_capi.cpp)."""
        out = np.empty(max(count * dim, 1), np.float32)
        self._check(self.lib.fkr_clustered_points(master, stream, count, dim, blobs, sigma, out))
        return out[: count * dim].reshape(count, dim)

    def bench_matrix_csv(self, n_queries: int, k_dim: int, kind: str, reps: int, n_list,
                         k_list=(8,), r_list=(float("inf"),), threads: int = 0) -> str:
        """flatkd::run_bench_matrix + write_bench_csv (bench.cpp:64-133), seed 1."""
        n_arr = (C.c_longlong * len(n_list))(*n_list)
        k_arr = (C.c_int * len(k_list))(*k_list)
        r_arr = (C.c_float * len(r_list))(*r_list)
        args = (n_queries, k_dim, int(kind == "knn"), reps, threads, n_arr, len(n_list), k_arr,
                len(k_list), r_arr, len(r_list))
        size = self.lib.fkr_bench_matrix_csv(*args, None, 0)
        if size < 0:
            raise OracleError(9, self.last_error())
        buf = C.create_string_buffer(size + 1)
        self.lib.fkr_bench_matrix_csv(*args, buf, size + 1)
        return buf.value.decode()

    def build_tree(self, points: np.ndarray) -> np.ndarray:
        pts = np.ascontiguousarray(points, np.float32)
        out = np.empty_like(pts)
        n, dim = pts.shape
        self._check(self.lib.fkr_build_tree(pts.reshape(-1), n, dim, out.reshape(-1)))
        return out

    def run_batch(self, nodes, queries, kind="fcp", k=1, max_radius=float("inf"), engine=0,
                  threads=0, collect_stats=False):
        """Returns (counts, hits, stats3, seconds_inside_run_batch)."""
        nodes = np.ascontiguousarray(nodes, np.float32)
        queries = np.ascontiguousarray(queries, np.float32)
        n, tdim = nodes.shape
        m, qdim = queries.shape
        stride = k if kind == "knn" else 1
        counts = np.zeros(max(m, 1), np.int32)
        hits = np.empty(max(m * stride, 1), HIT_DTYPE)
        st = np.zeros(3, np.int64)
        secs = C.c_double(0.0)
        self._check(self.lib.fkr_run_batch(nodes.reshape(-1), n, tdim, queries.reshape(-1), m, qdim,
                                           int(kind == "knn"), k, max_radius, engine, threads,
                                           int(collect_stats), counts, hits, st.ctypes.data,
                                           C.byref(secs)))
        return counts[:m], hits[: m * stride], st, secs.value

    def result_hash(self, counts, hits, stride) -> int:
        counts = np.ascontiguousarray(counts, np.int32)
        hits = np.ascontiguousarray(hits, HIT_DTYPE)
        if counts.size == 0:
            counts = np.zeros(1, np.int32)[:0]
        return self.lib.fkr_result_hash(np.ascontiguousarray(counts) if counts.size else np.zeros(1, np.int32),
                                        hits if hits.size else np.empty(1, HIT_DTYPE),
                                        len(counts), stride)

    def write_results(self, counts, hits, stride) -> str:
        counts = np.ascontiguousarray(counts, np.int32)
        hits = np.ascontiguousarray(hits, HIT_DTYPE)
        size = self.lib.fkr_write_results(counts, hits, len(counts), stride, None, 0)
        buf = C.create_string_buffer(size + 1)
        self.lib.fkr_write_results(counts, hits, len(counts), stride, buf, size + 1)
        return buf.value.decode()

    def query(self, nodes, q, kind="fcp", k=1, max_radius=float("inf"), trace_cap=0):
        nodes = np.ascontiguousarray(nodes, np.float32)
        n, dim = nodes.shape
        q = np.ascontiguousarray(q, np.float32)
        hits = np.empty(max(k, 1), HIT_DTYPE)
        cnt = C.c_int(0)
        st = np.zeros(3, np.int64)
        tr = np.zeros(max(trace_cap, 1), np.int32)
        tlen = C.c_longlong(0)
        self._check(self.lib.fkr_query(nodes.reshape(-1) if n else np.zeros(1, np.float32), n, dim,
                                       q, int(kind == "knn"), k, max_radius, hits, C.byref(cnt),
                                       st.ctypes.data, tr.ctypes.data, trace_cap, C.byref(tlen)))
        return hits[: cnt.value].copy(), st, tr[: min(tlen.value, trace_cap)].copy()

    def brute(self, points, q, kind="fcp", k=1, max_radius=float("inf")):
        points = np.ascontiguousarray(points, np.float32)
        n, dim = points.shape
        hits = np.empty(max(k, 1), HIT_DTYPE)
        cnt = C.c_int(0)
        self._check(self.lib.fkr_brute(points.reshape(-1) if n else np.zeros(1, np.float32), n, dim,
                                       np.ascontiguousarray(q, np.float32), int(kind == "knn"), k,
                                       max_radius, hits, C.byref(cnt)))
        return hits[: cnt.value].copy()

    def instance_rng(self, seed: int) -> "RefInstanceRng":
        return RefInstanceRng(self, seed)

    def trace_suite(self, seed=1, instances=1000, max_n=1024, qpt=20):
        out = C.c_longlong(0)
        fails = self.lib.fkr_trace_suite(seed, instances, max_n, qpt, C.byref(out))
        return fails, out.value, self.last_error()

    def oracle_suite(self, seed=1, instances=1000, max_n=1024, qpt=20):
        out = C.c_longlong(0)
        fails = self.lib.fkr_oracle_suite(seed, instances, max_n, qpt, C.byref(out))
        return fails, out.value, self.last_error()

    def structure_suite(self, max_shape_n=1024, sweep_n=100000):
        out = C.c_longlong(0)
        fails = self.lib.fkr_structure_suite(max_shape_n, sweep_n, C.byref(out))
        return fails, out.value, self.last_error()


class RefInstanceRng:
    def __init__(self, ref: Reference, seed: int):
        self.r = ref
        self.h = ref.lib.fkr_instance_rng_new(seed)

    def __del__(self):
        try:
            self.r.lib.fkr_instance_rng_free(self.h)
        except Exception:
            pass

    def next_u64(self) -> int:
        return self.r.lib.fkr_instance_rng_u64(self.h)

    def random_point_set(self, n, dim, grid=0, dup_fraction=0.0):
        out = np.empty(max(n * dim, 1), np.float32)
        self.r._check(self.r.lib.fkr_random_point_set(self.h, n, dim, grid, dup_fraction, out))
        return out[: n * dim].reshape(n, dim)

    def random_query(self, dim, points):
        pts = np.ascontiguousarray(points, np.float32).reshape(-1)
        if pts.size == 0:
            pts = np.zeros(1, np.float32)
        out = np.empty(dim, np.float32)
        self.r._check(self.r.lib.fkr_random_query(self.h, dim, pts, points.shape[0], out))
        return out
