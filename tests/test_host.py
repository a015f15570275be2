"""CPU-only checks of the product library: it loads, exports every symbol
include/fkd_b200.h declares, its host utilities match the oracle, its C++
headers compile, and without a GPU the query path refuses loudly (no CPU
fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2210_12859_b200 as fk
from paper_2210_12859_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fkd_b200.h")


def test_exports_every_declared_symbol():
    decl = set(re.findall(r"\b(fkd_[a-z_]+)\s*\(", open(HEADER).read()))
    assert decl == set(_lib.EXPORTS)
    lib = C.CDLL(_lib.LIB_PATH)
    for name in sorted(decl):
        assert hasattr(lib, name), name
    assert fk.LIB.fkd_version().decode().endswith("(sm_100a)")


def test_struct_layouts():
    assert C.sizeof(_lib.fkd_query_stats) == 24
    assert fk.HIT_DTYPE.itemsize == 8 and fk.HIT_DTYPE.fields["dist2"][1] == 4
    assert C.sizeof(_lib.fkd_batch_options) == 28
    o = _lib.fkd_batch_options()
    fk.LIB.fkd_default_options(C.byref(o))
    assert (o.kind, o.k, o.max_radius, o.engine, o.collect_stats) == (0, 1, float("inf"), 0, 0)


def test_sm100a_cubin_in_library():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_host_builder_matches_oracle(oracle):
    for n, dim in [(0, 3), (1, 1), (7, 2), (1000, 3), (4097, 4), (3000, 8), (500, 11)]:
        pts = oracle.random_points(31 + n, n, dim)
        assert np.array_equal(fk.build_level_order(pts), oracle.build_tree(pts)), (n, dim)
    rng = oracle.instance_rng(5)
    for _ in range(20):
        pts = rng.random_point_set(rng.next_int(1, 3000), rng.next_int(1, 4), 8, 0.2)
        assert np.array_equal(fk.build_level_order(pts), oracle.build_tree(pts))


def test_generators_and_hash_match_oracle(oracle):
    for s in (1, 2, 7):
        assert np.array_equal(fk.random_points(1, s, 1000, 3),
                              oracle.random_points(oracle.derive_stream_seed(1, s), 1000, 3))
    nodes = oracle.build_tree(oracle.random_points(3, 2000, 3))
    qs = oracle.random_points(4, 300, 3)
    for kind, k in (("fcp", 1), ("knn", 8)):
        c, h, _, _ = oracle.run_batch(nodes, qs, kind, k, 0.1)
        assert fk.result_hash(c, h, k) == oracle.result_hash(c, h, k)
        res = fk.BatchResult(k, c, h)
        assert res.result_hash() == oracle.result_hash(c, h, k)


def test_write_query_results_format(reference):
    nodes = reference.build_tree(np.array([[2, 3], [5, 4], [9, 6], [4, 7], [8, 1], [7, 2]], np.float32))
    for kind, k in (("fcp", 1), ("knn", 3)):
        c, h, _, _ = reference.run_batch(nodes, np.array([[9, 2], [2, 3], [100, 100]], np.float32), kind, k, 5.0)
        assert fk.write_query_results(fk.BatchResult(k, c, h)) == reference.write_results(c, h, k)


def test_clustered_generator_is_deterministic():
    a = fk.clustered_points(1, 2, 5000, 3)
    b = fk.clustered_points(1, 2, 5000, 3)
    assert np.array_equal(a, b) and np.isfinite(a).all()
    assert not np.array_equal(a, fk.clustered_points(1, 1, 5000, 3))


@pytest.mark.skipif(__import__("conftest").HAS_GPU, reason="checks the no-GPU refusal")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(fk.DeviceError, match="no CPU fallback"):
        fk.KdTree.from_level_order(np.zeros((4, 3), np.float32))


def test_cpp_shim_headers_compile(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "flatkd_b200/flatkd.hpp"\nstruct f3 { float x, y, z; };\n'
                   "int main() { flatkd::b200::BatchOptions o; auto c = o.to_c();\n"
                   "  static_assert(flatkd::b200::point_dim_v<f3> == 3); return c.k - 1; }\n")
    out = subprocess.run(["/usr/bin/g++", "-std=c++20", "-fsyntax-only", f"-I{ROOT}/include", str(src)],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr


def test_validation_order_in_options():
    with pytest.raises(fk.InvalidArgument):
        fk.run_batch(None, np.zeros((1, 3), np.float32), fk.BatchOptions(kind=fk.QueryKind.knn, k=0))


def test_workload_generators_match_reference_rng(reference):
    """bench.py's reference arm draws its inputs from the reference library
    (oracle/ref_capi.cpp) and the B200 arm from the product's host
    generators: both must be byte-identical, uniform and clustered."""
    for dim in (2, 3, 8):
        assert np.array_equal(fk.random_points(1, 2, 5000, dim), reference.stream_points(1, 2, 5000, dim))
        assert np.array_equal(fk.clustered_points(1, 1, 5000, dim, 64, 0.02),
                              reference.clustered_points(1, 1, 5000, dim, 64, 0.02))


def test_scale_goldens_agree_with_survey():
    """tests/golden/scale.json (reference run over the whole batches) against
    the hashes SURVEY.md §8(c) recorded at survey time."""
    import json

    g = json.load(open(os.path.join(ROOT, "tests", "golden", "scale.json")))["cases"]
    survey = {"fcp_3d_n10m_m1m": "0cca445a11013618", "knn8_3d_n10m_m1m": "5a71a6a204bbe790",
              "fcp_4d_n10m_m1m": "11d43fd7c68c62e6", "knn8_4d_n10m_m1m_r0.01": "7c5c62b9b41500e3",
              "knn16_2d_n10m_m200k": "6a39ab1bb32b6cb2", "knn16_4d_n10m_m200k": "563944befa0aff8b",
              "knn16_8d_n10m_m200k": "10a6147e5f8a5a07", "fcp_3d_n100m_m200k": "1fc44d5457a0fee4"}
    for name, h in survey.items():
        assert g[name]["hash"] == h, name
    assert {"c3_fcp_clustered_n10m_m10m", "c3_knn8_clustered_n10m_m10m"} <= set(g)
    # P-bar of the C3 batches (bench.py's algorithmic bytes) from the reference's counters
    assert abs(g["c3_knn8_clustered_n10m_m10m"]["stats"][2] / 1e7 - 126.4611659) < 1e-6
