"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/gg.h declares (no compute calls here)."""

import os
import re

from tests.conftest import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gg.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_driver_surface():
    names = declared_symbols()
    for must in ("gg_graph_create", "gg_edgeset_apply", "gg_bfs", "gg_pagerank",
                 "gg_sssp_delta", "gg_cc", "gg_bc", "gg_block_edges", "gg_pagerank_dist"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2012_07990_b200 import _lib
    lib = _lib.load()
    missing = [n for n in declared_symbols() if getattr(lib, n, None) is None]
    assert missing == []
    assert set(_lib.SIGNATURES) >= set(declared_symbols())


def test_library_reports_errors_without_a_device():
    import ctypes as C
    from paper_2012_07990_b200 import _lib
    lib = _lib.load()
    n = C.c_int32(-1)
    assert lib.gg_device_count(C.byref(n)) == 0
    assert n.value >= 0
    assert lib.gg_version().startswith(b"gg-b200")


# the reference package's export list (schedge/__init__.py:26-38)
REFERENCE_ALL = [
    "ALGO_LABELS", "ALGO_NAMES", "AlgoResult", "bc", "bfs", "bfs_levels", "cc_soman",
    "pagerank", "sssp_delta", "BlockedGraph", "apply_blocked", "block_edges", "BITMAP",
    "BOOLMAP", "SPARSE", "VertexSubset", "Graph", "GraphLoadError", "load_edge_list",
    "load_graph", "load_matrix_market", "out_degree", "with_random_weights", "UNREACHED",
    "BucketQueue", "EdgeContext", "EngineError", "ExecConfig", "RunStats", "Runtime",
    "HybridSchedule", "ParseError", "Schedule", "ScheduleError", "ScheduleProgram",
    "enumerate_space", "parse_schedule", "pretty_print", "validate", "edgeset_apply",
    "fused_loop", "hybrid_apply", "__version__",
]


def test_package_exports_the_reference_surface():
    import paper_2012_07990_b200 as gg
    assert [n for n in REFERENCE_ALL if not hasattr(gg, n)] == []
    assert set(REFERENCE_ALL) <= set(gg.__all__)


def test_every_algorithm_udf_has_a_device_id():
    from paper_2012_07990_b200 import _lib, udfs
    codes = {c.code for c in (udfs.BfsParent, udfs.CountInDegree, udfs.EnqueueDst,
                              udfs.PageRankGather, udfs.CcHook, udfs.BcForward,
                              udfs.BcBackward, udfs.SsspRelax)}
    assert codes == set(range(8))
    text = open(os.path.join(ROOT, "include", "gg.h")).read()
    for name in ("GG_UDF_CC_HOOK = 4", "GG_UDF_BC_FORWARD = 5", "GG_UDF_BC_BACKWARD = 6",
                 "GG_UDF_SSSP_RELAX = 7"):
        assert name in text
    assert _lib.UDF_SSSP_RELAX == 7
