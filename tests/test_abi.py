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
