"""paper_2012_07990_b200 — B200-native edgeset.apply engine (GG, arXiv 2012.07990).

Drop-in for the traversal hot path of the reference package ``schedge``:
same algorithm functions, schedule language and Graph API, executed by
hand-written sm_100a CUDA kernels in ``libgg.so`` (C ABI, include/gg.h).
"""

from .sched import (HybridSchedule, ParseError, Schedule, ScheduleError, ScheduleProgram,
                    enumerate_space, parse_schedule, pretty_print, validate)
from .runtime import EdgeContext, EngineError, ExecConfig, RunStats, Runtime
from .frontier import BITMAP, BOOLMAP, SPARSE, FrontierError, VertexSubset
from .graphio import (Graph, GraphLoadError, generate_grid, generate_kronecker, generate_rmat,
                      load_edge_list, load_graph, load_matrix_market, out_degree,
                      with_random_weights)
from .priority import UNREACHED, BucketQueue
from .blocking import BlockedGraph, apply_blocked, block_edges, default_blocking_size
from .engine import edgeset_apply, fused_loop, hybrid_apply
from .algos import (ALGO_LABELS, ALGO_NAMES, AlgoResult, bc, bfs, bfs_levels, cc_soman,
                    pagerank, sssp_delta)
from . import udfs

__version__ = "0.1.0"

__all__ = [
    "ALGO_LABELS", "ALGO_NAMES", "AlgoResult", "bc", "bfs", "bfs_levels", "cc_soman",
    "pagerank", "sssp_delta", "BlockedGraph", "apply_blocked", "block_edges",
    "default_blocking_size", "BucketQueue",
    "BITMAP", "BOOLMAP", "SPARSE", "VertexSubset", "FrontierError", "Graph", "GraphLoadError",
    "load_edge_list", "load_graph", "load_matrix_market", "out_degree", "with_random_weights", "generate_rmat",
    "generate_grid", "generate_kronecker", "UNREACHED", "EdgeContext", "EngineError",
    "ExecConfig", "RunStats", "Runtime", "HybridSchedule", "ParseError", "Schedule",
    "ScheduleError", "ScheduleProgram", "enumerate_space", "parse_schedule", "pretty_print",
    "validate", "edgeset_apply", "fused_loop", "hybrid_apply", "udfs", "__version__",
]
