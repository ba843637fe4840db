"""Phase breakdown of bench.py's e2e step (PageRank EB, RMAT-27): H2D + graph
create, EdgeBlocking layout build, 20 iterations, D2H."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2012_07990_b200 as gg
from paper_2012_07990_b200 import _lib
from paper_2012_07990_b200.engine import binding_pod

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
fp32 = len(sys.argv) > 2 and sys.argv[2] == "32"
g = gg.generate_rmat(scale, 16, seed=7, sort_by_source=True)
V, E = g.num_vertices, g.num_edges
src_h = torch.from_numpy(g.coo_src).pin_memory()
dst_h = torch.from_numpy(g.coo_dst).pin_memory()
g.close()
ranks_h = torch.empty(V, dtype=torch.float64).pin_memory()
sch = gg.Schedule(load_balance="EDGE_ONLY", blocking=True)
prog = gg.ScheduleProgram({"s0:s1": sch})
pod = binding_pod(sch)
# raw pinned H2D bandwidth
buf = torch.empty(E, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter(); buf.copy_(src_h, non_blocking=True); torch.cuda.synchronize()
print("raw H2D %.1f GB/s" % (4 * E / (time.perf_counter() - t) / 1e9))
del buf
torch.cuda.empty_cache()
for step in range(3):
    t0 = time.perf_counter()
    ge = gg.Graph.from_coo(V, src_h.numpy(), dst_h.numpy())
    t1 = time.perf_counter()
    pm = C.c_double()
    _lib.call("gg_pagerank_prepare", ge.handle, C.byref(pod), 1 if fp32 else 0, C.byref(pm))
    t2 = time.perf_counter()
    r = gg.pagerank(ge, prog, max_iters=20, tolerance=0.0, out=ranks_h.numpy(), contrib_fp32=fp32)
    t3 = time.perf_counter()
    ge.close()
    t4 = time.perf_counter()
    ps = gg.runtime.pool_stats()
    print("pool: %d mallocs %d frees %.1f GB cached" % (ps["mallocs"], ps["frees"], ps["cached_bytes"] / 2**30))
    print("step %d: create+H2D %.3f s  layout %.3f s  pagerank(20 it + D2H) %.3f s (kernel %.3f ms)  close %.3f s  total %.3f s"
          % (step, t1 - t0, t2 - t1, t3 - t2, r.stats.kernel_ms, t4 - t3, t4 - t0))
