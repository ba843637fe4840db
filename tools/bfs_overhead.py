"""C2 DO-BFS (RMAT-24): per-source call time vs the time inside the
edge-apply phases, rounds and launches -- how much of a source is host
round trips between levels."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2012_07990_b200 as gg

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = gg.generate_rmat(scale, 16, seed=2, symmetrize=True)
deg = np.diff(np.asarray(g.out_offsets, dtype=np.int64))
rng = np.random.default_rng(3)
srcs = [int(x) for x in rng.choice(np.flatnonzero(deg > 0), size=12, replace=False)]
thetas = [float(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0.0005]
parents = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
for theta in thetas:
    hy = gg.HybridSchedule(threshold=theta,
                           s1=gg.Schedule(direction="PUSH", load_balance="ETWC", dedup=False),
                           s2=gg.Schedule(direction="PULL", pull_frontier_repr="BITMAP",
                                          frontier_creation="UNFUSED_BITMAP"))
    prog = gg.ScheduleProgram({"s0:s1": hy})
    for s in srcs[:3]:
        gg.bfs(g, s, prog, out=parents)
    print("theta", theta)
    tot = []
    for s in srcs:
        t = time.perf_counter()
        r = gg.bfs(g, s, prog, out=parents)
        wall = (time.perf_counter() - t) * 1e3
        st = r.stats
        tot.append(st.kernel_ms)
        print("src %9d: call %.3f ms (wall %.3f) edge-phases %.3f ms over %d rounds, %d launches, dirs %s"
              % (s, st.kernel_ms, wall, st.edge_ms, st.rounds, st.gpu_launches,
                 "".join("P" if d == "PUSH" else "l" for d in st.direction_log)), flush=True)
    print("theta %g: mean %.3f ms, max %.3f" % (theta, sum(tot) / len(tot), max(tot)))
