"""One DO-BFS source on RMAT-24 (C2 graph, for ncu captures of single levels)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2012_07990_b200 as gg

src = int(sys.argv[1]) if len(sys.argv) > 1 else 8499673
g = gg.generate_rmat(24, 16, seed=2, symmetrize=True)
hy = gg.HybridSchedule(threshold=0.0005,
                       s1=gg.Schedule(direction="PUSH", load_balance="ETWC", dedup=False),
                       s2=gg.Schedule(direction="PULL", pull_frontier_repr="BITMAP",
                                      frontier_creation="UNFUSED_BITMAP"))
prog = gg.ScheduleProgram({"s0:s1": hy})
parents = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
r = gg.bfs(g, src, prog, out=parents)
print("rounds", r.stats.rounds, "edges", r.stats.edges_traversed, "ms", r.stats.kernel_ms)
