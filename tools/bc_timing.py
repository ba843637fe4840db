"""BC on Kronecker-25 (c4 graph): per-call device time for a few schedules,
repeated, to expose run-to-run variance."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2012_07990_b200 as gg

g = gg.generate_kronecker(25, 16, seed=5, symmetrize=True, sort_by_source=True)
V = g.num_vertices
deg = np.diff(np.asarray(g.out_offsets, dtype=np.int64))
rng = np.random.default_rng(6)
srcs = [int(x) for x in rng.choice(np.flatnonzero(deg > 0), size=4, replace=False)]
scores = torch.empty(V, dtype=torch.float64, device="cuda")
for lb in ["TWC", "ETWC", "TWC", "ETWC"]:
    prog = gg.ScheduleProgram({"s0:s1": gg.Schedule(direction="PUSH", load_balance=lb)})
    for rep in range(3):
        t = time.perf_counter()
        r = gg.bc(g, srcs, prog, out=scores)
        print("%s rep %d: kernel %.1f ms wall %.1f ms rounds %d" % (lb, rep, r.stats.kernel_ms,
              (time.perf_counter() - t) * 1e3, r.stats.rounds), flush=True)
