"""Run each fused schedule in its own subprocess with a watchdog; report hangs."""
import subprocess, sys, json
CASE = r'''
import sys; sys.path.insert(0, ".")
import numpy as np, paper_2012_07990_b200 as gg, oracle
algo, lb, direction, gname = sys.argv[1:5]
g = gg.generate_rmat(8, 8, seed=2, symmetrize=True, weights=(algo == "sssp"))
prog = gg.ScheduleProgram({"s0:s1": gg.Schedule(direction=direction, load_balance=lb), "s0": gg.Schedule(kernel_fusion=True)})
if algo == "bfs":
    r = gg.bfs(g, 0, prog)
    off, nbr, _ = oracle.csr(g.num_vertices, g.coo_src, g.coo_dst)
    ok = gg.bfs_levels(r.values) == oracle.bfs_levels(g.num_vertices, off, nbr, 0).tolist()
elif algo == "cc":
    r = gg.cc_soman(g, prog)
    ok = r.values == oracle.cc(g.num_vertices, g.coo_src, g.coo_dst)[0].tolist()
else:
    r = gg.sssp_delta(g, 0, prog)
    off, nbr, w = oracle.csr(g.num_vertices, g.coo_src, g.coo_dst, g.coo_weights)
    ok = np.array_equal(r.array, oracle.sssp_delta(g.num_vertices, off, nbr, w, 0, 1)[0])
print("OK" if ok else "MISMATCH", r.stats.rounds, r.stats.dispatch_count)
'''
open("/tmp/case.py", "w").write(CASE)
res = {}
for algo in ("bfs", "cc", "sssp"):
    for direction in ("PUSH", "PULL"):
        if algo == "sssp" and direction == "PULL":
            continue
        for lb in ("VERTEX_BASED", "CM", "WM", "STRICT", "EDGE_ONLY", "ETWC", "TWC"):
            key = "%s/%s/%s" % (algo, direction, lb)
            try:
                p = subprocess.run([sys.executable, "/tmp/case.py", algo, lb, direction, "x"],
                                   capture_output=True, text=True, timeout=60)
                res[key] = (p.stdout.strip() or p.stderr.strip()[-300:])
            except subprocess.TimeoutExpired:
                res[key] = "HANG"
            print(key, res[key], flush=True)
json.dump(res, open("gpurun_out/debug_fused.json", "w"), indent=1)
