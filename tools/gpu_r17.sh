#!/bin/bash
# ncu evidence: L2 hit rate EB off/on for PageRank at RMAT-27,
# warp execution efficiency ETWC vs TWC vs VERTEX_BASED (CC hook, Kron-25),
# full capture of the hot PR kernel; PR window-fraction sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__thread_inst_executed_per_inst_executed.ratio,l1tex__t_sector_hit_rate.pct
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 900 ncu --metrics $M --clock-control none -k "regex:k_pr_edges|k_edge_only|k_pr_vertex" -c 24 --csv --log-file gpurun_out/ncu_pr_eb.csv $B --schedule eb > gpurun_out/ncu_pr_eb.log 2>&1
timeout 900 ncu --metrics $M --clock-control none -k "regex:k_edge|k_pr" -c 6 --csv --log-file gpurun_out/ncu_pr_edge.csv $B --schedule edge > gpurun_out/ncu_pr_edge.log 2>&1
timeout 900 ncu --metrics $M --clock-control none --kernel-name-base demangled -k "regex:OpHook" -c 60 --csv --log-file gpurun_out/ncu_cc_lb.csv python bench.py --config c4 --lbs ETWC,TWC,VERTEX_BASED --steps 1 --warmup 1 --sources 1 > gpurun_out/ncu_cc_lb.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pr_edges_hot" -s 2 -c 1 -o gpurun_out/prof_pr_hot $B > gpurun_out/prof_pr_hot.log 2>&1
for w in 4 8 10; do
  GG_PR_WINDOW16=$w timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/win64_$w.json 2>&1
  GG_PR_WINDOW16=$w timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --fp32-contrib > gpurun_out/win32_$w.json 2>&1
done
