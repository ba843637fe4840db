#!/bin/bash
# caching allocator: full GPU suite, PR bench, C2-C4 lines, CC LB warp-efficiency evidence.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/smoke.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/pr64.json 2>&1
for t in 0.0005 0.002; do
  timeout 600 python bench.py --config c2 --theta $t > gpurun_out/c2_t$t.json 2>&1
  timeout 600 python bench.py --config c2 --theta $t --fusion > gpurun_out/c2_t${t}_fused.json 2>&1
done
timeout 900 python bench.py --config c4 --steps 2 > gpurun_out/c4.json 2>&1
GG_COOP_PER_SM=1 timeout 900 python bench.py --config c3 --steps 2 --warmup 1 --lb VERTEX_BASED > gpurun_out/c3.json 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__thread_inst_executed_per_inst_executed.ratio,l1tex__t_sector_hit_rate.pct
timeout 900 ncu --metrics $M --clock-control none --kernel-name-base demangled -k "regex:OpHook" -c 60 --csv --log-file gpurun_out/ncu_cc_lb.csv python bench.py --config c4 --lbs ETWC,TWC,VERTEX_BASED --steps 1 --warmup 1 --sources 1 > gpurun_out/ncu_cc_lb.log 2>&1
