#!/bin/bash
# dominant-kernel roofline fields; SSSP fused kernel full capture; BC launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/pr_default.json 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --fp32-contrib > gpurun_out/pr32.json 2>&1
GG_COOP_PER_SM=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_sssp_fused" -s 1 -c 1 -o gpurun_out/prof_sssp python bench.py --config c3 --side 2048 --delta 32768 --steps 1 --warmup 1 --lb VERTEX_BASED > gpurun_out/prof_sssp.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -c 2000 --csv --log-file gpurun_out/launch_bc.csv python bench.py --config c4 --lbs ETWC --sources 1 --steps 1 --warmup 1 > gpurun_out/launch_bc.log 2>&1
