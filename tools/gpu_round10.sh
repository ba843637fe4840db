#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_pr_vertex$" -s 2 -c 1 -o gpurun_out/prof_vertex python bench.py --steps 1 --warmup 1 --schedule eb --fp32-contrib --no-e2e --no-cpu > gpurun_out/ncu_vertex.log 2>&1
