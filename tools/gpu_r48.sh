#!/bin/bash
# full capture of the first bottom-up BFS level (C2)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pull_vb" -s 0 -c 1 -o gpurun_out/prof_pull python bench.py --config c2 --sources 1 --warmup 1 > gpurun_out/prof_pull.log 2>&1
