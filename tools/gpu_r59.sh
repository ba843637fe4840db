#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python tools/bc_timing.py > gpurun_out/bc_timing.txt 2>&1
M=gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none -c 1500 --csv --log-file gpurun_out/launch_bc2.csv python bench.py --config c4 --lbs TWC --sources 1 --steps 1 --warmup 1 > gpurun_out/launch_bc2.log 2>&1
