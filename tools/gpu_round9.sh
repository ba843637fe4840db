#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_eb.csv python bench.py --steps 1 --warmup 1 --schedule eb --fp32-contrib --no-e2e --no-cpu > gpurun_out/launches_eb.log 2>&1
