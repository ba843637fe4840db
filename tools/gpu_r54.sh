#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --fp32-contrib > gpurun_out/b_c5_32.json 2> gpurun_out/b_c5_32.err
timeout 300 python bench.py --config c1 --steps 5 > gpurun_out/b_c1.json 2> gpurun_out/b_c1.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5_f64.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/launches_c5_f64.log 2>&1
