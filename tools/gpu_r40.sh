#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
grep -q "rc=0" gpurun_out/pytest_gpu.txt || exit 1
timeout 600 python bench.py --config c2 --check > gpurun_out/c2.json 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -c 3000 --csv --log-file gpurun_out/launch_c2.csv python bench.py --config c2 --sources 3 --warmup 1 > gpurun_out/launch_c2.log 2>&1
