#!/bin/bash
# dist BFS/PR virtual-rank tests, PR defaults (128 KB hot cache), C2-C4 checks + launch lists.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x --timeout 300 > gpurun_out/pytest_dist.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist.txt
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/pr64.json 2>&1
timeout 300 $B --fp32-contrib > gpurun_out/pr32.json 2>&1
timeout 300 python bench.py --config c3 --side 512 --delta 64 --steps 1 --check > gpurun_out/c3_small.json 2>&1
timeout 300 python bench.py --config c4 --scale 16 --steps 1 --check > gpurun_out/c4_small.json 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -c 3000 --csv --log-file gpurun_out/launch_c2.csv python bench.py --config c2 --sources 3 --warmup 1 > gpurun_out/launch_c2.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -c 3000 --csv --log-file gpurun_out/launch_c4.csv python bench.py --config c4 --lbs TWC,ETWC --sources 1 --steps 1 --warmup 1 > gpurun_out/launch_c4.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -c 200 --csv --log-file gpurun_out/launch_c3.csv python bench.py --config c3 --delta 8192 --steps 1 --warmup 1 > gpurun_out/launch_c3.log 2>&1
