#!/bin/bash
# BFS per-level launch list (theta 0.002, unfused and fused); SSSP LB/coop sweep with checks.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_algos.py tests/test_gpu_engine.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_algos.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_algos.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -c 3000 --csv --log-file gpurun_out/launch_c2_t002.csv python bench.py --config c2 --sources 3 --warmup 1 --theta 0.002 > gpurun_out/launch_c2_t002.log 2>&1
timeout 600 python bench.py --config c2 --sources 16 --theta 0.002 --fusion > gpurun_out/c2_fused.json 2>&1
timeout 600 python bench.py --config c2 --sources 16 --theta 0.002 --pull-lb WM > gpurun_out/c2_wm.json 2>&1
GG_COOP_PER_SM=1 timeout 300 python bench.py --config c3 --side 512 --steps 1 --check > gpurun_out/c3_small_coop1.json 2>&1
for lb in VERTEX_BASED ETWC WM; do
  GG_COOP_PER_SM=1 timeout 900 python bench.py --config c3 --steps 1 --warmup 1 --lb $lb > gpurun_out/c3_$lb.json 2>&1
done
