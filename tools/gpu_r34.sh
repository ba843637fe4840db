#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
for lb in WM VERTEX_BASED; do
  GG_SSSP_PROFILE=1 GG_COOP_PER_SM=1 timeout 600 python bench.py --config c3 --steps 2 --warmup 1 --lb $lb > gpurun_out/c3_$lb.json 2> gpurun_out/c3_$lb.err
done
GG_COOP_PER_SM=1 timeout 300 python bench.py --config c3 --side 1024 --steps 1 --warmup 1 --lb WM --check > gpurun_out/c3_wm_check.json 2>&1
