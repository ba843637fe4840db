#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pr_pull<" -s 3 -c 1 -o gpurun_out/prof_pull python bench.py --steps 1 --warmup 1 --schedule pull_wm --fp32-contrib --no-e2e --no-cpu > gpurun_out/ncu_pull.log 2>&1
