#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --config c2 --check > gpurun_out/c2.json 2>&1
timeout 900 ncu --set full --clock-control none -k "regex:k_pull_vb" -s 0 -c 1 -o gpurun_out/prof_pull3 python bench.py --config c2 --sources 1 --warmup 1 > gpurun_out/prof_pull3.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
