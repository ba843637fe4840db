#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
for lb in CM STRICT; do
  timeout 600 python bench.py --config c2 --sources 16 --pull-lb $lb > gpurun_out/c2_pull_$lb.json 2>&1
done
timeout 600 python bench.py --config c2 > gpurun_out/c2.json 2>&1
