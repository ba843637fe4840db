#!/bin/bash
# BC warp-reduced backward, CC hook precheck; full suite; bench default; c4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/pr_default.json 2>&1
timeout 900 python bench.py --config c4 --steps 2 --check > gpurun_out/c4.json 2>&1
timeout 600 python bench.py --config c2 --check > gpurun_out/c2.json 2>&1
