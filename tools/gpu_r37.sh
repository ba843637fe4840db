#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --config c1 --steps 5 --fusion > gpurun_out/b_c1_fused.json 2> gpurun_out/b_c1_fused.err
timeout 600 python bench.py --steps 3 --warmup 3 --fusion --no-e2e --no-cpu > gpurun_out/b_c5_fused.json 2> gpurun_out/b_c5_fused.err
