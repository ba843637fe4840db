#!/bin/bash
# fused loops read pre-barrier data through L1 (ld_fresh)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
grep -q "rc=0" gpurun_out/pytest_gpu.txt || exit 1
timeout 600 python bench.py --config c2 --sources 32 --fusion > gpurun_out/c2_fused.json 2>&1
timeout 600 python bench.py --config c2 --sources 32 > gpurun_out/c2.json 2>&1
timeout 300 python bench.py --config c1 --steps 5 --fusion > gpurun_out/c1_fused.json 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --fusion --no-e2e --no-cpu > gpurun_out/c5_fused.json 2>&1
timeout 600 python bench.py --config c3 --steps 2 > gpurun_out/c3.json 2>&1
