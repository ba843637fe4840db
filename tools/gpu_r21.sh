#!/bin/bash
# lazy AlgoResult.values (e2e), hub-graph ETWC tests, BFS dedup-off.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/pr_default.json 2>&1
timeout 600 python tools/e2e_breakdown.py 27 > gpurun_out/e2e_breakdown.txt 2>&1
timeout 600 python bench.py --config c2 > gpurun_out/c2.json 2>&1
timeout 600 python bench.py --config c2 --no-dedup > gpurun_out/c2_nodedup.json 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2>&1
