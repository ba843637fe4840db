#!/bin/bash
# PR layout build rewrite (histogram + 32-bit keys): parity, bench with e2e, e2e breakdown; CC EB.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pagerank.py tests/test_gpu_dist.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_pr.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_pr.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/pr64.json 2>&1
timeout 600 python tools/e2e_breakdown.py 27 > gpurun_out/e2e_breakdown.txt 2>&1
timeout 900 python bench.py --config c4 --steps 2 --lbs ETWC,EB,EDGE --check > gpurun_out/c4_eb.json 2>&1
