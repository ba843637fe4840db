#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pagerank.py -m gpu -q -x --timeout 120 --timeout-method=thread > gpurun_out/pytest_gpu_pr.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_pr.txt
timeout 600 python bench.py --steps 3 --warmup 3 --schedule eb --fp32-contrib --no-e2e --no-cpu > gpurun_out/bench_eb32.json 2> gpurun_out/bench_eb32.err
GG_PR_NO_SMEM_CACHE=1 timeout 600 python bench.py --steps 3 --warmup 3 --schedule eb --fp32-contrib --no-e2e --no-cpu > gpurun_out/bench_eb32_nocache.json 2> gpurun_out/bench_eb32_nocache.err
timeout 600 python bench.py --steps 3 --warmup 3 --schedule eb --no-e2e --no-cpu > gpurun_out/bench_eb64.json 2> gpurun_out/bench_eb64.err
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_pr_edges_hot$" -c 1 -o gpurun_out/prof_hot python bench.py --steps 1 --warmup 1 --schedule eb --fp32-contrib --no-e2e --no-cpu > gpurun_out/ncu_hot.log 2>&1
