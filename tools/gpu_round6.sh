#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_algos.py -m gpu -v --timeout 120 --timeout-method=thread > gpurun_out/pytest_algos.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_algos.txt
timeout 600 python -m pytest tests/test_gpu_pagerank.py tests/test_gpu_engine.py tests/test_gpu_graph.py tests/test_gpu_dist.py -m gpu -q --timeout 120 --timeout-method=thread > gpurun_out/pytest_rest.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_rest.txt
timeout 600 python bench.py --steps 3 --warmup 3 --schedule eb --fp32-contrib --no-e2e --no-cpu > gpurun_out/bench_eb32.json 2> gpurun_out/bench_eb32.err
timeout 600 python bench.py --steps 3 --warmup 3 --schedule pull_wm --fp32-contrib --no-e2e --no-cpu > gpurun_out/bench_pull_wm32.json 2> gpurun_out/bench_pull_wm32.err
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_pr_seg$" -c 12 -o gpurun_out/prof_ebpull python bench.py --steps 1 --warmup 1 --schedule eb --fp32-contrib --no-e2e --no-cpu > gpurun_out/ncu_ebpull.log 2>&1
