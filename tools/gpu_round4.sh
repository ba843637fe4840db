#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/debug_fused.py > gpurun_out/debug_fused.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_pagerank.py tests/test_gpu_graph.py tests/test_gpu_engine.py tests/test_gpu_dist.py -m gpu -q -x > gpurun_out/pytest_gpu_pr.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_pr.txt
timeout 600 python bench.py --steps 3 --warmup 3 --schedule eb --fp32-contrib --no-e2e --no-cpu > gpurun_out/bench_eb32.json 2> gpurun_out/bench_eb32.err
timeout 600 python bench.py --steps 3 --warmup 3 --schedule eb --no-e2e --no-cpu > gpurun_out/bench_eb64.json 2> gpurun_out/bench_eb64.err
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_pr_seg$" -s 12 -c 2 -o gpurun_out/prof_ebpull python bench.py --steps 1 --warmup 1 --schedule eb --fp32-contrib --no-e2e --no-cpu > gpurun_out/ncu_ebpull.log 2>&1
