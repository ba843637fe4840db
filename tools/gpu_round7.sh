#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pagerank.py tests/test_gpu_dist.py -m gpu -q -x --timeout 120 --timeout-method=thread > gpurun_out/pytest_gpu_pr.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_pr.txt
for cfg in "eb --fp32-contrib" "eb" "pull --fp32-contrib"; do
  n=$(echo $cfg | tr -d ' -')
  timeout 600 python bench.py --steps 3 --warmup 3 --schedule $cfg --no-e2e --no-cpu > gpurun_out/bench_$n.json 2> gpurun_out/bench_$n.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_pr_tiles$" -c 12 -o gpurun_out/prof_tiles python bench.py --steps 1 --warmup 1 --schedule eb --fp32-contrib --no-e2e --no-cpu > gpurun_out/ncu_tiles.log 2>&1
