#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for t in "True-PUSH-EDGE_ONLY" "True-PUSH-ETWC" "True-PULL-TWC"; do
  timeout 120 python -m pytest "tests/test_gpu_algos.py::test_bfs_every_schedule[$t]" -q -x > gpurun_out/t_$t.txt 2>&1
  echo "rc=$?" >> gpurun_out/t_$t.txt
done
timeout 900 python -m pytest tests/test_gpu_pagerank.py -m gpu -q -x > gpurun_out/pytest_gpu_pr.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_pr.txt
timeout 600 python bench.py --steps 3 --warmup 3 --schedule eb --fp32-contrib --no-e2e --no-cpu > gpurun_out/bench_eb32.json 2> gpurun_out/bench_eb32.err
timeout 600 python bench.py --steps 3 --warmup 3 --schedule pull_wm --fp32-contrib --no-e2e --no-cpu > gpurun_out/bench_pull_wm32.json 2> gpurun_out/bench_pull_wm32.err
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_pr_seg$" -c 12 -o gpurun_out/prof_ebpull python bench.py --steps 1 --warmup 1 --schedule eb --fp32-contrib --no-e2e --no-cpu > gpurun_out/ncu_ebpull.log 2>&1
