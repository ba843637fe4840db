#!/bin/bash
# PR edge-case tests; fresh launch list + hot-kernel full capture of the default bench command.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pagerank.py tests/test_gpu_dist.py -m gpu -q -x --timeout 600 > gpurun_out/pytest_pr.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_pr.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5_f64.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/launches_c5_f64.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pr_edges_hot" -s 2 -c 1 -o gpurun_out/prof_pr_hot_f64 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof_pr_hot_f64.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pr_vertex" -s 2 -c 1 -o gpurun_out/prof_pr_vertex_f64 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof_pr_vertex_f64.log 2>&1
