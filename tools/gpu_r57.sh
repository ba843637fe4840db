#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_algos.py tests/test_gpu_engine.py tests/test_gpu_dist.py -m gpu -q -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_bfs.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_bfs.txt
grep -q "rc=0" gpurun_out/pytest_bfs.txt || exit 1
timeout 600 python bench.py --config c2 --check > gpurun_out/c2_x2.json 2>&1
M=gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -k "regex:k_pull_vb" -c 40 --csv --log-file gpurun_out/pull_x2.csv python bench.py --config c2 --sources 3 --warmup 1 > gpurun_out/pull_x2.log 2>&1
