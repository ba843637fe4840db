#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x -p no:cacheprovider --timeout=600 --timeout-method=thread > gpurun_out/r73_tests.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_push_huge -c 3 -o gpurun_out/bfs_push_huge -f python tools/bfs_one.py 8499673 > gpurun_out/r73_ncu.log 2>&1
ncu -i gpurun_out/bfs_push_huge.ncu-rep --page details --csv > gpurun_out/bfs_push_huge_details.csv 2>&1
