#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_algos.py tests/test_gpu_engine.py -q -x -p no:cacheprovider --timeout=600 --timeout-method=thread > gpurun_out/r66_tests.txt 2>&1
GG_ROUND_TRACE=1 timeout 600 python tools/bfs_overhead.py 24 0.0005,0.0001 > gpurun_out/bfs_rounds2.txt 2>&1
timeout 900 python bench.py --config c2 --check > gpurun_out/r66_c2.json 2> gpurun_out/r66_c2.err
timeout 900 python bench.py --config c4 > gpurun_out/r66_c4.json 2> gpurun_out/r66_c4.err
