#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_algos.py tests/test_gpu_engine.py -q -x -p no:cacheprovider --timeout=900 --timeout-method=thread > gpurun_out/r70_tests.txt 2>&1
timeout 900 python bench.py --config c4 > gpurun_out/r70_c4.json 2> gpurun_out/r70_c4.err
