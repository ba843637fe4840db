#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x -p no:cacheprovider --timeout=600 --timeout-method=thread > gpurun_out/r72_tests.txt 2>&1
timeout 900 python bench.py --config c3 > gpurun_out/r72_c3.json 2> gpurun_out/r72_c3.err
timeout 900 python bench.py > gpurun_out/r72_c5.json 2> gpurun_out/r72_c5.err
