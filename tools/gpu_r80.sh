#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_algos.py -q -x -p no:cacheprovider --timeout=60 --timeout-method=thread > gpurun_out/r80_tests.txt 2>&1 || exit 3
timeout 240 python bench.py --config c2 > gpurun_out/r80_c2.json 2> gpurun_out/r80_c2.err
timeout 300 python bench.py --config c4 > gpurun_out/r80_c4.json 2> gpurun_out/r80_c4.err
