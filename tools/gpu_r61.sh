#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_algos.py -q -x -k "pool or bc" -p no:cacheprovider --timeout=300 --timeout-method=thread > gpurun_out/r61_tests.txt 2>&1
GG_POOL_TRACE=1 timeout 900 python tools/bc_timing.py > gpurun_out/bc_timing3.txt 2> gpurun_out/bc_pool3.txt
timeout 900 python bench.py --config c4 > gpurun_out/r61_c4.json 2> gpurun_out/r61_c4.err
timeout 900 python bench.py > gpurun_out/r61_c5.json 2> gpurun_out/r61_c5.err
