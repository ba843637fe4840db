#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout=900 --timeout-method=thread > gpurun_out/r76_tests.txt 2>&1
timeout 900 python bench.py --config c2 --check > gpurun_out/r76_c2.json 2> gpurun_out/r76_c2.err
timeout 900 python bench.py --config c4 > gpurun_out/r76_c4.json 2> gpurun_out/r76_c4.err
