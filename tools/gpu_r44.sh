#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
grep -q "rc=0" gpurun_out/pytest_gpu.txt || exit 1
timeout 1200 python bench.py --config c4 --steps 2 --check > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
timeout 900 python bench.py > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err
