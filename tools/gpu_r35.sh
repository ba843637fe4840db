#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_algos.py -m gpu -q -x --timeout 120 --timeout-method=thread -k "sssp" > gpurun_out/pytest_sssp.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_sssp.txt
grep -q "rc=0" gpurun_out/pytest_sssp.txt || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
for lb in WM VERTEX_BASED; do
  GG_SSSP_PROFILE=1 timeout 400 python bench.py --config c3 --steps 2 --warmup 1 --lb $lb > gpurun_out/c3_$lb.json 2> gpurun_out/c3_$lb.err
done
timeout 300 python bench.py --config c3 --side 1024 --steps 1 --warmup 1 --lb WM --check > gpurun_out/c3_wm_check.json 2>&1
