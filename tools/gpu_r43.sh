#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_algos.py -m gpu -q -x --timeout 300 --timeout-method=thread -k "cc or hub" > gpurun_out/pytest_cc.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_cc.txt
for b in 1 0; do
  GG_EDGE_BATCH4=$b timeout 600 python bench.py --config c4 --steps 2 --lbs ETWC,EB,EDGE --sources 1 --check > gpurun_out/c4_b$b.json 2>&1
done
