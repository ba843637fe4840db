#!/bin/bash
# vertex pass without rank/L1 at tolerance 0; smaller cold windows
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
grep -q "rc=0" gpurun_out/pytest_gpu.txt || exit 1
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
for cw in 6 3 4 6 3 4; do
  GG_PR_COLD_WINDOW16=$cw timeout 300 $B >> gpurun_out/vw_$cw.jsonl 2>/dev/null
done
