#!/bin/bash
# one-segment layout (every edge in the hot kernel, evict-first gathers past the window) A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
GG_PR_ONE_SEGMENT=1 timeout 600 python -m pytest tests/test_gpu_pagerank.py -m gpu -q -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_one.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_one.txt
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
for o in 0 1 0 1; do
  GG_PR_ONE_SEGMENT=$o timeout 300 $B >> gpurun_out/one_$o.jsonl 2>/dev/null
done
GG_PR_ONE_SEGMENT=1 timeout 300 $B --fp32-contrib >> gpurun_out/one_1_32.jsonl 2>/dev/null
