#!/bin/bash
# merged cold segments A/B (f64, f32), with parity tests under the toggle
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
GG_PR_MERGE_COLD=1 timeout 600 python -m pytest tests/test_gpu_pagerank.py tests/test_gpu_dist.py -m gpu -q -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_merge.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_merge.txt
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
for m in 0 1 0 1; do
  GG_PR_MERGE_COLD=$m timeout 300 $B > gpurun_out/mc_$m.json 2>&1; cat gpurun_out/mc_$m.json >> gpurun_out/mc_all_$m.jsonl
done
GG_PR_MERGE_COLD=1 timeout 300 $B --fp32-contrib > gpurun_out/mc_1_32.json 2>&1
