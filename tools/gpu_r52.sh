#!/bin/bash
# cold window size A/B (f64 and f32)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
GG_PR_COLD_WINDOW16=16 timeout 600 python -m pytest tests/test_gpu_pagerank.py tests/test_gpu_dist.py -m gpu -q -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_cw.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_cw.txt
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
for cw in 6 10 16 32 6 16; do
  GG_PR_COLD_WINDOW16=$cw timeout 300 $B >> gpurun_out/cw_$cw.jsonl 2>/dev/null
done
GG_PR_COLD_WINDOW16=16 timeout 300 $B --fp32-contrib >> gpurun_out/cw_16_32.jsonl 2>/dev/null
