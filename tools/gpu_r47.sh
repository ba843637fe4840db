#!/bin/bash
# hot kernel: scan block 32 / 16 / 8 (fewer shuffle steps, more adds)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for sb in 8 16; do
  GG_PR_SCAN_BLOCK=$sb timeout 600 python -m pytest tests/test_gpu_pagerank.py -m gpu -q -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_sb$sb.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_sb$sb.txt
done
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
for sb in 32 8 16 32 8 16; do
  GG_PR_SCAN_BLOCK=$sb timeout 300 $B >> gpurun_out/sb_$sb.jsonl 2>/dev/null
done
GG_PR_SCAN_BLOCK=8 timeout 300 $B --fp32-contrib > gpurun_out/sb_8_32.json 2>&1
