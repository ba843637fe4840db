#!/bin/bash
# hot kernel gather flavour x hot-cache size (is L1 the staging for in-flight gathers?)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
for g in 1 2; do
  for kb in 128 192; do
    GG_PR_GATHER=$g GG_PR_HOT_KB=$kb timeout 300 $B > gpurun_out/ga${g}_${kb}.json 2>&1
    GG_PR_GATHER=$g GG_PR_HOT_KB=$kb timeout 300 $B --fp32-contrib > gpurun_out/ga${g}_${kb}_32.json 2>&1
  done
done
