#!/bin/bash
# C2 pull-side load balance sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lb in ETWC TWC CM STRICT VERTEX_BASED; do
  timeout 600 python bench.py --config c2 --sources 32 --pull-lb $lb > gpurun_out/c2_pull_$lb.json 2>&1
done
timeout 600 python bench.py --config c2 --sources 32 --theta 0.0002 > gpurun_out/c2_t0002.json 2>&1
timeout 600 python bench.py --config c2 --sources 32 --theta 0.001 > gpurun_out/c2_t001.json 2>&1
