#!/bin/bash
# ETWC grid-wide hub pass; BFS threshold sweep; SSSP coop-CTA sweep; CC flag fix.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
for t in 0.0005 0.002 0.01 0.05; do
  timeout 600 python bench.py --config c2 --sources 16 --theta $t > gpurun_out/c2_t$t.json 2>&1
done
timeout 900 python bench.py --config c4 --steps 2 --check > gpurun_out/c4.json 2>&1
for c in 1 2 4; do
  GG_COOP_PER_SM=$c timeout 600 python bench.py --config c3 --steps 1 --warmup 1 > gpurun_out/c3_coop$c.json 2>&1
done
