#!/bin/bash
# PR hot-segment variants (smem hot-source cache, edge prefetch) + C2-C4 bench bring-up.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
for fp in "" "--fp32-contrib"; do
  tag=${fp:+32}; tag=${tag:-64}
  GG_PR_HOT=0 GG_PR_PREFETCH=0 timeout 300 $B $fp > gpurun_out/v_${tag}_base.json 2>&1
  GG_PR_HOT=0 timeout 300 $B $fp > gpurun_out/v_${tag}_pf.json 2>&1
  timeout 300 $B $fp > gpurun_out/v_${tag}_hot1024.json 2>&1
  GG_PR_HOT_THREADS=512 timeout 300 $B $fp > gpurun_out/v_${tag}_hot512.json 2>&1
  GG_PR_PREFETCH=0 timeout 300 $B $fp > gpurun_out/v_${tag}_hot1024_nopf.json 2>&1
done
timeout 300 python bench.py --config c2 --scale 18 --sources 4 --check > gpurun_out/c2_small.json 2>&1
timeout 300 python bench.py --config c3 --side 512 --delta 64 --steps 1 --check > gpurun_out/c3_small.json 2>&1
timeout 300 python bench.py --config c4 --scale 16 --steps 1 --check > gpurun_out/c4_small.json 2>&1
timeout 600 python bench.py --config c2 > gpurun_out/c2.json 2>&1
timeout 900 python bench.py --config c3 --steps 2 > gpurun_out/c3.json 2>&1
timeout 900 python bench.py --config c4 --steps 2 > gpurun_out/c4.json 2>&1
