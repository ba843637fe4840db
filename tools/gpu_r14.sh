#!/bin/bash
# smem hot-cache size sweep (L1 left for miss staging), virtual-rank partition tests, C2-C4 bring-up.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x --timeout 300 > gpurun_out/pytest_dist.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist.txt
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
for n in 8192 16384 24576 32768; do
  GG_PR_NHOT=$n timeout 300 $B --fp32-contrib > gpurun_out/w_32_nhot$n.json 2>&1
done
for n in 4096 8192 16384; do
  GG_PR_NHOT=$n timeout 300 $B > gpurun_out/w_64_nhot$n.json 2>&1
done
timeout 300 python bench.py --config c2 --scale 18 --sources 4 --check > gpurun_out/c2_small.json 2>&1
timeout 300 python bench.py --config c3 --side 512 --delta 64 --steps 1 --check > gpurun_out/c3_small.json 2>&1
timeout 300 python bench.py --config c4 --scale 16 --steps 1 --check > gpurun_out/c4_small.json 2>&1
timeout 600 python bench.py --config c2 > gpurun_out/c2.json 2>&1
timeout 900 python bench.py --config c3 --steps 2 > gpurun_out/c3.json 2>&1
timeout 900 python bench.py --config c4 --steps 2 > gpurun_out/c4.json 2>&1
