#!/bin/bash
# grid barrier cost; f64 hot-cache size sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
(cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync gridsync.cu && ./gridsync) > gpurun_out/gridsync.txt 2>&1
for kb in 96 160 192; do
  GG_PR_HOT_KB=$kb timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/hot64_$kb.json 2>&1
done
GG_PR_HOT_KB=160 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --fp32-contrib > gpurun_out/hot32_160.json 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu23.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu23.txt
GG_COOP_PER_SM=1 timeout 900 python bench.py --config c3 --steps 2 --warmup 1 --lb VERTEX_BASED > gpurun_out/c3.json 2>&1
GG_COOP_PER_SM=1 timeout 300 python bench.py --config c3 --side 1024 --steps 1 --warmup 1 --lb VERTEX_BASED --check > gpurun_out/c3_check.json 2>&1
