#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
GG_POOL_TRACE=1 timeout 900 python tools/bc_timing.py > gpurun_out/bc_timing2.txt 2> gpurun_out/bc_pool.txt
