#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/e2e_breakdown.py > gpurun_out/e2e48.txt 2>&1
GG_POOL_MAX_GB=120 timeout 600 python tools/e2e_breakdown.py > gpurun_out/e2e120.txt 2>&1
