#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/bfs_overhead.py 24 0.0005,0.0002,0.0001,0.00005,0.00002 > gpurun_out/bfs_overhead.txt 2>&1
