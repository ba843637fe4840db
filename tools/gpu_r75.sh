#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python tools/bfs_overhead.py 24 0.0005,0.001,0.002,0.004,0.0002 > gpurun_out/bfs_theta2.txt 2>&1
