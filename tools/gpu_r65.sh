#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
GG_ROUND_TRACE=1 timeout 600 python tools/bfs_overhead.py 24 0.0005 > gpurun_out/bfs_rounds.txt 2>&1
