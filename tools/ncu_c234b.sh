#!/bin/bash
# Representative launches: capture several and keep all (the summary picks
# the longest): C2 push levels, C4 BC backward levels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=$1
timeout 1500 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:k_push_(etwc|huge)<gg::OpBfs>' -c 14 \
  -o gpurun_out/${tag}_c2_push python bench.py --config c2 --sources 2 --steps 1 --warmup 1 > gpurun_out/${tag}_c2_push.txt 2>&1
timeout 1500 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:OpBcBwdAoS' --launch-skip 2 -c 6 \
  -o gpurun_out/${tag}_c4_bc_bwd python bench.py --config c4 --lbs HYBRID --steps 1 --warmup 1 > gpurun_out/${tag}_c4_bc_bwd.txt 2>&1
