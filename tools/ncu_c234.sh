#!/bin/bash
# ncu --set full captures of the dominant kernels of C2 (DO-BFS), C3 (fused
# SSSP) and C4 (CC hook, BC backward) -- one launch each, picked with
# --launch-skip from the middle of the run (the first levels are tiny).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=$1
run() {  # name regex skip bench-args...
  local name=$1 re=$2 skip=$3; shift 3
  timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$re" --launch-skip $skip -c 1 \
    -o gpurun_out/${tag}_$name python bench.py "$@" > gpurun_out/${tag}_$name.txt 2>&1
}
run c2_pull 'k_pull_vb' 2 --config c2 --sources 2 --steps 1 --warmup 1
run c2_push 'k_push_etwc' 6 --config c2 --sources 2 --steps 1 --warmup 1
run c3_async 'k_sssp_async' 0 --config c3 --delta 8192 --steps 1 --warmup 1
run c4_cc_hook 'k_push_etwc' 0 --config c4 --lbs ETWC --steps 1 --warmup 1
run c4_bc_bwd 'k_push_etwc' 40 --config c4 --lbs HYBRID --steps 1 --warmup 1
