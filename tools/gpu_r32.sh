#!/bin/bash
# where a fused delta-stepping round's time goes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lb in VERTEX_BASED ETWC; do
  GG_SSSP_PROFILE=1 GG_COOP_PER_SM=1 timeout 600 python bench.py --config c3 --delta 32768 --steps 1 --warmup 1 --lb $lb > gpurun_out/c3_prof_$lb.json 2> gpurun_out/c3_prof_$lb.err
done
GG_SSSP_PROFILE=1 GG_COOP_PER_SM=2 timeout 600 python bench.py --config c3 --delta 32768 --steps 1 --warmup 1 --lb VERTEX_BASED > gpurun_out/c3_prof_coop2.json 2> gpurun_out/c3_prof_coop2.err
for c in 1 2 4; do
  GG_COOP_PER_SM=$c timeout 600 python bench.py --config c2 --sources 16 --fusion > gpurun_out/c2_fused_coop$c.json 2>&1
done
