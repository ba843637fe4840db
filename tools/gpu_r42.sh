#!/bin/bash
# CC EB/EDGE with and without the four-arc hook
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for b in 1 0; do
  GG_EDGE_BATCH4=$b timeout 600 python bench.py --config c4 --steps 2 --lbs EB,EDGE --sources 1 > gpurun_out/c4_b$b.json 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
timeout 600 ncu --metrics $M --clock-control none --kernel-name-base demangled -k "regex:OpHook" -c 20 --csv --log-file gpurun_out/ncu_cc_eb.csv python bench.py --config c4 --lbs EB,EDGE --steps 1 --warmup 1 --sources 1 > gpurun_out/ncu_cc_eb.log 2>&1
