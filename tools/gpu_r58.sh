#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi -q -d PCIE 2>/dev/null | grep -i "gen\|width" | head -8 > gpurun_out/pcie.txt
timeout 600 python tools/e2e_breakdown.py 27 > gpurun_out/e2e_breakdown.txt 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/f_c5.json 2> gpurun_out/f_c5.err
timeout 900 python bench.py --config c4 --steps 2 --lbs ETWC,TWC,HYBRID --sources 4 > gpurun_out/f_c4bc.json 2> gpurun_out/f_c4bc.err
