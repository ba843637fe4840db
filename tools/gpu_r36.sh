#!/bin/bash
# refresh every bench line with the current code
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --fp32-contrib > gpurun_out/b_c5_32.json 2> gpurun_out/b_c5_32.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
timeout 600 python bench.py --config c2 --check > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
timeout 600 python bench.py --config c3 --steps 2 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
timeout 900 python bench.py --config c4 --steps 2 --check > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
timeout 300 python bench.py --config c1 --steps 5 > gpurun_out/b_c1.json 2> gpurun_out/b_c1.err
